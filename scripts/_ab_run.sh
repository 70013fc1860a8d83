bash scripts/ab.sh cur:build_ab/lib_cur.so: u0r1:build_ab/lib_u0r1.so: u0r2:build_ab/lib_u0r2.so: 2>&1 | grep -E "tests|flat"
for L in cur u0r1 u0r2; do SWMD_LIB=build_ab/lib_$L.so timeout 600 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline --no-fusion | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$L c3 solve', d['kernels']['solve_ms'])"; done
