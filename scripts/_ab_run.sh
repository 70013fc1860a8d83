bash scripts/ab.sh cur:build_ab/lib_cur.so: sf1:build_ab/lib_sf1.so: cur2:build_ab/lib_cur.so: sf12:build_ab/lib_sf1.so: 2>&1 | grep -E "tests|flat|model\)"
for v in s32on s32off; do SWMD_LIB=build_ab/lib_$v.so timeout 600 python scripts/c4_probe.py 2 > gpurun_out/c4_$v.log 2>&1; echo "== $v"; grep -E "rep 2" gpurun_out/c4_$v.log; done
SWMD_LIB=build_ab/lib_s32off.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "c4 or f32 or batch" -p no:cacheprovider 2>&1 | tail -1
