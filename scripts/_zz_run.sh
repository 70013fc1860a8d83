# c5 long-query solve A/B: cta2_solve variants (rows per warp step, warps per column, CTAs per SM)
mkdir -p gpurun_out
run() { # label lib per_sm pick
  export SWMD_LIB=$2 SWMD_CTA_PER_SM=$3 SWMD_SOLVE_KERNEL=$4
  [ -z "$SWMD_SOLVE_KERNEL" ] && unset SWMD_SOLVE_KERNEL
  [ -z "$SWMD_CTA_PER_SM" ] && unset SWMD_CTA_PER_SM
  timeout 600 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --no-fusion > gpurun_out/zz_$1.json 2> gpurun_out/zz_$1.err
  python -c "import json; d=json.loads(open('gpurun_out/zz_$1.json').read().strip().splitlines()[-1]); print('$1', 'solve ms', round(d['kernels']['solve_ms'],2))" || tail -3 gpurun_out/zz_$1.err
}
SWMD_LIB=build_ab/lib_r4w4m2.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py -x -q -p no:cacheprovider > gpurun_out/zz_pytest.log 2>&1; tail -3 gpurun_out/zz_pytest.log
run r2m3 build_ab/lib_r2m3.so 3 ""
run r4w4m2 build_ab/lib_r4w4m2.so 2 ""
run r4w8m1 build_ab/lib_r4w8m1.so 1 ""
run r4w2m4 build_ab/lib_r4w2m4.so 4 ""
run r4w4m3 build_ab/lib_r4w4m3.so 3 ""
