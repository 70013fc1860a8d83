export SWMD_SOLVE_KERNEL=c
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "query_length or large_config or column_length or zero or tol or shard" > gpurun_out/clu_pytest.log 2>&1; echo "clu_pytest_rc=$?"; grep -v "^frame" gpurun_out/clu_pytest.log | tail -3
for C in 1 2 4; do SWMD_DEBUG=1 SWMD_CLUSTER=$C timeout 600 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --no-fusion > gpurun_out/clu_c5_$C.json 2> gpurun_out/clu_c5_$C.err; echo "clu C=$C rc=$?"; python -c "import json; d=json.load(open('gpurun_out/clu_c5_$C.json')); print('C=$C solve ms', d['kernels']['solve_ms'])"; done
unset SWMD_SOLVE_KERNEL
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "c4 or f32 or batch" > gpurun_out/f32_pytest.log 2>&1; echo "f32_pytest_rc=$?"; tail -2 gpurun_out/f32_pytest.log
timeout 600 python scripts/c4_probe.py 2 > gpurun_out/c4_ffma2.log 2>&1; echo "== ffma2"; grep -E "rep 2|v_r" gpurun_out/c4_ffma2.log
SWMD_LIB=build_ab/lib_base.so timeout 600 python scripts/c4_probe.py 2 > gpurun_out/c4_base2.log 2>&1; echo "== base"; grep -E "rep 2|v_r" gpurun_out/c4_base2.log
