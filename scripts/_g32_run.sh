# c4 Gram kernels: FFMA 64x64 (default), FFMA 128x128 (b), 3xTF32 mma.sync (m): parity + bench
export SWMD_LIB=${SWMD_LIB:-paper_2107_06433_b200/libswmd.so}
for m in b; do SWMD_GRAM32=$m timeout 600 python -m pytest tests/test_gpu_batch.py tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "batch or c4 or fp32" 2>&1 | tail -1; done
for m in f b f b; do SWMD_GRAM32=$m python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$m', 'cost ms', round(d['kernels']['cost_build_ms'],3), 'solves', round(d['kernels']['solves_ms'],2), 'step', round(d['ms_per_step'],2))"; done
