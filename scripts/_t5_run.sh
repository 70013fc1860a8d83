# tcgen05 Gram tile variants: parity + c4 cost build
for L in "$@"; do
  SWMD_LIB=$L timeout 600 python -m pytest tests/test_gpu_batch.py tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "batch or c4 or fp32 or gram" 2>&1 | tail -1
  for r in 1 2; do SWMD_LIB=$L timeout 300 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$L', 'cost ms', round(d['kernels']['cost_build_ms'],3), 'step', round(d['ms_per_step'],2))"; done
done
