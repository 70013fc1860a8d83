# cost build: DFMA side path for the words past the full DMMA tiles vs a padded tile
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py -x -q -p no:cacheprovider 2>&1 | tail -2
for m in 1 0 1 0; do SWMD_COST_EXTRA=$m python bench.py --steps 500 --no-cpu-baseline --no-c3 --no-fusion 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); k=d['kernels']; print('extra=$m c2 cost us', round(k['cost_build_ms']*1e3,2), 'solve', round(k['solve_ms']*1e3,2), 'step', round(d['ms_per_step']*1e3,2), 'e2e', round(d['e2e']['ms_per_step']*1e3,1))"; done
