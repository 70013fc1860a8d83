#!/bin/bash
# cost-build start-up A/B: bash scripts/_cb_run.sh label:lib ...  (parity, then the c2 bench line's cost build / step)
mkdir -p gpurun_out
for spec in "$@"; do
  IFS=: read -r label lib <<< "$spec"
  export SWMD_LIB=$lib
  timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/cb_${label}_test.log 2>&1
  echo "$label tests rc=$? $(tail -1 gpurun_out/cb_${label}_test.log)"
  for rep in 1 2; do
    timeout 600 python bench.py --steps 1000 --no-cpu-baseline --no-c3 --no-fusion | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$label c2 cost', round(d['kernels']['cost_build_ms']*1e3,2), 'solve', round(d['kernels']['solve_ms']*1e3,2), 'step', round(d['ms_per_step']*1e3,2), 'e2e', round(d['e2e']['ms_per_step']*1e3,1))"
  done
done
