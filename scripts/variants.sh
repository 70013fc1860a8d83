#!/bin/bash
# A/B the solve-kernel builds on the GPU box: parity subset + c2/c3 bench per variant.
# usage: scripts/variants.sh "label:SWMD_LIB:SWMD_SOLVE_KERNEL[:SWMD_COST_KERNEL]" ...
mkdir -p gpurun_out
for spec in "$@"; do
  IFS=: read -r label lib pick cpick <<< "$spec"
  export SWMD_LIB=${lib:-}
  export SWMD_SOLVE_KERNEL=${pick:-}
  [ -z "$SWMD_LIB" ] && unset SWMD_LIB
  [ -z "$SWMD_SOLVE_KERNEL" ] && unset SWMD_SOLVE_KERNEL
  export SWMD_COST_KERNEL=${cpick:-}
  [ -z "$SWMD_COST_KERNEL" ] && unset SWMD_COST_KERNEL
  timeout 300 python scripts/parity_report.py c1 c2 c3 > gpurun_out/var_${label}_parity.log 2>&1; cat gpurun_out/var_${label}_parity.log | sed "s/^/$label /"
  timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "solver or c2 or c3 or config or zero or tol or shard or column" > gpurun_out/var_${label}_test.log 2>&1
  echo "$label tests rc=$? $(tail -1 gpurun_out/var_${label}_test.log)"
  for cfg in c2 c3; do
    timeout 300 python bench.py --config $cfg --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/var_${label}_$cfg.log 2>&1
    python - "$label" "$cfg" <<'PY'
import json, sys
label, cfg = sys.argv[1:]
for ln in open(f"gpurun_out/var_{label}_{cfg}.log"):
    if ln.startswith("{"):
        d = json.loads(ln)
        k = d["kernels"]
        print(f"{label} {cfg}: step {d['ms_per_step']*1e3:.1f} us  solve {k['solve_ms']*1e3:.1f} us  cost {k['cost_build_ms']*1e3:.1f} us  e2e {d['e2e']['ms_per_step']*1e3:.1f} us")
        break
else:
    print(label, cfg, "FAILED")
PY
  done
done
