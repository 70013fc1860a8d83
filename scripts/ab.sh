#!/bin/bash
# A/B solve builds: scripts/ab.sh "label:lib:pick" ...  (parity + order probe per build)
mkdir -p gpurun_out
for spec in "$@"; do
  IFS=: read -r label lib pick <<< "$spec"
  export SWMD_LIB=$lib
  if [ -n "$pick" ]; then export SWMD_SOLVE_KERNEL=$pick; else unset SWMD_SOLVE_KERNEL; fi
  timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/ab_${label}_test.log 2>&1
  echo "$label tests rc=$? $(tail -1 gpurun_out/ab_${label}_test.log)"
  timeout 600 python scripts/order_probe.py ${CFG:-c2} ${REPS:-300} 2>&1 | sed "s/^/$label /"
done
