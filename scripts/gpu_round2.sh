#!/bin/bash
# Final GPU session of round 2: full tests, smoke, bench lines, launch list, ncu of the c5 long-query solve
set -u
mkdir -p gpurun_out
NCU=1 bash scripts/gpu_round.sh
timeout 600 python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline --no-fusion > gpurun_out/plain_c5.log 2>&1 && \
bash scripts/ncu_one.sh c5 cta2_solve 3 python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline --no-fusion
