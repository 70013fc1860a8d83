#!/bin/bash
# Final round-2 GPU session: full tests, smoke, contract bench line, reference arm,
# c3/c4/c5 lines, launch list, ncu --set full summaries of the c2 kernels.
set -u
mkdir -p gpurun_out
bash scripts/gpu_round.sh
bash scripts/ncu_one.sh c2solve reg_solve 2 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-c3 --no-fusion
bash scripts/ncu_one.sh c2cost cost_tmap 2 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-c3 --no-fusion
bash scripts/ncu_one.sh c4mq "reg_solve_mq" 3 python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline
