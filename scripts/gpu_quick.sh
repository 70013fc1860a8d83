#!/bin/bash
# Quick GPU check: the given pytest files, then short bench lines for the given configs.
mkdir -p gpurun_out
timeout 900 python -m pytest ${TESTS:-tests} -m gpu -x -q -p no:cacheprovider > gpurun_out/q_pytest.log 2>&1
echo "pytest_rc=$?"; tail -3 gpurun_out/q_pytest.log
for cfg in ${CONFIGS:-c2}; do
  timeout 900 python bench.py --config $cfg --steps ${STEPS:-200} --warmup 3 --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/q_bench_$cfg.json 2> gpurun_out/q_bench_$cfg.err
  echo "bench_${cfg}_rc=$?"; tail -2 gpurun_out/q_bench_$cfg.err | cut -c1-300
done
