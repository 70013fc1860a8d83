#!/bin/bash
# One GPU session: tests, smoke, bench lines (c2 contract line, reference arm, c3/c4/c5), launch list.
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest_rc=$?"; grep -E "passed|failed" gpurun_out/pytest_gpu.log | tail -2
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke_rc=$?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench_rc=$?"
tail -1 gpurun_out/bench_default.json | cut -c1-400
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_reference.json 2>/dev/null; echo "ref_rc=$?"; tail -1 gpurun_out/bench_reference.json | cut -c1-300
for cfg in ${CONFIGS-c3 c4 c5}; do
  timeout 900 python bench.py --config $cfg --steps ${STEPS:-10} --warmup 3 > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.err; echo "bench_${cfg}_rc=$?"
done
if [ "${NCU:-1}" = "1" ]; then
  timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-c3 --no-fusion > gpurun_out/plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
      python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-c3 --no-fusion > gpurun_out/ncu_launch.log 2>&1; echo "ncu_launch_rc=$?"
fi
