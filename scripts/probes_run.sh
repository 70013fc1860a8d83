#!/bin/bash
# Re-run the roofline microbenchmarks with an nvidia-smi clock record around each
# (raw logs for profiles/): L2 stream/gather peaks, DMMA peak, FFMA/FFMA2, cluster barrier.
mkdir -p gpurun_out
for p in l2_probe dmma_probe ffma_probe cluster_probe; do
  log=gpurun_out/probe_$p.log
  { echo "# $p $(date -u +%FT%TZ)"; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.draw,temperature.gpu,clocks_event_reasons.active --format=csv;
    nvidia-smi --query-gpu=clocks.sm,clocks_event_reasons.active --format=csv,noheader -lms 50 > /tmp/clk_$p.csv & spid=$!;
    ./scripts/$p; kill $spid; echo "# sm clock samples during the run (MHz, throttle mask):"; sort /tmp/clk_$p.csv | uniq -c; } > $log 2>&1
  echo "== $p"; cat $log | tail -25
done
