timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log; grep -v "^frame" gpurun_out/t.log | grep -A30 "FAILURES" | head -40
for P in 1 0 1 0; do SWMD_PDL=$P python scripts/e2e_breakdown.py 2>&1 | grep -E "plan.run|times" | sed "s/^/pdl=$P /"; done
