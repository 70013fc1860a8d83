SWMD_CTA_HOT=1 bash scripts/_zz_run.sh hot1:paper_2107_06433_b200/libswmd.so:
timeout 600 python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline --no-fusion > gpurun_out/plain_c5.log 2>&1 && \
bash scripts/ncu_one.sh c5hot cta2_solve 3 python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline --no-fusion
