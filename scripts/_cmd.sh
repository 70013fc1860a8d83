mkdir -p gpurun_out
timeout 600 python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/plain_c3.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none -k regex:"reg_solve|cost_tmap" -s 2 -c 2 -o gpurun_out/prof_c3 python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c3.log 2>&1; echo ncu_c3_rc=$?
timeout 600 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain_c5.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none -k regex:"cta_solve|cost_tmap" -s 8 -c 2 -o gpurun_out/prof_c5 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c5.log 2>&1; echo ncu_c5_rc=$?
