timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "c4 or f32 or batch" -p no:cacheprovider 2>&1 | tail -1
timeout 600 python scripts/c4_probe.py 2 > gpurun_out/c4_mq.log 2>&1; echo "== mq"; grep -E "rep 2" gpurun_out/c4_mq.log
bash scripts/ab.sh cur:build_ab/lib_cur.so: 2>&1 | grep -E "tests|flat|model\)"
