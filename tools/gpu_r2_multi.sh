# round 2: multi-rank graph path, replicated fused forms, loopback proxy, bench
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_multirank.py -q -x > gpurun_out/pytest_multirank.log 2>&1; echo multirank $?
tail -30 gpurun_out/pytest_multirank.log
timeout 900 python tools/loopback_proxy.py --eager > gpurun_out/loopback_proxy.log 2> gpurun_out/loopback_proxy.err; echo proxy $?
tail -12 gpurun_out/loopback_proxy.log | cut -c1-400
timeout 1200 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo bench $?
tail -c 3000 gpurun_out/bench_c4.json
