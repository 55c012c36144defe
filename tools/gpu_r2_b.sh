# round 2 (b): K-cycle multi-rank, multirank, full parity, weak loopback proxy
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_kcycle.py tests/test_gpu_multirank.py -q > gpurun_out/pytest_kc_mr.log 2>&1; echo kc_mr $?
tail -15 gpurun_out/pytest_kc_mr.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -q > gpurun_out/pytest_parity.log 2>&1; echo parity $?
tail -15 gpurun_out/pytest_parity.log
timeout 1500 python tools/loopback_proxy.py --weak --nps 1,2,4,8 > gpurun_out/loopback_weak.log 2> gpurun_out/loopback_weak.err; echo proxyw $?
tail -6 gpurun_out/loopback_weak.log | cut -c1-300
