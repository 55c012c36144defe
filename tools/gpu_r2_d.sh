nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_paper_method.py tests/test_gpu_parity.py tests/test_gpu_setup.py -q -x > gpurun_out/pytest_d.log 2>&1; echo pytest_d $?
tail -4 gpurun_out/pytest_d.log
bash tools/round2_snapshot.sh > gpurun_out/snap2.log 2>&1; echo snap $?
