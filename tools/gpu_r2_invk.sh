nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
lscpu | head -20 > gpurun_out/host_lscpu.txt; nproc >> gpurun_out/host_lscpu.txt; free -g >> gpurun_out/host_lscpu.txt
timeout 900 python -m pytest tests/test_gpu_invk.py -q > gpurun_out/pytest_invk.log 2>&1; echo invk $?
tail -30 gpurun_out/pytest_invk.log
timeout 1500 python -m pytest tests -m gpu -q --deselect tests/test_gpu_invk.py > gpurun_out/pytest_gpu.log 2>&1; echo pytest $?
tail -5 gpurun_out/pytest_gpu.log
