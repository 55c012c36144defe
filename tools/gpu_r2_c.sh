# round 2 (c): everything on the GPU after the distributed setup landed
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke $?; tail -2 gpurun_out/smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_all.log 2>&1; echo pytest $?
tail -8 gpurun_out/pytest_gpu_all.log
