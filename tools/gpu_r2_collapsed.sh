# A/B of the warp-per-row collapsed-level GEMV: parity tests that take the collapsed paths,
# then c4 / c2 / c2 KA1 bench lines (per-kernel times in kernels_per_iteration)
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kcycle.py tests/test_gpu_paper_method.py -m gpu -q -x > gpurun_out/pytest_collapsed.log 2>&1; echo pytest $?; tail -2 gpurun_out/pytest_collapsed.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/wc_c4.json 2>gpurun_out/wc_c4.err; echo c4 $?
timeout 900 python bench.py --config 2 --no-cpu-baseline > gpurun_out/wc_c2.json 2>/dev/null; echo c2 $?
timeout 900 python bench.py --method ka1 --config 2 --no-cpu-baseline > gpurun_out/wc_c2_ka1.json 2>/dev/null; echo c2ka1 $?
timeout 900 python bench.py --method ka1 --no-cpu-baseline > gpurun_out/wc_c4_ka1.json 2>/dev/null; echo c4ka1 $?
