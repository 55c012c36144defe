# A/B of the block-per-row collapsed-level GEMV with 16-byte loads (vs profiles/r02_{c4,c2}.json)
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kcycle.py -m gpu -q -x > gpurun_out/pytest_collapsed2.log 2>&1; echo pytest $?; tail -1 gpurun_out/pytest_collapsed2.log
for r in 1 2; do
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/wc2_c4_$r.json 2>/dev/null; echo c4 $?
timeout 900 python bench.py --config 2 --no-cpu-baseline > gpurun_out/wc2_c2_$r.json 2>/dev/null; echo c2 $?
done
