# A/B of the 16-byte k_axpy_rr (vs profiles/r02_{c4,c2}.json and r02_final_bench_c4.json), then the full GPU suite + smoke
for r in 1 2; do
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/ax_c4_$r.json 2>/dev/null; echo c4 $?
timeout 900 python bench.py --config 2 --no-cpu-baseline > gpurun_out/ax_c2_$r.json 2>/dev/null; echo c2 $?
done
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ax_smoke.log 2>&1; echo smoke $?; tail -1 gpurun_out/ax_smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/ax_pytest_gpu.log 2>&1; echo pytest $?; tail -1 gpurun_out/ax_pytest_gpu.log
