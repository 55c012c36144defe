python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log; grep -E "^FAILED|Error" gpurun_out/pytest_gpu.log | head
timeout 900 python bench.py --method ka1 --no-cpu-baseline > gpurun_out/snap_c4_ka1.json 2>/dev/null
timeout 900 python bench.py --method ka1 --config 2 --no-cpu-baseline > gpurun_out/snap_c2_ka1.json 2>/dev/null
python -c "
import json
for f in ['snap_c4_ka1','snap_c2_ka1']:
    d=json.load(open('gpurun_out/%s.json'%f)); print(f, d['ms_per_step'], d['iterations'], d['vcycle']['ms'])"
SOLVE_K='regex:^k_(sdia|sell|csrv|csrb|axpy_rr|pcg_init|dense_gemv|xfinal|pupdate|pupdate_fcg|dot|finish|pack|unpack|coarse_cg|kupd1|kpupd|kupd2|tail)$'
AMG_EAGER=1 timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k "$SOLVE_K" -c 3000 --csv --log-file gpurun_out/prof_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/prof_ncu_launch.log 2>&1
tail -2 gpurun_out/prof_ncu_launch.log
