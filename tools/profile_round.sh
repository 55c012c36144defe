#!/bin/bash
# Round profiling on one B200 (run under gpurun from the repo root):
#   1. bench.py (c4, default) -> gpurun_out/prof_bench_c4.json
#   2. ncu launch list (gpu__time_duration only, eager launches: ncu cannot profile
#      kernel nodes of graphs with conditional nodes) of the same command
#   3. one ncu --set full capture of the level-0 kernels (resid0 / post-sweep / q=Ap)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/prof_bench.json 2> gpurun_out/prof_bench.err || exit 2
# solve-phase kernels only (the GPU setup's kernels run first and would fill the count)
SOLVE_K='regex:^k_(sdia|sell|csrv|csrb|axpy_rr|pcg_init|dense_gemv|xfinal|pupdate|pupdate_fcg|dot|finish|pack|unpack|coarse_cg|kupd1|collapsed|tail)$'
AMG_EAGER=1 timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k "$SOLVE_K" -c ${NCU_COUNT:-3000} --csv \
    --log-file gpurun_out/prof_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} \
    > gpurun_out/prof_ncu_launch.log 2>&1
AMG_EAGER=1 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_sdia -s ${NCU_SKIP:-2} -c 4 \
    -o gpurun_out/prof_full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} \
    > gpurun_out/prof_ncu_full.log 2>&1
ncu -i gpurun_out/prof_full.ncu-rep --page raw --csv > gpurun_out/prof_full_raw.csv 2>/dev/null
echo done
