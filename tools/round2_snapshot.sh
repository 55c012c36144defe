#!/bin/bash
# Round-2 snapshot on one B200: benches of every config / method, the reference arm, the ncu
# launch list of the default bench and one ncu --set full capture of the dominant kernel of an
# iteration (q = A p with the fused direction update, k_sdia<GPz, ESpmvDotPz>).
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
AMG_SETUP_TIMING=1 timeout 900 python bench.py > gpurun_out/snap2_c4.json 2> gpurun_out/snap2_c4.err
for c in 1 2 3; do timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/snap2_c$c.json 2>/dev/null; done
timeout 900 python bench.py --config 5 --grid 192x192x192 --no-cpu-baseline > gpurun_out/snap2_c5_192.json 2>/dev/null
timeout 900 python bench.py --config 5 --grid 256x256x256 --no-cpu-baseline > gpurun_out/snap2_c5_256.json 2>/dev/null
for m in va3s5cs1 ka1; do timeout 900 python bench.py --method $m --no-cpu-baseline > gpurun_out/snap2_c4_$m.json 2>/dev/null; done
timeout 900 python bench.py --method ka1 --config 2 --no-cpu-baseline > gpurun_out/snap2_c2_ka1.json 2>/dev/null
AMG_SETUP_TIMING=1 timeout 1500 python bench.py --method va3s3cs1 --no-cpu-baseline > gpurun_out/snap2_c4_va3s3cs1.json 2> gpurun_out/snap2_c4_va3s3cs1.err
timeout 900 python bench.py --method va3s3cs1 --config 2 --no-cpu-baseline > gpurun_out/snap2_c2_va3s3cs1.json 2>/dev/null
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/snap2_ref.json 2> gpurun_out/snap2_ref.err
SOLVE_K='regex:^k_(sdia|sell|csrv|csrb|axpy_rr|pcg_init|dense_gemv|xfinal|pupdate|pupdate_fcg|dot|finish|pack|unpack|unpack_pz|coarse_cg|kupd1|kupd2|kpupd|kpq2|collapsed|collapsed_kq|collapsed_kw)$'
AMG_EAGER=1 timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k "$SOLVE_K" -c 600 --csv \
    --log-file gpurun_out/prof2_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
    > gpurun_out/prof2_ncu_launch.log 2>&1
AMG_EAGER=1 timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:k_sdia<amgk::GPz' -s 5 -c 1 -o gpurun_out/prof2_full_pupd -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
    > gpurun_out/prof2_ncu_full.log 2>&1
ncu -i gpurun_out/prof2_full_pupd.ncu-rep --page raw --csv > gpurun_out/prof2_full_pupd_raw.csv 2>/dev/null
echo snapshot done
