# Final round-2 ncu evidence on the final code: launch list (time + DRAM bytes per launch) of the
# default bench's solve kernels, and one --set full capture of the dominant kernel of an iteration.
SOLVE_K='regex:^k_(sdia|sell|csrv|csrb|axpy_rr|pcg_init|dense_gemv|xfinal|pupdate|pupdate_fcg|dot|finish|pack|unpack|unpack_pz|coarse_cg|kupd1|kupd2|kpupd|kpq2|collapsed|collapsed_kq|collapsed_kw)$'
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/fin_bench.json 2>/dev/null; echo bench $?
AMG_EAGER=1 timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k "$SOLVE_K" -c 600 --csv \
    --log-file gpurun_out/fin_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
    > gpurun_out/fin_ncu_launch.log 2>&1; echo launches $?
AMG_EAGER=1 timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:k_sdia<amgk::GPz' -s 5 -c 1 -o gpurun_out/fin_full_pupd -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
    > gpurun_out/fin_ncu_full.log 2>&1; echo full $?
ncu -i gpurun_out/fin_full_pupd.ncu-rep --page raw --csv > gpurun_out/fin_full_pupd_raw.csv 2>/dev/null
ncu -i gpurun_out/fin_full_pupd.ncu-rep --page details --csv > gpurun_out/fin_full_pupd_details.csv 2>/dev/null
echo done
