# ncu --set full of the c5 level-0 kernels (27-point SDIA): post-sweep with dot vs residual
AMG_EAGER=1 timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:k_sdia<amgk::GVec, amgk::EPost1<\(bool\)1' -s 3 -c 1 -o gpurun_out/c5_post -f \
    python bench.py --config 5 --grid 256x256x256 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/c5_ncu1.log 2>&1; echo ncu1 $?
AMG_EAGER=1 timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:k_sdia<amgk::GVec, amgk::EResid>' -s 6 -c 1 -o gpurun_out/c5_resid -f \
    python bench.py --config 5 --grid 256x256x256 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/c5_ncu2.log 2>&1; echo ncu2 $?
for r in c5_post c5_resid; do ncu -i gpurun_out/$r.ncu-rep --page details --csv > gpurun_out/${r}_details.csv 2>/dev/null; ncu -i gpurun_out/$r.ncu-rep --page source --csv > gpurun_out/${r}_source.csv 2>/dev/null; done
ls -la gpurun_out/c5_*
