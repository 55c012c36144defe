# determinism probe after the legacy-stream fix: 20 builds of the c5 256^3 analogue
timeout 900 python tools/repro_c5.py 256x256x256 10 > gpurun_out/rpf1.txt 2>&1
timeout 900 env AMG_NO_C16=1 python tools/repro_c5.py 256x256x256 10 > gpurun_out/rpf2.txt 2>&1
for f in rpf1 rpf2; do echo "== $f"; grep build gpurun_out/$f.txt | sed 's/sizes \[[0-9, ]*\] //'; done
