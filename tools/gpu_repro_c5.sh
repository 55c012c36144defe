# Determinism probe of the c5 analogue (one A/B run took 36 iterations instead of 19): repeated builds
# per setting, each line: sizes, aggregate hash, iterations of 4 solves, x / z hashes
set -x
timeout 600 python tools/repro_c5.py 128x128x128 12 > gpurun_out/rp_128.txt 2>&1
timeout 900 env AMG_EAGER=1 python tools/repro_c5.py 256x256x256 6 > gpurun_out/rp_eager.txt 2>&1
timeout 900 env AMG_NO_C16=1 python tools/repro_c5.py 256x256x256 6 > gpurun_out/rp_noc16.txt 2>&1
timeout 900 env AMG_PDL=0 python tools/repro_c5.py 256x256x256 6 > gpurun_out/rp_nopdl.txt 2>&1
timeout 900 python tools/repro_c5.py 256x256x256 6 > gpurun_out/rp_def.txt 2>&1
for f in rp_128 rp_eager rp_noc16 rp_nopdl rp_def; do echo "== $f"; grep build gpurun_out/$f.txt | sed 's/sizes \[[0-9, ]*\] //'; done
