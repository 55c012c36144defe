#!/bin/bash
# Full GPU snapshot: tests, smoke, benches for every method/config, profiles.
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1 || exit 1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
AMG_SETUP_TIMING=1 timeout 900 python bench.py > gpurun_out/snap_c4.json 2> gpurun_out/snap_c4.err
for c in 1 2 3; do timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/snap_c$c.json 2>/dev/null; done
timeout 900 python bench.py --config 5 --grid 192x192x192 --no-cpu-baseline > gpurun_out/snap_c5_192.json 2>/dev/null
AMG_SETUP_TIMING=1 timeout 900 python bench.py --config 5 --grid 256x256x256 --no-cpu-baseline > gpurun_out/snap_c5_256.json 2> gpurun_out/snap_c5_256.err
for m in va3s5cs1 ka1 invk; do timeout 900 python bench.py --method $m --no-cpu-baseline > gpurun_out/snap_c4_$m.json 2>/dev/null; done
timeout 900 python bench.py --method ka1 --config 2 --no-cpu-baseline > gpurun_out/snap_c2_ka1.json 2>/dev/null
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/snap_ref.json 2>/dev/null
bash tools/profile_round.sh > gpurun_out/prof_round.log 2>&1
echo snapshot done
