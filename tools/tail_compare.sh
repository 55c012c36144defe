python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_tail.py tests/test_gpu_kcycle.py -x -q 2>&1 | tail -2
for args in "--config 2" "--config 4" "--config 2 --method ka1" "--method ka1"; do
  for t in 0 40000; do
    timeout 600 python bench.py $args --tail-rows $t --no-cpu-baseline > gpurun_out/tc.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/tc.json')); print('$args tail=$t', round(d['ms_per_step'],3), d['iterations'], round(d['vcycle']['ms'],4))"
  done
done
