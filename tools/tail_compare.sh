python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for args in "--config 2" "--config 2 --method ka1" "--method ka1"; do
  for t in "--tail-bytes 0" "--tail-bytes 131072" "--tail-bytes 524288" "--tail-bytes 2097152"; do
    timeout 600 python bench.py $args $t --no-cpu-baseline > gpurun_out/tc.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/tc.json')); print('$args $t', round(d['ms_per_step'],3), d['iterations'], round(d['vcycle']['ms'],4))"
  done
done
