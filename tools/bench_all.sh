python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for a in "--config 4" "--config 3" "--config 2" "--config 5 --grid 192x192x192" "--method ka1"; do
  timeout 900 python bench.py $a --no-cpu-baseline > gpurun_out/ba.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ba.json')); print('$a', round(d['ms_per_step'],3), d['iterations'], round(d['vcycle']['ms'],4), round(d['vcycle']['frac_of_8TBps'],3))"
done
