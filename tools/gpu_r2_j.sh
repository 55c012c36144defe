# full verification (smoke, every GPU test, default bench) + A/B of the |a| recompute cut (AMG_ABS_ROW_CUT)
bash tools/gpu_r2_full.sh
for i in 1 2; do
  for args in "--config 4 --steps 20" "--config 5 --grid 256x256x256 --steps 10" "--config 3 --steps 10"; do
    tag=$(echo "$args" | tr -d ' -')
    for cut in 40 20 1000; do
      AMG_ABS_ROW_CUT=$cut timeout 900 python bench.py $args --no-cpu-baseline > gpurun_out/abs_${tag}_c${cut}_$i.json 2>/dev/null
    done
  done
done
python - <<'PY'
import json,glob,collections
res=collections.defaultdict(list)
for f in sorted(glob.glob('gpurun_out/abs_*.json')):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        key=f.split('/')[-1].rsplit('_',1)[0]
        ps=[round(k[1],4) for k in d['kernels_per_vcycle'] if k[0].startswith('postsweep')]
        res[key].append((round(d['ms_per_step'],3), round(d['vcycle']['ms'],4), ps))
    except Exception as e: print(f,'ERR',e)
for k,v in sorted(res.items()): print(k, v)
PY
