# A/B: fewer blocks for small operators so the next (PDL) kernel can become resident early
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for i in 1 2; do
  for knob in none 40000:4 40000:2 300000:4 300000:6; do
    for args in "--config 2 --steps 50" "--config 4 --steps 20" "--config 2 --method ka1 --steps 50"; do
      tag=$(echo "$args" | tr -d ' -')
      k=$(echo $knob | tr ':' 'x')
      if [ $knob = none ]; then env=""; else env="AMG_SMALL_GRID=$knob"; fi
      env $env timeout 600 python bench.py $args --no-cpu-baseline > gpurun_out/sg_${tag}_${k}_$i.json 2>/dev/null
    done
  done
done
python - <<'PY'
import json,glob,collections
res=collections.defaultdict(list)
for f in sorted(glob.glob('gpurun_out/sg_*.json')):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        key=f.split('/')[-1].rsplit('_',1)[0]
        res[key].append((round(d['ms_per_step'],3), round(d['vcycle']['ms'],4)))
    except Exception as e: print(f,'ERR',e)
for k,v in sorted(res.items()): print(k, v)
PY
