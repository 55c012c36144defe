# 16-bit columns on the K-cycle / short-row hierarchies: default (rows >= 4 entries), >= 16, off
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for i in 1 2; do
  for args in "--method ka1 --config 2 --steps 30" "--method ka1 --steps 10" "--config 2 --steps 50" "--method va3s3cs1 --config 2 --steps 30" "--config 1 --steps 100"; do
    tag=$(echo "$args" | tr -d ' -')
    timeout 900 python bench.py $args --no-cpu-baseline > gpurun_out/c16b_${tag}_m4_$i.json 2>/dev/null
    AMG_C16_MIN_MEAN=16 timeout 900 python bench.py $args --no-cpu-baseline > gpurun_out/c16b_${tag}_m16_$i.json 2>/dev/null
    AMG_NO_C16=1 timeout 900 python bench.py $args --no-cpu-baseline > gpurun_out/c16b_${tag}_off_$i.json 2>/dev/null
  done
done
python - <<'PY'
import json,glob,collections
res=collections.defaultdict(list)
for f in sorted(glob.glob('gpurun_out/c16b_*.json')):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        key=f.split('/')[-1].rsplit('_',1)[0]
        res[key].append((round(d['ms_per_step'],3), round(d['vcycle']['ms'],4), d['iterations']))
    except Exception as e: print(f,'ERR',e)
for k,v in sorted(res.items()): print(k, v)
PY
