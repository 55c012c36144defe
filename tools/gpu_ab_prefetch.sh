# A/B: L2 prefetch of the epilogue operands before each row reduction (default build) vs none
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
NOPF=$PWD/paper_2006_16147_b200/libamg_b200_nopf.so
for i in 1 2; do
  for args in "--config 4 --steps 20" "--config 5 --grid 256x256x256 --steps 10" "--config 2 --steps 50" "--config 3 --steps 10"; do
    tag=$(echo "$args" | tr -d ' -')
    timeout 900 python bench.py $args --no-cpu-baseline > gpurun_out/pf_${tag}_on_$i.json 2>/dev/null
    AMG_LIB_PATH=$NOPF timeout 900 python bench.py $args --no-cpu-baseline > gpurun_out/pf_${tag}_off_$i.json 2>/dev/null
  done
done
python - <<'PY'
import json,glob,collections
res=collections.defaultdict(list)
for f in sorted(glob.glob('gpurun_out/pf_*.json')):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        key=f.split('/')[-1].rsplit('_',1)[0]
        res[key].append((round(d['ms_per_step'],3), round(d['vcycle']['ms'],4), round(d['roofline']['ms_per_launch'],4), d['roofline']['kernel']))
    except Exception as e: print(f,'ERR',e)
for k,v in sorted(res.items()): print(k, v)
PY
