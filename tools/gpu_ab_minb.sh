# A/B: dominant-kernel launch bounds (8 blocks/SM with spills vs 6 without), c4 and c2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for i in 1 2; do
  timeout 600 python bench.py --steps 20 --no-cpu-baseline > gpurun_out/ab_def_c4_$i.json 2>/dev/null
  AMG_LIB_PATH=$PWD/paper_2006_16147_b200/libamg_b200_minb6.so timeout 600 python bench.py --steps 20 --no-cpu-baseline > gpurun_out/ab_mb6_c4_$i.json 2>/dev/null
  timeout 600 python bench.py --config 2 --steps 50 --no-cpu-baseline > gpurun_out/ab_def_c2_$i.json 2>/dev/null
  AMG_LIB_PATH=$PWD/paper_2006_16147_b200/libamg_b200_minb6.so timeout 600 python bench.py --config 2 --steps 50 --no-cpu-baseline > gpurun_out/ab_mb6_c2_$i.json 2>/dev/null
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/ab_*.json')):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        r=d['roofline']
        print(f, round(d['ms_per_step'],3), r['kernel'], round(r['ms_per_launch'],4), round(r['frac'],3))
    except Exception as e: print(f, 'ERR', e)
PY
