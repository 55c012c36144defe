# 16-bit columns: GPU parity (all parity + multi-rank tests incl. the new bitwise c16 == c32 cases), then A/B
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py tests/test_gpu_kcycle.py -m gpu -q -x > gpurun_out/pytest_k.log 2>&1; echo pytest_k $?; tail -3 gpurun_out/pytest_k.log
for i in 1 2; do
  for args in "--config 4 --steps 20" "--config 5 --grid 256x256x256 --steps 10" "--config 2 --steps 50" "--config 3 --steps 10"; do
    tag=$(echo "$args" | tr -d ' -')
    timeout 900 python bench.py $args --no-cpu-baseline > gpurun_out/c16_${tag}_on_$i.json 2>/dev/null
    AMG_NO_C16=1 timeout 900 python bench.py $args --no-cpu-baseline > gpurun_out/c16_${tag}_off_$i.json 2>/dev/null
  done
done
python - <<'PY'
import json,glob,collections
res=collections.defaultdict(list)
for f in sorted(glob.glob('gpurun_out/c16_*.json')):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        key=f.split('/')[-1].rsplit('_',1)[0]
        res[key].append((round(d['ms_per_step'],3), round(d['vcycle']['ms'],4), d['iterations']))
    except Exception as e: print(f,'ERR',e)
for k,v in sorted(res.items()): print(k, v)
PY
