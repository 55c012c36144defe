nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py tests/test_gpu_kcycle.py tests/test_gpu_tail.py -q -x > gpurun_out/pytest_h.log 2>&1; echo pytest_h $?; tail -3 gpurun_out/pytest_h.log
for i in 1 2; do
  for args in "--config 2 --steps 50" "--config 4 --steps 20" "--config 5 --grid 256x256x256 --steps 10"; do
    tag=$(echo "$args" | tr -d ' -')
    AMG_SETUP_TIMING=1 timeout 900 python bench.py $args --no-cpu-baseline > gpurun_out/c2x_${tag}_on_$i.json 2> gpurun_out/c2x_${tag}_on_$i.err
    AMG_NO_COLLAPSE2=1 timeout 900 python bench.py $args --no-cpu-baseline > gpurun_out/c2x_${tag}_off_$i.json 2>/dev/null
  done
done
python - <<'PY'
import json,glob,collections
res=collections.defaultdict(list)
for f in sorted(glob.glob('gpurun_out/c2x_*.json')):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        key=f.split('/')[-1].rsplit('_',1)[0]
        res[key].append((round(d['ms_per_step'],3), round(d['vcycle']['ms'],4), round(d['setup_s'],1)))
    except Exception as e: print(f,'ERR',e)
for k,v in sorted(res.items()): print(k, v)
PY
grep "second collapse" gpurun_out/c2x_*on_1.err
