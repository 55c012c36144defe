# SDIA offsets in a register (k_sdia<G,E,true>): bitwise tests, then A/B: on (chunk 8) / on (chunk 4 build) / off
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "register or vcycle_parity or pcg_parity" > gpurun_out/pytest_m.log 2>&1; echo pytest_m $?; tail -3 gpurun_out/pytest_m.log
OC4=$PWD/paper_2006_16147_b200/libamg_b200_oc4.so
for i in 1 2; do
  for args in "--config 4 --steps 20" "--config 5 --grid 256x256x256 --steps 10" "--config 3 --steps 10" "--config 2 --steps 50"; do
    tag=$(echo "$args" | tr -d ' -')
    timeout 900 python bench.py $args --no-cpu-baseline > gpurun_out/ofr_${tag}_on8_$i.json 2>/dev/null
    AMG_LIB_PATH=$OC4 timeout 900 python bench.py $args --no-cpu-baseline > gpurun_out/ofr_${tag}_on4_$i.json 2>/dev/null
    AMG_SDIA_OFFREG=0 timeout 900 python bench.py $args --no-cpu-baseline > gpurun_out/ofr_${tag}_off_$i.json 2>/dev/null
  done
done
python - <<'PY'
import json,glob,collections
res=collections.defaultdict(list)
for f in sorted(glob.glob('gpurun_out/ofr_*.json')):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        key=f.split('/')[-1].rsplit('_',1)[0]
        k=d['kernels_per_iteration']
        l0=[(n,t) for n,t,_ in k if n in ('resid0','postsweep_dot','spmv_dot_pupd')]
        res[key].append((round(d['ms_per_step'],3), round(d['vcycle']['ms'],4), d['iterations'], [round(t,4) for n,t in l0][:1]+[round(t,4) for n,t in l0][-2:]))
    except Exception as e: print(f,'ERR',e)
for k,v in sorted(res.items()): print(k, v)
PY
