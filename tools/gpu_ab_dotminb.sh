# A/B: dot-fused sweep kernels at 6 blocks/SM (40 registers, default) vs 8 (32 registers, libamg_b200_dotminb8.so)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
V8=$PWD/paper_2006_16147_b200/libamg_b200_dotminb8.so
run() {  # name args...
  local n=$1; shift
  for i in 1 2; do
    timeout 900 python bench.py "$@" --no-cpu-baseline > gpurun_out/abd_${n}_def_$i.json 2>/dev/null
    AMG_LIB_PATH=$V8 timeout 900 python bench.py "$@" --no-cpu-baseline > gpurun_out/abd_${n}_mb8_$i.json 2>/dev/null
  done
}
run c4 --steps 20
run c5 --config 5 --grid 256x256x256 --steps 10
run c3 --config 3 --steps 10
run c2 --config 2 --steps 50
run va3s5cs1 --method va3s5cs1 --steps 10
run ka1c2 --method ka1 --config 2 --steps 30
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/abd_*.json')):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        k={e[0]:e[1] for e in d['kernels_per_iteration']}
        print(f.split('/')[-1], round(d['ms_per_step'],3), d['iterations'], 'postsweep_dot', k.get('postsweep_dot'), 'clk', d['clocks']['sm_mhz'])
    except Exception as e: print(f, 'ERR', e)
PY
