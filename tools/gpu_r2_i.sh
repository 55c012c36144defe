timeout 1800 python -m pytest tests/test_gpu_parity.py -k "compact or vcycle_parity or pcg_parity" tests/test_gpu_multirank.py -q -x > gpurun_out/pytest_i.log 2>&1; echo pytest_i $?; tail -3 gpurun_out/pytest_i.log
for i in 1 2; do timeout 900 python bench.py --config 2 --steps 50 --no-cpu-baseline > gpurun_out/i_c2_$i.json 2>/dev/null; timeout 900 python bench.py --steps 20 --no-cpu-baseline > gpurun_out/i_c4_$i.json 2>/dev/null; done
python -c "
import json
for f in ['i_c2_1','i_c2_2','i_c4_1','i_c4_2']:
    d=json.loads(open('gpurun_out/'+f+'.json').read().strip().splitlines()[-1]); print(f, d['ms_per_step'], d['vcycle']['ms'])"
