nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_kcycle.py tests/test_gpu_invk.py -q -x > gpurun_out/pytest_f.log 2>&1; echo pytest_f $?
tail -3 gpurun_out/pytest_f.log
for i in 1 2; do timeout 600 python bench.py --steps 20 --no-cpu-baseline > gpurun_out/f_c4_$i.json 2>/dev/null; done
python -c "
import json
for i in (1,2):
    d=json.loads(open(f'gpurun_out/f_c4_{i}.json').read().strip().splitlines()[-1]); print('c4', d['ms_per_step'], d['roofline']['ms_per_launch'])"
timeout 1500 python tools/loopback_proxy.py --weak --nps 1,2,4,8 > gpurun_out/loopback_weak3.log 2>&1; tail -5 gpurun_out/loopback_weak3.log | cut -c1-220
timeout 900 python tools/loopback_proxy.py --nps 1,2,4,8 > gpurun_out/loopback_strong3.log 2>&1; tail -5 gpurun_out/loopback_strong3.log | cut -c1-220
bash tools/gpu_ab_l2.sh > gpurun_out/l2.log 2>&1; tail -12 gpurun_out/l2.log
