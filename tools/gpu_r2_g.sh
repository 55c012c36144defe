timeout 900 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_kcycle.py -q -x > gpurun_out/pytest_g.log 2>&1; echo pytest_g $?; tail -2 gpurun_out/pytest_g.log
timeout 1500 python tools/loopback_proxy.py --weak --nps 1,2,4,8 > gpurun_out/loopback_weak4.log 2>&1
grep '^{"np"' gpurun_out/loopback_weak4.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['np'], round(d['ms_per_iter'],3), round(d['t_over_t1'],3), d['launches_per_iter'])"
timeout 900 python tools/loopback_breakdown.py > gpurun_out/breakdown2.log 2>&1; tail -22 gpurun_out/breakdown2.log
