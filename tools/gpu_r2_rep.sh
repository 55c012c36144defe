for rep in 134217728 268435456; do
  timeout 1500 python tools/loopback_proxy.py --weak --nps 1,2,4,8 --rep $rep > gpurun_out/loopback_weak_rep$rep.log 2>&1
  grep '"np"' gpurun_out/loopback_weak_rep$rep.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print($rep, d['np'], round(d['ms_per_iter'],3), round(d['t_over_t1'],3), d['launches_per_iter'])"
done
timeout 900 python tools/loopback_breakdown.py 134217728 > gpurun_out/breakdown_rep128.log 2>&1; tail -14 gpurun_out/breakdown_rep128.log
