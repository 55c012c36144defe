nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
bash tools/gpu_ab_minb.sh > gpurun_out/ab.log 2>&1; tail -10 gpurun_out/ab.log
AMG_EAGER=1 timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:k_sdia<amgk::GPz' -s 5 -c 1 -o gpurun_out/prof2_full_pupd -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
    > gpurun_out/prof2_ncu_full.log 2>&1; echo ncu $?
ncu -i gpurun_out/prof2_full_pupd.ncu-rep --page raw --csv > gpurun_out/prof2_full_pupd_raw.csv 2>/dev/null
ncu -i gpurun_out/prof2_full_pupd.ncu-rep --page details --csv > gpurun_out/prof2_full_pupd_details.csv 2>/dev/null
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/snap2_ref.json 2> gpurun_out/snap2_ref.err; echo ref $?
timeout 1500 python tools/loopback_proxy.py --weak --nps 1,2 > gpurun_out/loopback_weak2.log 2>&1
python - <<'PY'
import sys; sys.path.insert(0,'.')
import torch, paper_2006_16147_b200 as amg
from inputs import config_problem
A,b,_=config_problem(4,grid=(256,256,512))
ctx=amg.Context(device=0)
h=amg.Hierarchy(ctx,A,cfg=amg.make_config(max_coarse_size=400,emulate_ranks=2))
prof=h.profile_iteration(torch.tensor(b,device='cuda:0'),5)
import collections
agg=collections.OrderedDict()
for k in prof: agg.setdefault(k['name'],[0,0.0]); agg[k['name']][0]+=1; agg[k['name']][1]+=k['ms']
tot=sum(v[1] for v in agg.values())
for n,(c,t) in sorted(agg.items(), key=lambda x:-x[1][1]): print(f"{n:20s} {c:4d} {t:8.4f} {t/tot:6.3f}")
print('total kernel ms per iteration', tot)
PY
