import sys, collections, json
sys.path.insert(0,'.')
import torch, paper_2006_16147_b200 as amg
from inputs import config_problem
ctx=amg.Context(device=0)
res={}
for np_ in (1, 8):
    A,b,_=config_problem(4,grid=(256,256,256*np_))
    h=amg.Hierarchy(ctx,A,cfg=amg.make_config(max_coarse_size=200*np_,emulate_ranks=np_,replicate_below_bytes=int(sys.argv[1]) if len(sys.argv)>1 else 64<<20))
    prof=h.profile_iteration(torch.tensor(b,device='cuda:0'),5,cap=4096)
    agg=collections.OrderedDict()
    for k in prof:
        agg.setdefault(k['name'],[0,0.0]); agg[k['name']][0]+=1; agg[k['name']][1]+=k['ms']
    res[np_]=agg
    print(np_, h.sizes(), [h.level_info(l)['format'] for l in range(h.nlevels)])
    h.close(); del A
print(f"{'kernel':20s} {'n1':>4s} {'ms1':>8s} {'n8':>4s} {'ms8':>8s} {'ms8/8':>8s} {'ratio':>6s}")
for name in res[8]:
    c1,t1=res[1].get(name,[0,0.0]); c8,t8=res[8][name]
    print(f"{name:20s} {c1:4d} {t1:8.4f} {c8:4d} {t8:8.4f} {t8/8:8.4f} {t8/8/t1 if t1 else 0:6.2f}")
print('totals', sum(v[1] for v in res[1].values()), sum(v[1] for v in res[8].values())/8)
