import os,sys,json,statistics
os.environ["MANDEL_B200_LIB"]=sys.argv[1] if sys.argv[1]!="base" else ""
sys.path.insert(0,"/root/repo")
import torch, paper_2206_02255_b200 as mb, workloads as W
flush=torch.empty(256<<20,dtype=torch.uint8,device="cuda")
w=W.CONFIGS["C3"]; out=torch.empty((w.n,w.n),dtype=torch.int32,device="cuda"); ws=mb.workspace(w.n,w.g,w.r,w.B)
def ev(fn):
    fn();fn();ts=[]
    for _ in range(7):
        flush.zero_(); s,e=torch.cuda.Event(True),torch.cuda.Event(True); s.record(); fn(); e.record(); e.synchronize(); ts.append(s.elapsed_time(e))
    return round(statistics.median(ts),4)
A=lambda **k: mb.ask(w.region,w.n,w.maxdwell,w.g,w.r,w.B,out=out,ws=ws,**k)
r={"v":sys.argv[1],"plain":ev(lambda:A()),"sampled":ev(lambda:A(tile_cost="sampled"))}
A(tile_cost="sampled",timing=True); torch.cuda.synchronize()
kt={}
for k in mb.kernel_times(): kt[k["kind"]]=round(kt.get(k["kind"],0)+k["ms"],4)
A(timing=True); torch.cuda.synchronize()
kp={}
for k in mb.kernel_times(): kp[k["kind"]]=round(kp.get(k["kind"],0)+k["ms"],4)
r["k_sampled"]=kt; r["k_plain"]=kp
print(json.dumps(r))
