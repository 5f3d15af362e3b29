set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 120 python -c "
import sys; sys.path.insert(0,'.')
import torch, numpy as np, oracle, workloads as W, paper_2206_02255_b200 as mb
for w in list(W.random_small_workloads(30, seed=W.SEED + 12, max_n=512)):
    ws = mb.workspace(w.n, w.g, w.r, w.B)
    for sch in ('b200','flow'):
        out = torch.full((w.n, w.n), -9, dtype=torch.int32, device='cuda')
        mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, out=out, ws=ws, scheme=sch, stats=True)
        torch.cuda.synchronize()
        A, st = oracle.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B)
        o = out.cpu().numpy()
        bad = np.argwhere(o != A)
        print(w.name, w.n, w.g, w.r, w.B, sch, 'mismatches', len(bad), bad[:6].tolist(), [int(o[i,j]) for i,j in bad[:6]], [int(A[i,j]) for i,j in bad[:6]])
    if w.n <= 8 and len(bad):
        print(o); print(A)
"
