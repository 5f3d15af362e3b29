set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 120 python -c "
import sys; sys.path.insert(0,'.')
import torch, numpy as np, oracle, workloads as W, paper_2206_02255_b200 as mb
w = W.C1
ws = mb.workspace(w.n, w.g, w.r, w.B)
out = mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, ws=ws, scheme='flow', stats=True)
torch.cuda.synchronize()
A, st = oracle.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B)
o = out.cpu().numpy()
print('C1 flow mismatches', int((o != A).sum()))
print(mb.ask_stats(ws))
print(st)
"
echo rc=$?
timeout 600 python -m pytest tests -m gpu -x -q -k "flow" > gpurun_out/pytest33.log 2>&1; tail -5 gpurun_out/pytest33.log
