# README usage snippet, checked on the GPU box: PYTHONPATH=. python tools/readme_snippet_check.py
import torch, paper_2206_02255_b200 as mb
region, n, maxdwell, g, r, B = (-1.5, 0.5, -1.0, 1.0), 4096, 2048, 16, 2, 32
ws = mb.workspace(n, g, r, B)
img = mb.ask(region, n, maxdwell, g, r, B, ws=ws)
ex = mb.exhaustive(region, n, maxdwell)
host = torch.empty(n * n, dtype=torch.uint16).pin_memory()
mb.ask_to_host(region, n, maxdwell, g, r, B, host, img, ws)
import numpy as np
assert np.array_equal(host.numpy().reshape(n, n).astype(np.int32), img.cpu().numpy())
print("readme snippet ok", float((img != ex).float().mean()))
