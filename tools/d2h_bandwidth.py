import torch, time
n = 4 << 30
d = torch.empty(n, dtype=torch.uint8, device='cuda'); d.fill_(1)
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
torch.cuda.synchronize()
def run(parts, nstreams):
    streams = [torch.cuda.Stream() for _ in range(nstreams)]
    chunk = n // parts
    torch.cuda.synchronize()
    t = time.perf_counter()
    for i in range(parts):
        s = streams[i % nstreams]
        with torch.cuda.stream(s):
            h[i*chunk:(i+1)*chunk].copy_(d[i*chunk:(i+1)*chunk], non_blocking=True)
    torch.cuda.synchronize()
    return n / (time.perf_counter() - t) / 1e9
for parts, ns in [(1,1),(4,1),(4,2),(4,4),(16,4),(64,8)]:
    bw = [run(parts, ns) for _ in range(3)]
    print(parts, ns, ["%.1f" % b for b in bw])
# H2D for reference
t=time.perf_counter(); d.copy_(h, non_blocking=True); torch.cuda.synchronize(); print("h2d", n/(time.perf_counter()-t)/1e9)
