"""Host-side bandwidth on the GPU box (dev tool): pinned-buffer fill and copy GB/s by thread
count, and the plain 4 GiB D2H copy; decided against expanding ASK fill lists on the host
for the end-to-end path."""
import time, torch, os
print("cpus", len(os.sched_getaffinity(0)))
n = 32768
h = torch.empty(n * n, dtype=torch.int32).pin_memory()
for th in (1, 4, 8, 16, 32):
    torch.set_num_threads(th)
    h.fill_(1)
    t0 = time.perf_counter(); h.fill_(7); dt = time.perf_counter() - t0
    print("threads", th, "fill GB/s %.1f" % (4 * n * n / dt / 1e9))
src = torch.empty(n * n // 8, dtype=torch.int32).pin_memory(); src.fill_(3)
torch.set_num_threads(16)
t0 = time.perf_counter()
for k in range(8):
    h[k * (n * n // 8):(k + 1) * (n * n // 8)].copy_(src)
dt = time.perf_counter() - t0
print("copy GB/s %.1f" % (4 * n * n / dt / 1e9))
d = torch.empty(n * n, dtype=torch.int32, device="cuda")
torch.cuda.synchronize()
t0 = time.perf_counter(); h.copy_(d); torch.cuda.synchronize(); dt = time.perf_counter() - t0
print("D2H GB/s %.1f" % (4 * n * n / dt / 1e9))
