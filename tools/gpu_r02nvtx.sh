# Final sanity with the NVTX build: GPU tests, smoke, C3 bench; an ncu NVTX-range filter check.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r02h.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu_r02h.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"; echo smoke=$?
timeout 900 python bench.py > gpurun_out/bench_C3_r02h.json 2> gpurun_out/bench_C3_r02h.err; echo "bench rc=$?"
timeout 600 ncu --nvtx --nvtx-include "mandel_ask_tiles/" -k regex:k_init -c 1 --metrics gpu__time_duration.sum \
  python -c "import paper_2206_02255_b200 as m, workloads as W; w=W.C1; m.ask(w.region,w.n,w.maxdwell,w.g,w.r,w.B); import torch; torch.cuda.synchronize()" > gpurun_out/ncu_nvtx.log 2>&1
grep -E "k_init|No kernels|NVTX" gpurun_out/ncu_nvtx.log | head -5
