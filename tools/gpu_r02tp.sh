# Tail pool A/B: parity subset on the default build, then gpu_ab3 (C3/C5 + 8-way C3 rank) for
# RF_TAILPOOL=0 vs 1, and the C4 8-way rank.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "ask_c1 or random_small or edge or maxdwell or one_graph or tiles or c3_full" 2>&1 | tail -2
PA="RF_TAILPOOL=0" PB="RF_TAILPOOL=1" bash tools/gpu_ab3.sh 2>&1
