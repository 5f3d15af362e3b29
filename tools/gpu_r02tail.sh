# Tail re-pass: parity subset + full-image digests, then A/B vs RF_TAIL=0 (C3, C5, C3r8, C4r8).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "ask_c1 or random_small or edge or maxdwell or one_graph or tiles or c3_full or nondyadic" 2>&1 | tail -2
timeout 1500 python tools/ab_variants.py run --workloads C3,C5,C3r8,C4r8 --rounds 3 --reps 5 --check notail base > gpurun_out/ab_tail.jsonl 2>&1; tail -6 gpurun_out/ab_tail.jsonl
