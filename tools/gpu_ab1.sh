mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "ask_c1 or random_small or edge or maxdwell or one_graph" 2>&1 | tail -3
timeout 2400 python tools/ab_variants.py run base nodir spre8 spre16 bk16 bt4 bt16 bpack bpack8 lpre8 lpre24 --rounds 3 --reps 5 --check > gpurun_out/ab1.jsonl 2>&1
tail -8 gpurun_out/ab1.jsonl
