set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python -m pytest tests -m gpu -x -q -k "groups" 2>&1 | tail -2
for G in 1 2 3 4; do timeout 600 python tools/emulate_scaling.py C3 --ranks 1,8 --deals costrank --groups $G > gpurun_out/emu32_g$G.jsonl 2>&1; tail -3 gpurun_out/emu32_g$G.jsonl | cut -c1-600; done
