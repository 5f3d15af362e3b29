set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build11.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu11.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu11.log
timeout 600 python tools/ab.py C3 C5 --variants g1,g2,g4,g8 > gpurun_out/ab11.jsonl 2>&1; cat gpurun_out/ab11.jsonl | cut -c1-400
for G in 1 2 4; do timeout 900 python tools/emulate_scaling.py C3 --deals costrank --groups $G > gpurun_out/emul11_g$G.jsonl 2>&1; head -4 gpurun_out/emul11_g$G.jsonl | cut -c1-200; done
