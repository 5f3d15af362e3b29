set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build6.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu6.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu6.log
timeout 600 python tools/ab.py C3 C5 --variants b200,serial,sbr,sbr_serial > gpurun_out/ab6.jsonl 2>&1; cat gpurun_out/ab6.jsonl
timeout 1200 python tools/tune_refill.py C3 C5 --points ";RFL_K=16,RFL_T=8;RFL_K=32,RFL_T=8;RFB_T=8;RFB_CH=32;RFL_CH=64;RFL_K=32,RFL_T=2;RFB_K=32,RFB_CH=64" > gpurun_out/tune6.txt 2>&1; cat gpurun_out/tune6.txt
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench6.json 2> gpurun_out/bench6.err; cat gpurun_out/bench6.json; tail -3 gpurun_out/bench6.err
