# 16-bit host image: parity tests of the to_host paths, the bench GPU test, C3 bench line.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench.py -q -x -k "to_host or single_gpu" > gpurun_out/pytest_u16.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_u16.log
timeout 900 python bench.py > gpurun_out/bench_u16.json 2> gpurun_out/bench_u16.err; echo "bench rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench_u16.json')); print(d['ms_per_step'], d['e2e'])"
