# Exercise bench.py's N > 1 path on a one-GPU box: 2 and 4 ranks sharing cuda:0 over a gloo
# process group (MANDEL_DIST_BACKEND=gloo).  Times are not scaling numbers (ranks share the GPU).
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for N in 2 4; do
  MANDEL_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port $((29500+N)) bench.py --gpus $N --steps 5 --warmup 3 --workload C1 \
    > gpurun_out/multirank_C1_$N.json 2> gpurun_out/multirank_C1_$N.err; echo rc=$?; cat gpurun_out/multirank_C1_$N.json | cut -c1-1500; tail -3 gpurun_out/multirank_C1_$N.err
done
MANDEL_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29510 bench.py --gpus 2 --steps 5 --warmup 3 \
  > gpurun_out/multirank_C3_2.json 2> gpurun_out/multirank_C3_2.err; echo rc=$?; cat gpurun_out/multirank_C3_2.json | cut -c1-2500; tail -3 gpurun_out/multirank_C3_2.err
