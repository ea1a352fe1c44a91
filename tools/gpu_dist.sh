# Multi-rank schedule on one GPU (gloo, host-side exchanges only; no kernel waits on another rank)
set -x
timeout 900 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build $?
for c in 0 2; do
SDPC_BENCH_BACKEND=gloo SDPC_BENCH_DEVICE=0 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 2 --warmup 3 --config $c > gpurun_out/dist2_c$c.json 2> gpurun_out/dist2_c$c.err; echo dist2_c$c $?
done
SDPC_BENCH_BACKEND=gloo SDPC_BENCH_DEVICE=0 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 \
  --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 --steps 2 --warmup 3 --config 1 > gpurun_out/dist4_c1.json 2> gpurun_out/dist4_c1.err; echo dist4 $?
