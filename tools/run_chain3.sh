# Fused diagonal update: trace, GPU tests, bench c1/c2.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 120 python tools/dag_trace.py 2000 > gpurun_out/dag_trace_small.log 2>&1; echo trace_small $?
timeout 300 python tools/dag_trace.py > gpurun_out/dag_trace_fused.log 2>&1; echo trace $?
timeout 400 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo bench $?
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest $?
timeout 300 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline --no-measure-peak > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench2 $?
