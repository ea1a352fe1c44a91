# Blocked TRSM A/B: trace of the product build and of the previous schedule (variant lib), GPU tests, bench.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/dag_trace.py > gpurun_out/dag_trace_new.log 2>&1; echo trace $?
SDPC_LIB=variants/lib_oldtrsm.so timeout 300 python tools/dag_trace.py > gpurun_out/dag_trace_old.log 2>&1; echo trace_old $?
timeout 400 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo bench $?
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest $?
for c in 2 4; do timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-measure-peak > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; echo bench$c $?; done
