# Task-graph Cholesky check: build, Cholesky GPU tests, trace, c1/c2 bench lines.
set -x
timeout 900 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build $?
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "cholesky or 3x3 or config0" > gpurun_out/pytest_chol.log 2>&1; echo pytest $?
timeout 300 python tools/dag_trace.py 10000 > gpurun_out/trace_10000.log 2>&1; echo trace $?
timeout 300 python tools/dag_trace.py 7201 > gpurun_out/trace_7201.log 2>&1; echo trace2 $?
timeout 400 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo bench $?
