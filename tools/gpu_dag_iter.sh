set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "cholesky or potrf or sce or smoke" > gpurun_out/pytest_chol.log 2>&1; echo pytest $?
timeout 300 python tools/dag_trace.py 10000 > gpurun_out/dag_trace.log 2>&1; echo trace $?
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-measure-peak > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo bench $?
