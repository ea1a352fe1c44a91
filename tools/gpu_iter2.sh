set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python bench.py --no-cpu-baseline --no-measure-peak > gpurun_out/j_bench_c1.json 2> gpurun_out/j_bench_c1.err; echo bench $?
SDPC_LIB=$GRAFT_REPO_ROOT/variants/libsdpc_pipe.so timeout 300 python bench.py --no-cpu-baseline --no-measure-peak > gpurun_out/j_bench_c1_pipe.json 2> gpurun_out/j_bench_c1_pipe.err; echo benchpipe $?
timeout 300 python bench.py --config 2 --no-cpu-baseline --no-measure-peak > gpurun_out/j_bench_c2.json 2> gpurun_out/j_bench_c2.err; echo bench2 $?
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "config2 or small or theta or reproducible or fused" > gpurun_out/j_pytest.log 2>&1; echo pytest $?; tail -3 gpurun_out/j_pytest.log
SDPC_LIB=$GRAFT_REPO_ROOT/variants/libsdpc_pipe.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "cholesky" > gpurun_out/j_pytest_pipe.log 2>&1; echo pytestpipe $?; tail -3 gpurun_out/j_pytest_pipe.log
