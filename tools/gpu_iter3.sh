set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for i in 1 2; do
timeout 300 python bench.py --no-cpu-baseline --no-measure-peak > gpurun_out/k_bench_c1_$i.json 2> gpurun_out/k_bench_c1.err; echo bench $?
SDPC_LIB=$GRAFT_REPO_ROOT/variants/libsdpc_p512.so timeout 300 python bench.py --no-cpu-baseline --no-measure-peak > gpurun_out/k_bench_c1_p512_$i.json 2> gpurun_out/k_bench_c1_p512.err; echo bench512 $?
done
SDPC_LIB=$GRAFT_REPO_ROOT/variants/libsdpc_p512.so timeout 300 python bench.py --config 5 --no-cpu-baseline --no-measure-peak > gpurun_out/k_bench_c5_p512.json 2> gpurun_out/k_bench_c5_p512.err; echo bench512c5 $?
timeout 300 python bench.py --config 5 --no-cpu-baseline --no-measure-peak > gpurun_out/k_bench_c5.json 2> gpurun_out/k_bench_c5.err; echo benchc5 $?
SDPC_LIB=$GRAFT_REPO_ROOT/variants/libsdpc_p512.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/k_pytest_p512.log 2>&1; echo pytest512 $?; tail -n 3 gpurun_out/k_pytest_p512.log
