set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for i in 1 2; do for v in s3 s3c288; do
SDPC_LIB=$GRAFT_REPO_ROOT/variants/libsdpc_$v.so timeout 300 python bench.py --no-cpu-baseline --no-measure-peak > gpurun_out/o_bench_c1_${v}_$i.json 2> gpurun_out/o_bench.err; echo bench $?
done; done
for c in 2 3 5; do SDPC_LIB=$GRAFT_REPO_ROOT/variants/libsdpc_s3.so timeout 300 python bench.py --config $c --no-cpu-baseline --no-measure-peak > gpurun_out/o_bench_c${c}_s3.json 2> gpurun_out/o_bench_c$c.err; echo benchc$c $?; done
SDPC_LIB=$GRAFT_REPO_ROOT/variants/libsdpc_s3.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_direction.py -m gpu -q -x > gpurun_out/o_pytest_s3.log 2>&1; echo pytests3 $?; tail -n 3 gpurun_out/o_pytest_s3.log
