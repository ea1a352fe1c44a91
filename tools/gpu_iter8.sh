set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for i in 1 2; do for v in cap160 cap240; do
SDPC_LIB=$GRAFT_REPO_ROOT/variants/libsdpc_$v.so timeout 300 python bench.py --no-cpu-baseline --no-measure-peak > gpurun_out/q_bench_c1_${v}_$i.json 2> gpurun_out/q_bench.err; echo bench $?
done; done
for v in cap160 cap240; do SDPC_LIB=$GRAFT_REPO_ROOT/variants/libsdpc_$v.so timeout 300 python bench.py --config 5 --no-cpu-baseline --no-measure-peak > gpurun_out/q_bench_c5_$v.json 2> gpurun_out/q_bench_c5.err; echo benchc5 $?; done
