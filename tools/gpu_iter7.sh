set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for i in 1 2; do
timeout 300 python bench.py --no-cpu-baseline --no-measure-peak > gpurun_out/p_bench_c1_$i.json 2> gpurun_out/p_bench.err; echo bench $?
done
for c in 3 5 4; do timeout 600 python bench.py --config $c --no-cpu-baseline --no-measure-peak > gpurun_out/p_bench_c$c.json 2> gpurun_out/p_bench_c$c.err; echo benchc$c $?; done
SDPC_LIB=$GRAFT_REPO_ROOT/variants/libsdpc_rev2.so timeout 600 python bench.py --config 4 --no-cpu-baseline --no-measure-peak > gpurun_out/p_bench_c4_rev2.json 2> gpurun_out/p_bench_c4_rev2.err; echo benchc4rev2 $?
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/p_pytest.log 2>&1; echo pytest $?; tail -n 3 gpurun_out/p_pytest.log
