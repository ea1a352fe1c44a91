set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for c in 6 4 0; do timeout 500 python bench.py --config $c --no-cpu-baseline --no-measure-peak > gpurun_out/v_bench_c$c.json 2> gpurun_out/v_bench_c$c.err; echo benchc$c $?; done
