set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python bench.py --config 3 --no-cpu-baseline --no-measure-peak > gpurun_out/t_bench_c3.json 2> gpurun_out/t_bench_c3.err; echo benchc3 $?
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/t_pytest.log 2>&1; echo pytest $?; tail -n 3 gpurun_out/t_pytest.log
