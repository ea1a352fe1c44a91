set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r_smoke.log 2>&1; echo smoke $?; tail -n 1 gpurun_out/r_smoke.log
timeout 1500 python -m pytest tests -m gpu -q -x --durations=6 > gpurun_out/r_pytest.log 2>&1; echo pytest $?; tail -n 3 gpurun_out/r_pytest.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/r_bench_c1.json 2> gpurun_out/r_bench.err; echo bench $?
