set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/u_smoke.log 2>&1; echo smoke $?; tail -n 1 gpurun_out/u_smoke.log
timeout 300 python bench.py --config 3 --no-cpu-baseline --no-measure-peak > gpurun_out/u_bench_c3.json 2> gpurun_out/u_bench_c3.err; echo benchc3 $?
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/u_bench_c1.json 2> gpurun_out/u_bench_c1.err; echo benchc1 $?
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "small or config0 or theta or fused or reproducible" > gpurun_out/u_pytest.log 2>&1; echo pytest $?; tail -n 2 gpurun_out/u_pytest.log
