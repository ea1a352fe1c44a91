set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python bench.py --config 3 --no-cpu-baseline --no-measure-peak > gpurun_out/s_bench_c3.json 2> gpurun_out/s_bench_c3.err; echo benchc3 $?
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -m gpu -q -x -k "blockarrow or small or dist or theta or config0 or fused" > gpurun_out/s_pytest.log 2>&1; echo pytest $?; tail -n 3 gpurun_out/s_pytest.log
