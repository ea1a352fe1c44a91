set -x
timeout 600 python tools/chol_accuracy.py 1 > gpurun_out/acc.log 2>&1; echo acc $?
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-measure-peak > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo bench $?
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "cholesky or potrf or dist or smoke" > gpurun_out/pytest_chol.log 2>&1; echo pytest $?
timeout 600 python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/pytest_dist.log 2>&1; echo pytestdist $?
