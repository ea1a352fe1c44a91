set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_direction.py -x -q > gpurun_out/pytest_solve.log 2>&1; echo pytest $?
for c in 1 3 5; do timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-measure-peak > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; echo bench$c $?; done
