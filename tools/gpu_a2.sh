set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest $?
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-measure-peak > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo bench $?
timeout 300 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline --no-measure-peak > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo bench5 $?
