# One GPU session: smoke, GPU tests, bench lines.  Every step under its own timeout.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build $?
timeout 240 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1 || { echo smoke failed; exit 3; }
timeout 400 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo bench $?
timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo pytest $?
for c in 2 3; do timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-measure-peak > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; echo bench$c $?; done
