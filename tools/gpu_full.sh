# Full GPU check: build, smoke, all GPU tests, default bench (c1) and c2/c3 lines.
set -x
timeout 900 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build $?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke $?
timeout 1800 python -m pytest tests -m gpu -q -x --durations=8 > gpurun_out/pytest_gpu.log 2>&1; echo pytest $?
timeout 400 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo bench $?
for c in 2 3; do timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-measure-peak > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; echo bench$c $?; done
