set -x
timeout 900 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build $?
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "maxcut3d or sampled_columns and 5" --durations=5 > gpurun_out/pytest_3d.log 2>&1; echo pytest $?
timeout 600 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline --no-measure-peak > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo bench5 $?
timeout 900 python bench.py --config 6 --steps 2 --warmup 3 --no-cpu-baseline --no-measure-peak > gpurun_out/bench_c6.json 2> gpurun_out/bench_c6.err; echo bench6 $?
