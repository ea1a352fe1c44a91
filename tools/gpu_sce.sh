set -x
timeout 900 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build $?
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_direction.py -q -x -k "sce or direction_matches or configs or after_direction" > gpurun_out/pytest_sce.log 2>&1; echo pytest $?
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-measure-peak > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo bench $?
