# SCE solve check: build, SCE parity tests, c1 and c4 bench lines (next_rows.sce_solve_ms).
set -x
timeout 900 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build $?
timeout 300 python -m pytest tests -m gpu -q -x -k "sce or scm_solve" > gpurun_out/pytest_sce.log 2>&1; echo t $?
timeout 400 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo b $?
timeout 300 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-measure-peak > gpurun_out/bench_c3.json 2>gpurun_out/bench_c3.err; echo b3 $?
