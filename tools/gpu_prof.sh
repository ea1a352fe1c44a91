# GPU tests, bench, ncu launch list, and full captures of the diag and solve kernels.
set -x
timeout 900 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build $?
timeout 240 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1 || { echo smoke failed; exit 3; }
timeout 1500 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo pytest $?
timeout 400 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo bench $?
timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-measure-peak > gpurun_out/b1.json 2>gpurun_out/b1.err && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv \
   python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-measure-peak > gpurun_out/ncu_launch.log 2>&1; echo ncu1 $?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k 'regex:potrf_diag' --launch-skip 20 --launch-count 1 -o gpurun_out/diag_full -f \
   python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-measure-peak > gpurun_out/ncu_full2.log 2>&1; echo ncu3 $?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k 'regex:inverse_panel' --launch-skip 1 --launch-count 1 -o gpurun_out/solve_full -f \
   python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-measure-peak > gpurun_out/ncu_full3.log 2>&1; echo ncu4 $?
