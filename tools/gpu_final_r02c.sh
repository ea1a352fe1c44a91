# Round-2 closing evidence on the HEAD build: smoke, default bench line (driver command), GPU tests, reference
# arm, c1 launch list, full captures of the dominant kernel, the accumulate and the solve kernel, other configs.
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/h_smoke.log 2>&1 || { echo smoke failed; tail -20 gpurun_out/h_smoke.log; exit 3; }
timeout 600 python bench.py > gpurun_out/h_bench.json 2> gpurun_out/h_bench.err; echo bench $?
timeout 1500 python -m pytest tests -m gpu -q -x --durations=8 > gpurun_out/h_pytest_gpu.log 2>&1; echo pytest $?
timeout 900 python bench.py --impl reference > gpurun_out/h_ref.json 2> gpurun_out/h_ref.err; echo ref $?
for c in 2 3 5; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/h_bench_c$c.json 2> gpurun_out/h_bench_c$c.err; echo benchc$c $?; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/h_launches_c1.csv \
   python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-measure-peak > gpurun_out/h_ncu_l.log 2>&1; echo ncu1 $?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k 'regex:chol_dag_kernel' --launch-skip 3 --launch-count 1 -o gpurun_out/h_dag -f \
   python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-measure-peak > gpurun_out/h_ncu_d.log 2>&1; echo ncu2 $?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k 'regex:scm_maxcut' --launch-skip 3 --launch-count 1 -o gpurun_out/h_scm -f \
   python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-measure-peak > gpurun_out/h_ncu_c.log 2>&1; echo ncu3 $?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k 'regex:inverse_panel' --launch-skip 6 --launch-count 1 -o gpurun_out/h_solve -f \
   python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-measure-peak > gpurun_out/h_ncu_s.log 2>&1; echo ncu4 $?
