# Measurement session: bench c1 (with cpu_baseline), reference arm c1, ncu captures of the dominant kernels.
set -x
timeout 900 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build $?
nproc > gpurun_out/host.txt; lscpu | grep "Model name" >> gpurun_out/host.txt; free -g >> gpurun_out/host.txt
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c1_full.json 2> gpurun_out/bench_c1_full.err; echo bench $?
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref_c1.json 2> gpurun_out/ref_c1.err; echo ref $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:chol_dag_kernel --launch-skip 3 --launch-count 1 -o gpurun_out/dag_c1 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-measure-peak > gpurun_out/ncu1.log 2>&1; echo ncu1 $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:inverse_panel_kernel --launch-skip 6 --launch-count 2 -o gpurun_out/solve_c1 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-measure-peak > gpurun_out/ncu2.log 2>&1; echo ncu2 $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scm_ --launch-skip 3 --launch-count 1 -o gpurun_out/scm_c1 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-measure-peak > gpurun_out/ncu3.log 2>&1; echo ncu3 $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scm_ --launch-skip 3 --launch-count 2 -o gpurun_out/scm_c2 -f python bench.py --config 2 --steps 1 --warmup 3 --no-cpu-baseline --no-measure-peak > gpurun_out/ncu4.log 2>&1; echo ncu4 $?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-measure-peak > gpurun_out/ncu_launch.log 2>&1; echo ncul $?
