# Round-2 final evidence: smoke, GPU tests, default bench line (driver command), reference arm, launch list,
# full captures of the dominant kernel and of the new (a2)/(b) kernels.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 240 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f2_smoke.log 2>&1 || { echo smoke failed; exit 3; }
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/f2_pytest_gpu.log 2>&1; echo pytest $?
timeout 600 python bench.py > gpurun_out/f2_bench.json 2> gpurun_out/f2_bench.err; echo bench $?
timeout 900 python bench.py --impl reference > gpurun_out/f2_ref.json 2> gpurun_out/f2_ref.err; echo ref $?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f2_launches_c1.csv \
   python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-measure-peak > gpurun_out/f2_ncu_l.log 2>&1; echo ncu1 $?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k 'regex:chol_dag_kernel' --launch-skip 3 --launch-count 1 -o gpurun_out/f2_dag -f \
   python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-measure-peak > gpurun_out/f2_ncu_d.log 2>&1; echo ncu2 $?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k 'regex:front_thin_kernel' --launch-skip 100 --launch-count 1 -o gpurun_out/f2_thin -f \
   python tools/iter_once.py 5 > gpurun_out/f2_ncu_t.log 2>&1; echo ncu3 $?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k 'regex:inverse_panel' --launch-skip 2 --launch-count 1 -o gpurun_out/f2_solve -f \
   python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-measure-peak > gpurun_out/f2_ncu_s.log 2>&1; echo ncu4 $?
