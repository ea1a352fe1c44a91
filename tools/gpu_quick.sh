# Quick GPU cycle: microbench, yardstick, smoke, GPU tests, bench, launch list.
set -x
./tools/mb_warpchol > gpurun_out/mb.log 2>&1; echo mb $?
timeout 120 python tools/time_tiles.py > gpurun_out/tiles.log 2>&1; echo tiles $?
timeout 120 python tools/yardstick_potrf.py 10000 > gpurun_out/yardstick.log 2>&1; echo yard $?
timeout 900 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build $?
timeout 240 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1 || { echo smoke failed; exit 3; }
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/pytest_gpu.log 2>&1; echo pytest $?
timeout 400 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo bench $?
for c in 2 3; do timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-measure-peak > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; echo bench$c $?; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv \
   python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-measure-peak > gpurun_out/ncu_launch.log 2>&1; echo ncu1 $?
if [ -n "$NCU_KERNELS" ]; then
  i=0
  for k in $NCU_KERNELS; do
    i=$((i+1))
    timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k "regex:$k" --launch-skip 5 --launch-count 1 -o gpurun_out/prof_$i -f \
      python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-measure-peak > gpurun_out/ncu_$i.log 2>&1; echo ncu_k$i $?
  done
fi
