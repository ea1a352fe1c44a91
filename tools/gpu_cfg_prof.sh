# Launch list and one full capture of a kernel for a given config: CFG=3 KERNEL=inverse_panel
set -x
CFG=${CFG:-3}
KERNEL=${KERNEL:-inverse_panel}
timeout 900 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build $?
timeout 300 python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline --no-measure-peak > gpurun_out/cfg_b1.json 2>gpurun_out/cfg_b1.err; echo b1 $?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c$CFG.csv \
   python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline --no-measure-peak > gpurun_out/ncu_l.log 2>&1; echo ncu1 $?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k "regex:$KERNEL" --launch-skip 2 --launch-count 1 -o gpurun_out/cfgprof -f \
   python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline --no-measure-peak > gpurun_out/ncu_c.log 2>&1; echo ncu2 $?
