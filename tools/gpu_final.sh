# Final evidence for the round: default bench line (driver command), launch list, full capture of
# the dominant kernel, all configs' bench lines.
set -x
timeout 900 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build $?
timeout 240 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1 || { echo smoke failed; exit 3; }
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/final_pytest_gpu.log 2>&1; echo pytest $?
timeout 600 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo bench $?
timeout 600 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err; echo ref $?
for c in 0 2 3 4; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-measure-peak > gpurun_out/final_c$c.json 2> gpurun_out/final_c$c.err; echo c$c $?; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches_c1.csv \
   python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-measure-peak > gpurun_out/ncu_l.log 2>&1; echo ncu1 $?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k 'regex:gemm_nt_kernel<.int.2' --launch-skip 60 --launch-count 1 -o gpurun_out/final_upd -f \
   python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-measure-peak > gpurun_out/ncu_u.log 2>&1; echo ncu2 $?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k 'regex:inverse_panel' --launch-skip 2 --launch-count 1 -o gpurun_out/final_solve -f \
   python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-measure-peak > gpurun_out/ncu_s.log 2>&1; echo ncu3 $?
