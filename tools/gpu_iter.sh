# quick iteration: parity subset, c1 bench, c2/c3 launch lists
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/i_pytest.log 2>&1; echo pytest $?; tail -3 gpurun_out/i_pytest.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/i_bench_c1.json 2> gpurun_out/i_bench_c1.err; echo bench $?
for c in 2 3; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/i_launches_c$c.csv \
   python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-measure-peak > gpurun_out/i_ncu_l$c.log 2>&1; echo ncu$c $?
done
