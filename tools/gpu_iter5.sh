set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/n_pytest.log 2>&1; echo pytest $?; tail -n 3 gpurun_out/n_pytest.log
for i in 1 2; do
timeout 300 python bench.py --no-cpu-baseline --no-measure-peak > gpurun_out/n_bench_c1_$i.json 2> gpurun_out/n_bench.err; echo bench $?
done
for c in 3 5; do timeout 300 python bench.py --config $c --no-cpu-baseline --no-measure-peak > gpurun_out/n_bench_c$c.json 2> gpurun_out/n_bench_c$c.err; echo benchc$c $?; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/n_launches_c1.csv \
   python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-measure-peak > gpurun_out/n_ncu_l.log 2>&1; echo ncu1 $?
