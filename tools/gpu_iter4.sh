set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for i in 1 2; do for v in l256 l512; do
SDPC_LIB=$GRAFT_REPO_ROOT/variants/libsdpc_$v.so timeout 300 python bench.py --no-cpu-baseline --no-measure-peak > gpurun_out/m_bench_c1_${v}_$i.json 2> gpurun_out/m_bench.err; echo bench $?
done; done
SDPC_LIB=$GRAFT_REPO_ROOT/variants/libsdpc_l512.so timeout 300 python bench.py --config 5 --no-cpu-baseline --no-measure-peak > gpurun_out/m_bench_c5_l512.json 2> gpurun_out/m_bench_c5.err; echo benchc5 $?
SDPC_LIB=$GRAFT_REPO_ROOT/variants/libsdpc_l512.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/m_launches_c1_l512.csv \
   python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-measure-peak > gpurun_out/m_ncu_l.log 2>&1; echo ncu1 $?
SDPC_LIB=$GRAFT_REPO_ROOT/variants/libsdpc_l512.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/m_pytest_l512.log 2>&1; echo pytest512 $?; tail -n 3 gpurun_out/m_pytest_l512.log
