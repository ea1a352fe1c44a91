# POTRF / chain experiments: warp-Cholesky microbenchmarks (both variants), the task-graph trace of the
# product build, the Cholesky parity tests.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in 0 1; do ./tools/mb_wchol_dag_v$v; ./tools/mb_potrf_v$v; done > gpurun_out/mb_chain.log 2>&1; echo mb $?
timeout 300 python tools/dag_trace.py > gpurun_out/dag_trace.log 2>&1; echo trace $?
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "cholesky or smoke or config" > gpurun_out/pytest_chol.log 2>&1; echo pytest $?
timeout 400 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo bench $?
