set -x
timeout 900 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build $?
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "cholesky or 3x3 or config0" > gpurun_out/pytest_chol.log 2>&1; echo pytest $?
for m in 10000 7202; do timeout 300 python tools/dag_trace.py $m > gpurun_out/trace_$m.log 2>&1; echo trace $m $?; done
for m in 10000 7202; do SDPC_LIB=paper_1310_6919_b200/libsdpc_bk32.so timeout 300 python tools/dag_trace.py $m > gpurun_out/trace_bk32_$m.log 2>&1; echo trace $m $?; done
