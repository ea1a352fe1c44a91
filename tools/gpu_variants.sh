timeout 200 python tools/dag_trace.py 10000 > gpurun_out/dv_base.log 2>&1
for v in ms8 chain3 ms2; do SDPC_LIB=variants/libsdpc_$v.so timeout 200 python tools/dag_trace.py 10000 > gpurun_out/dv_$v.log 2>&1; done
timeout 200 python tools/dag_trace.py 10000 > gpurun_out/dv_base2.log 2>&1
