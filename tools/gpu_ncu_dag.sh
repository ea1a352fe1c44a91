set -x
timeout 900 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build $?
timeout 120 python tools/chol_once.py 10000 1 2 > gpurun_out/once.log 2>&1; echo once $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:chol_dag_kernel --launch-skip 1 --launch-count 1 -o gpurun_out/dag_full -f python tools/chol_once.py 10000 1 2 > gpurun_out/ncu_dag.log 2>&1; echo ncu $?
