set -x
timeout 900 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build $?
timeout 900 python -m pytest tests/test_gpu_dist.py -q -x -k abi --durations=5 > gpurun_out/pytest_distabi.log 2>&1; echo pytest $?
