./tools/mb_lat > gpurun_out/mb_lat.log 2>&1
bash tools/gpu_dag.sh
