./tools/mb_potrf > gpurun_out/mb_potrf.log 2>&1
bash tools/gpu_dag3.sh
