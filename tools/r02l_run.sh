mkdir -p gpurun_out/r02l
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02l/gputests.log 2>&1; echo gputests_rc=$?
bash tools/ab_sweep.sh gpurun_out/r02l GoToDoor-8x8-v0,DoorKey-8x8-v0,Dynamic-Obstacles-8x8-v0 65536,262144,1048576 kcsched
