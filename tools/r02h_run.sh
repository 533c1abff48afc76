mkdir -p gpurun_out/r02h
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02h/gputests.log 2>&1; echo gputests_rc=$?
bash tools/ab_sweep.sh gpurun_out/r02h Dynamic-Obstacles-8x8-v0 65536,1048576 unified
timeout 600 python tools/sweep.py --envs DoorKey-8x8-v0,Dynamic-Obstacles-8x8-v0,KeyCorridorS3R3-v0,LavaGapS7-v0 --sizes 65536,262144,1048576 --steps 512 --runs 3 --desync --out gpurun_out/r02h/sweep_desync.json > gpurun_out/r02h/sweep_desync.txt 2>&1
timeout 600 python tools/sweep.py --envs DoorKey-8x8-v0,Dynamic-Obstacles-8x8-v0,KeyCorridorS3R3-v0,LavaGapS7-v0 --sizes 65536,262144,1048576 --steps 512 --runs 3 --out gpurun_out/r02h/sweep_sync.json > gpurun_out/r02h/sweep_sync.txt 2>&1
ARGS="--env DoorKey-8x8-v0 --envs-per-gpu 1048576 --steps 20 --warmup 3 --no-cpu-baseline --no-graph --rollout-steps 0 --categorical-steps 0 --e2e-steps 2 --steady-steps 0"
timeout 300 python bench.py $ARGS > gpurun_out/r02h/plain_traffic.log 2>&1 && timeout 600 ncu --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:navix_step_persistent -s 6 -c 8 --csv --log-file gpurun_out/r02h/traffic_steady_dk8.csv python bench.py $ARGS > /dev/null 2>&1; echo ncu_rc=$?
ARGS2="--env Dynamic-Obstacles-8x8-v0 --envs-per-gpu 1048576 --steps 20 --warmup 3 --no-cpu-baseline --no-graph --rollout-steps 0 --categorical-steps 0 --e2e-steps 2 --steady-steps 0"
timeout 300 python bench.py $ARGS2 > gpurun_out/r02h/plain_traffic2.log 2>&1 && timeout 600 ncu --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:navix_step_persistent -s 6 -c 8 --csv --log-file gpurun_out/r02h/traffic_steady_do8.csv python bench.py $ARGS2 > /dev/null 2>&1; echo ncu2_rc=$?
