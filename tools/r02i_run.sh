mkdir -p gpurun_out/r02i
timeout 900 python -m pytest tests -m gpu -x -q -k "wide or parity_cfg1 or parity_cfg2 or tiny or canary" > gpurun_out/r02i/gputests.log 2>&1; echo gputests_rc=$?
for W in 0 1000000; do
  NAVIX_WIDE_MAX=$W timeout 600 python tools/sweep.py --envs Empty-5x5-v0,Empty-8x8-v0,DoorKey-8x8-v0,Dynamic-Obstacles-8x8-v0,KeyCorridorS3R3-v0,LavaGapS7-v0 --sizes 1,8,1024,2048,16384,65536 --steps 512 --runs 3 --out gpurun_out/r02i/sweep_wide$W.json > gpurun_out/r02i/sweep_wide$W.txt 2>&1
done
