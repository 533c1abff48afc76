mkdir -p gpurun_out/r02m
timeout 1200 python -m pytest tests -m gpu -x -q -k "wide or rollout or canary or direct_oracle or categorical" > gpurun_out/r02m/gputests.log 2>&1; echo gputests_rc=$?
for W in 0 100000; do
  NAVIX_WIDE_MAX_ROLLOUT=$W timeout 600 python tools/sweep.py --envs DoorKey-8x8-v0,Empty-5x5-v0,Dynamic-Obstacles-8x8-v0,KeyCorridorS3R3-v0 --sizes 16,128,1024,2048,4096,8192,16384,65536 --rollout-k 256 --runs 3 --out gpurun_out/r02m/rollout_wide$W.json > gpurun_out/r02m/rollout_wide$W.txt 2>&1
done
