mkdir -p gpurun_out/r02t
timeout 1200 python -m pytest tests -m gpu -x -q -k "vis_table or LavaGap or Crossing or lava or canary or random_states or wide or rollout" > gpurun_out/r02t/gputests.log 2>&1; echo gputests_rc=$?
bash tools/ab_sweep.sh gpurun_out/r02t LavaGapS7-v0,SimpleCrossingS11N5-v0,SimpleCrossingS9N3-v0 2048,262144,1048576 dkvis
