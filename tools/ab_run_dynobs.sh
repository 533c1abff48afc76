mkdir -p gpurun_out/r02z
timeout 1200 python -m pytest tests -m gpu -x -q -k "dynobs or Dynamic or canary or vis_table or wide or rollout or random_states or categorical" > gpurun_out/r02z/gputests.log 2>&1; echo gputests_rc=$?
bash tools/ab_sweep.sh gpurun_out/r02z Dynamic-Obstacles-8x8-v0 65536,262144,1048576 r2h5
