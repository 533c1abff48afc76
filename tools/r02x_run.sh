mkdir -p gpurun_out/r02x
timeout 900 python -m pytest tests -m gpu -x -q -k "GoToDoor or gotodoor or variants or random_states or canary or Dynamic or dynobs" > gpurun_out/r02x/gputests.log 2>&1; echo gputests_rc=$?
bash tools/ab_sweep.sh gpurun_out/r02x GoToDoor-8x8-v0,Dynamic-Obstacles-Random-6x6 2048,65536,262144,1048576 r2h4
