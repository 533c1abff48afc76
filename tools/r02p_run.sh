mkdir -p gpurun_out/r02p
timeout 1200 python -m pytest tests -m gpu -x -q -k "Empty or DistShift or Dynamic or dynobs or canary or random_states or wide" > gpurun_out/r02p/gputests.log 2>&1; echo gputests_rc=$?
bash tools/ab_sweep.sh gpurun_out/r02p Empty-5x5-v0,Empty-8x8-v0,Empty-Random-8x8,DistShift1-v0,Empty-16x16-v0 2048,65536,1048576 vt r2h2
