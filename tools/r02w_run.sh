mkdir -p gpurun_out/r02w
timeout 900 python -m pytest tests -m gpu -x -q -k "Crossing or crossing or lava or vis_table or canary" > gpurun_out/r02w/gputests.log 2>&1; echo gputests_rc=$?
bash tools/ab_sweep.sh gpurun_out/r02w Crossings-S9N3-v0,Crossings-S11N5-v0,SimpleCrossingS9N3-v0 2048,262144,1048576 r2h4
