mkdir -p gpurun_out/r02n
timeout 900 python -m pytest tests -m gpu -x -q -k "KeyCorridor or keycorridor or kc or random_states or canary" > gpurun_out/r02n/gputests.log 2>&1; echo gputests_rc=$?
for tag in new r2head; do
  if [ $tag = new ]; then LIB=""; else LIB=build/ab/libnavix_$tag.so; fi
  NAVIX_LIBRARY=$LIB timeout 600 python tools/sweep.py --envs KeyCorridorS3R3-v0,KeyCorridorS6R3-v0 --sizes 65536,262144,1048576 --steps 540 --runs 3 --desync --out gpurun_out/r02n/kc_desync_$tag.json > gpurun_out/r02n/kc_desync_$tag.txt 2>&1
done
timeout 300 python tools/steady_steps.py KeyCorridorS3R3-v0 65536 20 > gpurun_out/r02n/plain_kc.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:navix_step_persistent -s 10 -c 1 -o gpurun_out/r02n/prof_kc65k python tools/steady_steps.py KeyCorridorS3R3-v0 65536 20 > gpurun_out/r02n/ncu.log 2>&1; echo ncu_rc=$?
