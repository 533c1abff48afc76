mkdir -p gpurun_out/r02q
timeout 1200 python -m pytest tests -m gpu -x -q -k "DoorKey or doorkey or canary or random_states or wide or rollout or bench or smoke or cfg" > gpurun_out/r02q/gputests.log 2>&1; echo gputests_rc=$?
bash tools/ab_sweep.sh gpurun_out/r02q DoorKey-8x8-v0,DoorKey-6x6-v0 2048,65536,262144,1048576,4194304 r2h2
for tag in new r2h2; do
  if [ $tag = new ]; then LIB=""; else LIB=build/ab/libnavix_$tag.so; fi
  NAVIX_LIBRARY=$LIB timeout 600 python tools/sweep.py --envs DoorKey-8x8-v0 --sizes 262144,1048576 --steps 540 --runs 3 --desync --out gpurun_out/r02q/desync_$tag.json > gpurun_out/r02q/desync_$tag.txt 2>&1
done
