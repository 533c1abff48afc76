mkdir -p gpurun_out/r02v
timeout 900 python -m pytest tests -m gpu -x -q -k "wide or cfg1 or tiny or rollout" > gpurun_out/r02v/gputests.log 2>&1; echo gputests_rc=$?
for tag in new r2h3; do
  if [ $tag = new ]; then LIB=""; else LIB=build/ab/libnavix_$tag.so; fi
  NAVIX_LIBRARY=$LIB timeout 600 python tools/sweep.py --envs DoorKey-8x8-v0,Empty-5x5-v0,Dynamic-Obstacles-8x8-v0,LavaGapS7-v0 --sizes 1,16,512 --steps 512 --runs 3 --out gpurun_out/r02v/small_$tag.json > gpurun_out/r02v/small_$tag.txt 2>&1
  NAVIX_LIBRARY=$LIB timeout 600 python tools/sweep.py --rollout-k 256 --envs DoorKey-8x8-v0,Empty-5x5-v0,Dynamic-Obstacles-8x8-v0,LavaGapS7-v0 --sizes 16,2048,4096 --runs 3 --out gpurun_out/r02v/rollout_$tag.json > gpurun_out/r02v/rollout_$tag.txt 2>&1
done
