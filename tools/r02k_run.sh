mkdir -p gpurun_out/r02k
timeout 900 python -m pytest tests -m gpu -x -q -k "KeyCorridor or keycorridor or kc" > gpurun_out/r02k/gputests.log 2>&1; echo gputests_rc=$?
for tag in new kcsched; do
  if [ $tag = new ]; then LIB=""; else LIB=build/ab/libnavix_$tag.so; fi
  NAVIX_LIBRARY=$LIB timeout 600 python tools/sweep.py --envs KeyCorridorS3R3-v0 --sizes 65536,262144,1048576 --steps 540 --runs 3 --desync --out gpurun_out/r02k/kc_desync_$tag.json > gpurun_out/r02k/kc_desync_$tag.txt 2>&1
  NAVIX_LIBRARY=$LIB timeout 600 python tools/sweep.py --envs KeyCorridorS3R3-v0 --sizes 65536,262144,1048576 --steps 540 --runs 3 --out gpurun_out/r02k/kc_sync_$tag.json > gpurun_out/r02k/kc_sync_$tag.txt 2>&1
done
for W in 0 100000; do
  NAVIX_WIDE_MAX=$W timeout 600 python tools/sweep.py --envs DoorKey-8x8-v0,Empty-5x5-v0,Dynamic-Obstacles-8x8-v0,KeyCorridorS3R3-v0 --sizes 1,16,128,256,512,1024 --steps 512 --runs 3 --out gpurun_out/r02k/small_wide$W.json > gpurun_out/r02k/small_wide$W.txt 2>&1
done
