mkdir -p gpurun_out/r02j
timeout 900 python -m pytest tests -m gpu -x -q -k "KeyCorridor or keycorridor or kc or wide" > gpurun_out/r02j/gputests.log 2>&1; echo gputests_rc=$?
for tag in new unified; do
  if [ $tag = new ]; then LIB=""; else LIB=build/ab/libnavix_$tag.so; fi
  NAVIX_LIBRARY=$LIB timeout 600 python tools/sweep.py --envs KeyCorridorS3R3-v0 --sizes 65536,262144,1048576 --steps 540 --runs 3 --desync --out gpurun_out/r02j/kc_desync_$tag.json > gpurun_out/r02j/kc_desync_$tag.txt 2>&1
  NAVIX_LIBRARY=$LIB timeout 600 python tools/sweep.py --envs KeyCorridorS3R3-v0 --sizes 65536,262144,1048576 --steps 540 --runs 3 --out gpurun_out/r02j/kc_sync_$tag.json > gpurun_out/r02j/kc_sync_$tag.txt 2>&1
done
KREGEX=navix_step_wide SKIP=5 bash tools/prof.sh full wide2048 DoorKey-8x8-v0 2048 > gpurun_out/r02j/prof.log 2>&1; mv gpurun_out/prof_wide2048.ncu-rep gpurun_out/r02j/
NAVIX_WIDE_MAX=0 KREGEX=navix_step_persistent SKIP=5 bash tools/prof.sh full pers2048 DoorKey-8x8-v0 2048 >> gpurun_out/r02j/prof.log 2>&1; mv gpurun_out/prof_pers2048.ncu-rep gpurun_out/r02j/
