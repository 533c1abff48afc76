mkdir -p gpurun_out/r02o
timeout 1200 python -m pytest tests -m gpu -x -q -k "dynobs or Dynamic or rollout or canary or random_states or wide or direct" > gpurun_out/r02o/gputests.log 2>&1; echo gputests_rc=$?
bash tools/ab_sweep.sh gpurun_out/r02o Dynamic-Obstacles-8x8-v0,Dynamic-Obstacles-6x6 65536,262144,1048576 r2h2
NAVIX_LIBRARY= timeout 600 python tools/sweep.py --rollout-k 64 --runs 3 --envs Dynamic-Obstacles-8x8-v0 --sizes 65536,262144 --out gpurun_out/r02o/rollout_new.json > gpurun_out/r02o/rollout_new.txt 2>&1
NAVIX_LIBRARY=build/ab/libnavix_r2h2.so timeout 600 python tools/sweep.py --rollout-k 64 --runs 3 --envs Dynamic-Obstacles-8x8-v0 --sizes 65536,262144 --out gpurun_out/r02o/rollout_old.json > gpurun_out/r02o/rollout_old.txt 2>&1
