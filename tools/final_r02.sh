#!/bin/bash
# Round-2 evidence run on the GPU box (one GPU): the GPU suite, the bench line
# (both arms), sweeps (synchronised and steady state), the ncu launch list and
# one ncu --set full capture of the headline step kernel.
OUT=${1:-gpurun_out/final}
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q > $OUT/gputests.log 2>&1; echo gputests_rc=$?
timeout 600 python bench.py > $OUT/bench_line.json 2> $OUT/bench.err; echo bench_rc=$?
timeout 600 python bench.py --impl reference > $OUT/bench_reference_line.json 2> $OUT/bench_ref.err; echo ref_rc=$?
timeout 900 python tools/sweep.py --steps 512 --runs 5 --out $OUT/sweep.json > $OUT/sweep.txt 2>&1; echo sweep_rc=$?
timeout 900 python tools/sweep.py --steps 540 --runs 3 --desync --envs DoorKey-8x8-v0,Dynamic-Obstacles-8x8-v0,KeyCorridorS3R3-v0,LavaGapS7-v0,Empty-5x5-v0,Empty-8x8-v0 --sizes 2048,65536,262144,1048576 --out $OUT/sweep_steady.json > $OUT/sweep_steady.txt 2>&1; echo steady_rc=$?
timeout 900 python tools/sweep.py --rollout-k 256 --runs 3 --envs DoorKey-8x8-v0,Dynamic-Obstacles-8x8-v0,KeyCorridorS3R3-v0,LavaGapS7-v0,Empty-5x5-v0,Empty-8x8-v0 --sizes 16,2048,65536,262144,1048576 --out $OUT/sweep_rollout.json > $OUT/sweep_rollout.txt 2>&1; echo rollout_rc=$?
timeout 1500 python tools/sweep.py --catalog --steps 256 --runs 3 --out $OUT/sweep_catalog.json > $OUT/sweep_catalog.txt 2>&1; echo catalog_rc=$?
ARGS="--steps 20 --warmup 3 --no-cpu-baseline --no-graph --rollout-steps 8 --categorical-steps 8 --e2e-steps 2 --steady-steps 0"
timeout 300 python bench.py $ARGS > $OUT/plain_launches.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python bench.py $ARGS > /dev/null 2>&1; echo launches_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:navix_step_persistent -s 8 -c 1 -o $OUT/prof_dk8 python bench.py $ARGS > $OUT/ncu_full.log 2>&1; echo ncu_full_rc=$?
