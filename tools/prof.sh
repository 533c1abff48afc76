#!/bin/bash
# profiling helper run ON the GPU box: bench + launch list + one full ncu capture of the step kernel
# usage: bash tools_prof.sh <tag> [env] [envs_per_gpu]
TAG=$1; ENV=${2:-DoorKey-8x8-v0}; NE=${3:-1048576}
mkdir -p gpurun_out
ARGS="--env $ENV --envs-per-gpu $NE --steps 20 --warmup 3 --no-cpu-baseline --no-graph --rollout-steps 0 --categorical-steps 0 --e2e-steps 2"
timeout 300 python bench.py $ARGS > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py $ARGS > /dev/null 2>&1; echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-navix_step_persistent} -s 5 -c 1 -o gpurun_out/prof_$TAG python bench.py $ARGS > gpurun_out/ncu_full_$TAG.log 2>&1; echo "ncu full rc=$?"
