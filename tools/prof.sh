#!/bin/bash
# profiling helper run ON the GPU box.  One ncu invocation per call, and only
# after the same bench command has exited 0 without ncu.
# usage: bash tools/prof.sh launches|full <tag> [env] [envs_per_gpu]
#   launches: plain bench + the ncu launch list (gpu__time_duration per launch)
#   full:     plain bench + one `ncu --set full` capture of the step kernel
MODE=$1; TAG=$2; ENV=${3:-DoorKey-8x8-v0}; NE=${4:-1048576}
mkdir -p gpurun_out
ARGS="--env $ENV --envs-per-gpu $NE --steps 20 --warmup 3 --no-cpu-baseline --no-graph --rollout-steps 0 --categorical-steps 0 --e2e-steps 2"
timeout 300 python bench.py $ARGS > gpurun_out/plain_$TAG.log 2>&1 || { echo "plain bench failed"; exit 1; }
if [ "$MODE" = launches ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py $ARGS > /dev/null 2>&1; echo "launch list rc=$?"
else
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-navix_step_persistent} -s ${SKIP:-5} -c 1 \
    -o gpurun_out/prof_$TAG python bench.py $ARGS > gpurun_out/ncu_full_$TAG.log 2>&1; echo "ncu full rc=$?"
fi
