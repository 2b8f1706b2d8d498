#!/bin/bash
# Profile capture on the GPU box (one GPU): launch list of the bench at the given
# config, then one `ncu --set full` capture per kernel regex, exported as CSV.
# usage: tools/profile_cfg.sh TAG CONFIG "regex1 regex2 ..." [extra bench args]
TAG=$1; CFG=$2; KS=$3; shift 3
mkdir -p gpurun_out
timeout 600 python bench.py --config $CFG --steps 3 --warmup 3 --no-cpu-baseline --no-e2e "$@" > gpurun_out/plain_$TAG.log 2>&1
echo rc=$? >> gpurun_out/plain_$TAG.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu-baseline --no-e2e "$@" \
    > gpurun_out/ncu_launch_$TAG.log 2>&1
for k in $KS; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$k" -c 1 -o /tmp/p_${TAG}_$k \
      python bench.py --config $CFG --profile --steps 1 --warmup 3 "$@" > gpurun_out/ncu_${TAG}_$k.log 2>&1
  ncu -i /tmp/p_${TAG}_$k.ncu-rep --page raw --csv > gpurun_out/raw_${TAG}_$k.csv
  ncu -i /tmp/p_${TAG}_$k.ncu-rep --page details > gpurun_out/details_${TAG}_$k.txt
  ncu -i /tmp/p_${TAG}_$k.ncu-rep --page source --csv > gpurun_out/source_${TAG}_$k.csv
done
