#!/bin/bash
# Quick check + profile of the config 5 kernels on a T prefix (bounded ncu replays).
# usage: tools/r02_prof.sh TAG "kernel regexes" [pytest -k expr]
TAG=$1; KS=$2; K=$3
O=gpurun_out; mkdir -p $O
if [ -n "$K" ]; then
  timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -k "$K" > $O/t_$TAG.log 2>&1; echo rc=$? >> $O/t_$TAG.log
fi
B="--steps 5 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 python bench.py --config 5 $B > $O/b5_$TAG.log 2>&1; echo rc=$? >> $O/b5_$TAG.log
timeout 300 python bench.py --config 3 $B > $O/b3_$TAG.log 2>&1; echo rc=$? >> $O/b3_$TAG.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" --csv \
    --log-file $O/launches5_$TAG.csv python bench.py --config 5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e \
    > $O/ncu_launch5_$TAG.log 2>&1
for k in $KS; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_$k" -c 1 -o /tmp/p5_${TAG}_$k \
      python bench.py --config 5 --t 96 --profile --steps 1 --warmup 3 > $O/ncu5_${TAG}_$k.log 2>&1
  ncu -i /tmp/p5_${TAG}_$k.ncu-rep --page raw --csv > $O/raw5_${TAG}_$k.csv
  ncu -i /tmp/p5_${TAG}_$k.ncu-rep --page details > $O/details5_${TAG}_$k.txt
  ncu -i /tmp/p5_${TAG}_$k.ncu-rep --page source --csv > $O/source5_${TAG}_$k.csv
done
