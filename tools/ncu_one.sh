#!/bin/bash
# ncu --set full of one launch of kernel regex $2 in `bench.py $3...` (plain run first, then ncu);
# exports details / raw / source CSV pages and keeps the report only under /tmp on the box.
# usage: tools/ncu_one.sh TAG KREGEX bench-args...
TAG=$1; KRE=$2; shift 2
mkdir -p gpurun_out
python bench.py "$@" > gpurun_out/ncu_plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"$KRE" -c 1 -o /tmp/prof_$TAG python bench.py "$@" > gpurun_out/ncu_$TAG.log 2>&1
echo rc=$? >> gpurun_out/ncu_$TAG.log
if [ -f /tmp/prof_$TAG.ncu-rep ]; then
  ncu -i /tmp/prof_$TAG.ncu-rep --page details > gpurun_out/details_$TAG.txt 2>&1
  ncu -i /tmp/prof_$TAG.ncu-rep --page raw --csv > gpurun_out/raw_$TAG.csv 2>&1
  ncu -i /tmp/prof_$TAG.ncu-rep --page source --csv > gpurun_out/source_$TAG.csv 2>&1
fi
