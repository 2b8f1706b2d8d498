#!/bin/bash
# GPU iteration for one kernel: parity subset, bench, ncu (source + raw) of kernel regex $2
TAG=$1; KRE=$2; K=${3:-"stream or config or quantize or stats or fill or fit"}
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/t_$TAG.log 2>&1; echo rc=$? >> gpurun_out/t_$TAG.log
timeout 400 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"$KRE" -c 1 -o /tmp/e_$TAG python bench.py --profile --cubes 4 --steps 1 --warmup 3 > /dev/null 2>&1
ncu -i /tmp/e_$TAG.ncu-rep --page source --csv > gpurun_out/source_$TAG.csv
ncu -i /tmp/e_$TAG.ncu-rep --page details > gpurun_out/details_$TAG.txt
ncu -i /tmp/e_$TAG.ncu-rep --page raw --csv > gpurun_out/raw_$TAG.csv
