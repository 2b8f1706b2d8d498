#!/bin/bash
# pipe-rate microbenchmark + ncu --set full of the given config 5 kernels (T = 96 prefix)
TAG=$1; KS=$2
O=gpurun_out; mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pipe_rates tools/pipe_rates.cu > $O/pipe_rates_$TAG.txt 2>&1 && /tmp/pipe_rates >> $O/pipe_rates_$TAG.txt 2>&1
cuobjdump -sass /tmp/pipe_rates | grep -E "Function|FFMA2|DFMA|HFMA2" | sort | uniq -c | sort -rn | head -40 > $O/pipe_rates_sass_$TAG.txt 2>&1
for k in $KS; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_$k" -c 1 -o /tmp/p5_${TAG}_$k \
      python bench.py --config 5 --t 96 --profile --steps 1 --warmup 3 > $O/ncu5_${TAG}_$k.log 2>&1
  ncu -i /tmp/p5_${TAG}_$k.ncu-rep --page raw --csv > $O/raw5_${TAG}_$k.csv
  ncu -i /tmp/p5_${TAG}_$k.ncu-rep --page details > $O/details5_${TAG}_$k.txt
  ncu -i /tmp/p5_${TAG}_$k.ncu-rep --page source --csv > $O/source5_${TAG}_$k.csv
done
