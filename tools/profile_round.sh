#!/bin/bash
# Round profile capture (run on the GPU box, one GPU): launch list of the
# default bench + one `ncu --set full` capture per hot kernel, exported as CSV
# into gpurun_out/ for tools/make_profiles.py.
TAG=${1:-r01}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e \
    > gpurun_out/ncu_launch_$TAG.log 2>&1
for k in eval_ssim quantize_planar stats_vec; do
  ncu --set full --clock-control none --import-source on -k regex:"k_$k" -c 1 -o /tmp/p_$k \
      python bench.py --profile --cubes 4 --steps 1 --warmup 3 > gpurun_out/ncu_$k.log 2>&1
  ncu -i /tmp/p_$k.ncu-rep --page raw --csv > gpurun_out/raw_$k.csv
  ncu -i /tmp/p_$k.ncu-rep --page details > gpurun_out/details_$k.txt
  ncu -i /tmp/p_$k.ncu-rep --page source --csv > gpurun_out/source_$k.csv
done
