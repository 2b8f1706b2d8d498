#!/bin/bash
# Round-2 final GPU pass (one GPU): smoke, -m gpu suite, default bench (config 5, e2e + CPU baseline),
# config 2 full bench, configs 1/3/4, reference arm, launch lists, ncu --set full per hot kernel.
TAG=${1:-r02}
O=gpurun_out; mkdir -p $O
nvidia-smi > $O/smi_$TAG.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$TAG.log 2>&1; echo rc=$? >> $O/smoke_$TAG.log
timeout 1800 python -m pytest tests -m gpu -q --timeout 600 > $O/t_$TAG.log 2>&1; echo rc=$? >> $O/t_$TAG.log
timeout 900 python bench.py > $O/bench5_$TAG.log 2>&1; echo rc=$? >> $O/bench5_$TAG.log
timeout 600 python bench.py --config 2 --steps 10 --warmup 3 > $O/bench2_$TAG.log 2>&1; echo rc=$? >> $O/bench2_$TAG.log
for c in 1 3 4; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench${c}_$TAG.log 2>&1; echo rc=$? >> $O/bench${c}_$TAG.log
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/benchref_$TAG.log 2>&1; echo rc=$? >> $O/benchref_$TAG.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" --csv \
    --log-file $O/launches5_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e \
    > $O/ncu_launch5_$TAG.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" --csv \
    --log-file $O/launches2_$TAG.csv python bench.py --config 2 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e \
    > $O/ncu_launch2_$TAG.log 2>&1
for k in eval_ssim8 gram12 pca_project12 quantize_planar; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_$k" -c 1 -o /tmp/p5_${TAG}_$k \
      python bench.py --config 5 --t 96 --profile --steps 1 --warmup 3 > $O/ncu5_${TAG}_$k.log 2>&1
  ncu -i /tmp/p5_${TAG}_$k.ncu-rep --page raw --csv > $O/raw5_${TAG}_$k.csv
  ncu -i /tmp/p5_${TAG}_$k.ncu-rep --page details > $O/details5_${TAG}_$k.txt
  ncu -i /tmp/p5_${TAG}_$k.ncu-rep --page source --csv > $O/source5_${TAG}_$k.csv
done
for k in eval_ssim8 quantize_planar stats_vec; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_$k" -c 1 -o /tmp/p2_${TAG}_$k \
      python bench.py --config 2 --cubes 4 --profile --steps 1 --warmup 3 > $O/ncu2_${TAG}_$k.log 2>&1
  ncu -i /tmp/p2_${TAG}_$k.ncu-rep --page raw --csv > $O/raw2_${TAG}_$k.csv
  ncu -i /tmp/p2_${TAG}_$k.ncu-rep --page details > $O/details2_${TAG}_$k.txt
  ncu -i /tmp/p2_${TAG}_$k.ncu-rep --page source --csv > $O/source2_${TAG}_$k.csv
done
cuobjdump -sass paper_2506_19656_b200/lib/libcvb200.so 2>/dev/null | grep -E "Function : .*k_eval_ssim8|UBLKCP|UTMALDG|FFMA2|SYNCS" | awk '/Function/{f=$0; next} {c[f" "$2]++} END{for(k in c) print c[k], k}' | sort -rn | head -40 > $O/sass_counts_$TAG.txt 2>&1
