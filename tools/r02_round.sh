#!/bin/bash
# Round-2 GPU pass on the box (one GPU): smoke, -m gpu suite, default bench (config 5) with
# e2e + CPU baseline, config 2/3 benches, ncu launch list of the default bench, one
# `ncu --set full` capture per hot kernel (T = 96 prefix of config 5 so the replays stay
# bounded), compute-sanitizer memcheck / racecheck over a parity subset.
# usage: tools/r02_round.sh TAG [skip-list: tests,bench,ncu,san]
TAG=${1:-r02}; SKIP=${2:-""}
O=gpurun_out; mkdir -p $O
nvidia-smi > $O/smi_$TAG.txt 2>&1
has() { case ",$SKIP," in *",$1,"*) return 0;; *) return 1;; esac; }

timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$TAG.log 2>&1; echo rc=$? >> $O/smoke_$TAG.log
if ! has tests; then
  timeout 1800 python -m pytest tests -m gpu -q -x --timeout 600 > $O/t_$TAG.log 2>&1; echo rc=$? >> $O/t_$TAG.log
fi
if ! has bench; then
  timeout 900 python bench.py > $O/bench5_$TAG.log 2>&1; echo rc=$? >> $O/bench5_$TAG.log
  timeout 600 python bench.py --config 2 --steps 10 --warmup 3 > $O/bench2_$TAG.log 2>&1; echo rc=$? >> $O/bench2_$TAG.log
  for c in 1 3 4; do
    timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench${c}_$TAG.log 2>&1; echo rc=$? >> $O/bench${c}_$TAG.log
  done
fi
if ! has ncu; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" --csv \
      --log-file $O/launches5_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e \
      > $O/ncu_launch5_$TAG.log 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" --csv \
      --log-file $O/launches2_$TAG.csv python bench.py --config 2 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e \
      > $O/ncu_launch2_$TAG.log 2>&1
  for k in eval_ssim8 quantize_planar gram_px pca_project_px stats_vec; do
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_$k" -c 1 -o /tmp/p5_${TAG}_$k \
        python bench.py --config 5 --t 96 --profile --steps 1 --warmup 3 > $O/ncu5_${TAG}_$k.log 2>&1
    ncu -i /tmp/p5_${TAG}_$k.ncu-rep --page raw --csv > $O/raw5_${TAG}_$k.csv
    ncu -i /tmp/p5_${TAG}_$k.ncu-rep --page details > $O/details5_${TAG}_$k.txt
    ncu -i /tmp/p5_${TAG}_$k.ncu-rep --page source --csv > $O/source5_${TAG}_$k.csv
  done
  for k in eval_ssim7; do
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_$k" -c 1 -o /tmp/p2_${TAG}_$k \
        python bench.py --config 2 --cubes 4 --profile --steps 1 --warmup 3 > $O/ncu2_${TAG}_$k.log 2>&1
    ncu -i /tmp/p2_${TAG}_$k.ncu-rep --page raw --csv > $O/raw2_${TAG}_$k.csv
    ncu -i /tmp/p2_${TAG}_$k.ncu-rep --page details > $O/details2_${TAG}_$k.txt
    ncu -i /tmp/p2_${TAG}_$k.ncu-rep --page source --csv > $O/source2_${TAG}_$k.csv
  done
fi
if ! has san; then
  SUB="test_stream_golden or test_stream_nan_then_pca or test_ssim_bulk_kernel_shapes or test_pca_golden or test_forward_fill_golden or test_stream_edge_shapes"
  timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -m gpu -q -x \
      --timeout 1200 -k "$SUB" > $O/san_memcheck_$TAG.log 2>&1; echo rc=$? >> $O/san_memcheck_$TAG.log
  timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -m gpu -q -x \
      --timeout 1200 -k "test_stream_golden or test_ssim_bulk_kernel_shapes or test_stream_nan_then_pca" \
      > $O/san_racecheck_$TAG.log 2>&1; echo rc=$? >> $O/san_racecheck_$TAG.log
fi
