#!/bin/bash
# GPU iteration: GPU tests (optionally filtered), then quick benches of the given configs.
# usage: tools/gpu_iter.sh TAG "pytest -k expr" "5 2"
TAG=$1; K=$2; CFGS=${3:-"5 2"}
mkdir -p gpurun_out
if [ -n "$K" ]; then KX=(-k "$K"); else KX=(); fi
timeout 600 python -m pytest tests -m gpu -x -q --timeout 120 "${KX[@]}" > gpurun_out/t_$TAG.log 2>&1; echo rc=$? >> gpurun_out/t_$TAG.log
for c in $CFGS; do
  timeout 240 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b${c}_$TAG.log 2>&1; echo rc=$? >> gpurun_out/b${c}_$TAG.log
done
