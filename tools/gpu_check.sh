#!/bin/bash
# One GPU iteration on the box: full -m gpu suite, then the default bench.
# usage: tools/gpu_check.sh TAG [pytest -k expr] [bench args...]
TAG=$1; K=${2:-""}; shift 2; BARGS="$@"
mkdir -p gpurun_out
if [ -n "$K" ]; then KX=(-k "$K"); else KX=(); fi
timeout 1500 python -m pytest tests -m gpu -x -q "${KX[@]}" > gpurun_out/t_$TAG.log 2>&1; echo rc=$? >> gpurun_out/t_$TAG.log
timeout 900 python bench.py $BARGS > gpurun_out/bench_$TAG.log 2>&1; echo rc=$? >> gpurun_out/bench_$TAG.log
