#!/bin/bash
# Full GPU check on the box: -m gpu suite, smoke, default bench (config 5), config 2 bench.
# usage: tools/gpu_round.sh TAG
TAG=$1
mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi_$TAG.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t_$TAG.log 2>&1; echo rc=$? >> gpurun_out/t_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo rc=$? >> gpurun_out/smoke_$TAG.log
timeout 900 python bench.py > gpurun_out/bench5_$TAG.log 2>&1; echo rc=$? >> gpurun_out/bench5_$TAG.log
timeout 600 python bench.py --config 2 --steps 10 --warmup 3 > gpurun_out/bench2_$TAG.log 2>&1; echo rc=$? >> gpurun_out/bench2_$TAG.log
