#!/bin/bash
# GPU iteration: smoke, GPU suite, quick benches, launch list of config 5.
TAG=$1; K=$2
O=gpurun_out; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$TAG.log 2>&1; echo rc=$? >> $O/smoke_$TAG.log
if [ -n "$K" ]; then KX=(-k "$K"); else KX=(); fi
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 "${KX[@]}" > $O/t_$TAG.log 2>&1; echo rc=$? >> $O/t_$TAG.log
B="--steps 5 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 python bench.py --config 5 $B > $O/b5_$TAG.log 2>&1; echo rc=$? >> $O/b5_$TAG.log
timeout 300 python bench.py --config 3 $B > $O/b3_$TAG.log 2>&1; echo rc=$? >> $O/b3_$TAG.log
timeout 300 python bench.py --config 5 $B --variant gram12=0 --variant proj12=0 > $O/b5old_$TAG.log 2>&1; echo rc=$? >> $O/b5old_$TAG.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" --csv \
    --log-file $O/launches5_$TAG.csv python bench.py --config 5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e \
    > $O/ncu_launch5_$TAG.log 2>&1
