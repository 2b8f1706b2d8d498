#!/bin/bash
# GPU iteration: smoke, GPU suite, quick benches (config 5 / 3 / 2, optional variants).
# usage: tools/r02_iter.sh TAG ["pytest -k expr"]
TAG=$1; K=$2
O=gpurun_out; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$TAG.log 2>&1; echo rc=$? >> $O/smoke_$TAG.log
if [ -n "$K" ]; then KX=(-k "$K"); else KX=(); fi
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 "${KX[@]}" > $O/t_$TAG.log 2>&1; echo rc=$? >> $O/t_$TAG.log
B="--steps 5 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 python bench.py --config 5 $B > $O/b5_$TAG.log 2>&1; echo rc=$? >> $O/b5_$TAG.log
timeout 300 python bench.py --config 3 $B > $O/b3_$TAG.log 2>&1; echo rc=$? >> $O/b3_$TAG.log
timeout 300 python bench.py --config 2 $B > $O/b2_$TAG.log 2>&1; echo rc=$? >> $O/b2_$TAG.log
timeout 300 python bench.py --config 2 $B --variant eval_kernel=8 > $O/b2k8_$TAG.log 2>&1; echo rc=$? >> $O/b2k8_$TAG.log
timeout 300 python bench.py --config 5 $B --variant proj12=0 --variant gram_checks=1 > $O/b5old_$TAG.log 2>&1; echo rc=$? >> $O/b5old_$TAG.log
