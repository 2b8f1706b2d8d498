#!/bin/bash
TAG=$1
tail -3 gpurun_out/t_$TAG.log
python -c "
import json
d=json.loads(open('gpurun_out/bench_$TAG.log').read().strip().splitlines()[-1]); print(round(d['value'],2), round(d['ms_per_step'],2), {k:round(v['ms'],2) for k,v in d['kernels'].items()})
" || tail -5 gpurun_out/bench_$TAG.log
python tools/ncu_ops.py gpurun_out/source_$TAG.csv 227e6 | head -${3:-14}
grep -E "Duration|Issue Slots|Achieved Occ|Registers Per|Warp Cycles Per Issued|bank" gpurun_out/details_$TAG.txt | head -12
