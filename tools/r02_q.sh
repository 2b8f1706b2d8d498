O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -k "quant or stream or config or golden or psnr or batch or sharded or streamer or variants or fill" > $O/t_i19.log 2>&1; echo rc=$? >> $O/t_i19.log
B="--steps 5 --warmup 3 --no-e2e --no-cpu-baseline"
for c in 2 4 1 5; do timeout 300 python bench.py --config $c $B > $O/b${c}_i19.log 2>&1; echo rc=$? >> $O/b${c}_i19.log; done
timeout 300 python bench.py --config 2 $B --variant qp_runtime_c=1 > $O/b2old_i19.log 2>&1
