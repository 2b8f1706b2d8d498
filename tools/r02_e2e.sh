O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_streamer.py -m gpu -q --timeout 300 > $O/t_i15.log 2>&1; echo rc=$? >> $O/t_i15.log
timeout 900 python bench.py > $O/bench5_i15.log 2>&1; echo rc=$? >> $O/bench5_i15.log
timeout 600 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench2_i15.log 2>&1; echo rc=$? >> $O/bench2_i15.log
