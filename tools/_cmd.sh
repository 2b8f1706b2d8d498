mkdir -p gpurun_out
TAG=s8k
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo rc=$? >> gpurun_out/smoke_$TAG.log
if grep -q "rc=0" gpurun_out/smoke_$TAG.log; then
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/t_$TAG.log 2>&1; echo rc=$? >> gpurun_out/t_$TAG.log
for c in 5 2 3; do
  timeout 200 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b${c}_$TAG.log 2>&1; echo rc=$? >> gpurun_out/b${c}_$TAG.log
done
fi
