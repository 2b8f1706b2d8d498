mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -m gpu -x -q -k "fullsize or variants or gram_kernels" > gpurun_out/t_a2.log 2>&1; echo rc=$? >> gpurun_out/t_a2.log
bash tools/profile_cfg.sh c5 5 "k_eval_ssim7 k_gram_px k_pca_project_px k_quantize_planar" --t 96
