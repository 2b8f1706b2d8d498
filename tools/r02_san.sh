#!/bin/bash
# compute-sanitizer over a GPU parity subset (mbarrier / cp.async / named-barrier kernels).
# usage: tools/r02_san.sh TAG
TAG=${1:-r02}
O=gpurun_out; mkdir -p $O
SUB="test_stream_golden or test_stream_nan_then_pca or test_ssim_bulk_kernel_shapes or test_pca_golden or test_forward_fill_golden or test_stream_edge_shapes or test_pca_variants_bit_identical or test_psnr_stream_kernel"
timeout 1700 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -m gpu -q \
    --timeout 1600 -p no:cacheprovider -k "$SUB" > $O/san_memcheck_$TAG.log 2>&1; echo rc=$? >> $O/san_memcheck_$TAG.log
timeout 1700 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -m gpu -q \
    --timeout 1600 -p no:cacheprovider -k "test_stream_golden or test_ssim_bulk_kernel_shapes or test_stream_nan_then_pca" \
    > $O/san_racecheck_$TAG.log 2>&1; echo rc=$? >> $O/san_racecheck_$TAG.log
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -m gpu -q \
    --timeout 800 -p no:cacheprovider -k "test_stream_golden or test_ssim_bulk_kernel_shapes" \
    > $O/san_synccheck_$TAG.log 2>&1; echo rc=$? >> $O/san_synccheck_$TAG.log
