#!/bin/bash
# compute-sanitizer stand-in (the tool is closed on this GPU pool): the whole GPU
# test suite against a build with device-side bounds asserts (UUV_BOUNDS_CHECK,
# uuv_kernels.cuh UUV_CHECK: env rows, band lists and chunks, flag bytes, staged
# rows, skip masks) -- any violation traps the kernel and fails its test.
#   python -m paper_2410_14117_b200.build -D UUV_BOUNDS_CHECK --out _variants/bounds/libuuvsim_core.so
#   tools/bounds_run.sh
cd "$(dirname "$0")/.."
export UUVSIM_B200_LIB=$PWD/_variants/bounds/libuuvsim_core.so
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2_bounds_check.log 2>&1
echo "rc=$?" >> gpurun_out/r2_bounds_check.log
tail -3 gpurun_out/r2_bounds_check.log
