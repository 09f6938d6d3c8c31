#!/bin/bash
# Round-2 end-of-round evidence: GPU tests, the default bench line and the
# reference arm (each as the driver runs them), copied to gpurun_out/.
cd "$(dirname "$0")/.."
python -m pytest tests -m gpu -q > gpurun_out/r2_gpu_tests.log 2>&1
tail -2 gpurun_out/r2_gpu_tests.log
python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err
echo "bench rc=$?"
python bench.py --impl reference > gpurun_out/r2_bench_reference.json 2> gpurun_out/r2_bench_reference.err
echo "reference rc=$?"
