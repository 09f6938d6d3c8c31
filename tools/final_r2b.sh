#!/bin/bash
# Round-2 evidence, part 2: the same bench with the fp64 band off (round-1
# fp32-only engine, same box) and the strict parity reports (65,536 envs x every
# config; 2^20 envs x the bench configs).
cd "$(dirname "$0")/.."
python bench.py --band64 off --no-cpu --no-ncu > gpurun_out/r2_bench_band_off.json 2> gpurun_out/r2_bench_band_off.err
echo "bench band-off rc=$?"
python tools/parity_report.py --envs 65536 --out gpurun_out/r2_parity.json --md gpurun_out/r2_parity.md > gpurun_out/parity.log 2>&1
echo "parity rc=$?"
python tools/parity_report.py --envs 1048576 --configs bench_c5,bench_c3,station_heavy,lemniscate_heavy_drep,mixed_station_dr \
    --out gpurun_out/r2_parity_1m.json --md gpurun_out/r2_parity_1m.md > gpurun_out/parity_1m.log 2>&1
echo "parity 1m rc=$?"
