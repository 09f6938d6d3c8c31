#!/bin/bash
# Round-2 ncu evidence for profiles/: plain runs first (each must exit 0 without
# ncu), then launch lists (C2, C5 bench commands) and full captures of the step
# kernel and the concurrent fp64 band kernel in the tumbling regime (C2, C5, C3).
cd "$(dirname "$0")/.."
set -x
B="python bench.py --steps 30 --warmup 3 --no-sweep --no-cpu --no-ncu"
P="python bench.py --ncu-probe"
$B > gpurun_out/plain_c2.log 2>&1 && $B --config c5 > gpurun_out/plain_c5.log 2>&1 && \
$B --config c3 > gpurun_out/plain_c3.log 2>&1 || exit 1
$P c2 && $P c5 && $P c3 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r2_launches_c2.csv $B > gpurun_out/ncu_l2.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r2_launches_c5.csv $B --config c5 > gpurun_out/ncu_l5.log 2>&1
for c in c2 c5 c3; do
  ncu --set full --clock-control none --import-source on -k regex:k_step --launch-skip 300 -c 1 -o gpurun_out/r2_step_$c -f $P $c > gpurun_out/ncu_step_$c.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:k_band --launch-skip 300 -c 1 -o gpurun_out/r2_band_$c -f $P $c > gpurun_out/ncu_band_$c.log 2>&1
done
ls -la gpurun_out | tail -20
python tools/profile_summary.py --tag r2 gpurun_out/r2_step_c2.ncu-rep:c2:4096 \
  gpurun_out/r2_step_c5.ncu-rep:c5:1048576 gpurun_out/r2_step_c3.ncu-rep:c3:65536 \
  gpurun_out/r2_band_c2.ncu-rep:c2:4096:band gpurun_out/r2_band_c5.ncu-rep:c5:1048576:band \
  gpurun_out/r2_band_c3.ncu-rep:c3:65536:band \
  --launches gpurun_out/r2_launches_c2.csv --launches gpurun_out/r2_launches_c5.csv
cp profiles/r2_ncu_summary.md gpurun_out/
# keep the copy-back under 64 MiB: only the C5 step capture travels back
rm -f gpurun_out/r2_step_c2.ncu-rep gpurun_out/r2_step_c3.ncu-rep gpurun_out/r2_band_*.ncu-rep
