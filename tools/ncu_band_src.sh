#!/bin/bash
# ncu source-level capture of the band kernel (k_band) on C2 with every env a
# band candidate (device.band_margin = 10): two blocks replaying ~32 envs per
# thread back to back -- long enough for per-instruction stall sampling.
#   tools/ncu_band_src.sh [out-name]
cd "$(dirname "$0")/.."
out=${1:-band_c2_all}
ncu --set full --import-source on --warp-sampling-interval 0 --clock-control none -k regex:k_band --launch-skip 20 --launch-count 1 \
    -f -o gpurun_out/$out python -c "
import sys; sys.path.insert(0,'.')
import torch, bench, paper_2410_14117_b200 as uuv
cfg,_=bench.build_config('c2',0,'fp32')
cfg['device']['band_margin'] = 10.0
e=uuv.B200EnvBatch(cfg); a=e.bench_actions_tensor()
for _ in range(30): e.step_tensors(a)
torch.cuda.synchronize()" > gpurun_out/$out.log 2>&1
ncu -i gpurun_out/$out.ncu-rep --page source --csv --print-source sass > gpurun_out/$out.src.csv 2>/dev/null
rm -f gpurun_out/$out.ncu-rep
