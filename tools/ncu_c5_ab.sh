#!/bin/bash
# ncu A/B of the C5 step kernel: band64 off vs on (per-launch time, instructions, DRAM bytes)
cd "$(dirname "$0")/.."
for b in off on; do
  ncu --clock-control none --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread \
      --csv -k regex:"k_step|k_band" --launch-skip 40 --launch-count 4 \
      python -c "
import sys; sys.path.insert(0,'.')
import torch, bench, paper_2410_14117_b200 as uuv
cfg,_=bench.build_config('c5',0,'fp32',band64=('$b'=='on'))
e=uuv.B200EnvBatch(cfg); a=e.bench_actions_tensor()
for _ in range(30): e.step_tensors(a)
torch.cuda.synchronize()" 2>/dev/null | grep -E '"k_|k_step|k_band' | python3 -c "
import sys,csv
for r in csv.reader(sys.stdin):
    print('$b', r[4][:28], r[-3][:34], r[-1])
"
done
