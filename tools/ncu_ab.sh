#!/bin/bash
# ncu A/B of a workload's step kernel with band64 off / on (per-launch time, instructions)
#   tools/ncu_ab.sh c3
cd "$(dirname "$0")/.."
c=${1:-c3}
for b in off on; do
  ncu --clock-control none --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --csv -k regex:"k_step|k_band" --launch-skip 320 --launch-count 6 \
      python -c "
import sys; sys.path.insert(0,'.')
import torch, bench, paper_2410_14117_b200 as uuv
cfg,_=bench.build_config('$c',0,'fp32',band64=('$b'=='on'))
e=uuv.B200EnvBatch(cfg); a=e.bench_actions_tensor()
for _ in range(330): e.step_tensors(a)
torch.cuda.synchronize()" 2>/dev/null | grep -E 'k_step|k_band' | python3 -c "
import sys,csv
for r in csv.reader(sys.stdin):
    print('$b', r[4][:28], r[-3][:30], r[-1])
"
done
