cd $GRAFT_REPO_ROOT
ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.max,smsp__inst_executed.sum --clock-control none -k regex:k_band --launch-skip 20 --launch-count 3 --csv python -c "
import sys; sys.path.insert(0,'.')
import torch, bench, paper_2410_14117_b200 as uuv
cfg,_=bench.build_config('c2',0,'fp32')
cfg['device']['band_margin'] = 10.0
e=uuv.B200EnvBatch(cfg); a=e.bench_actions_tensor()
for _ in range(30): e.step_tensors(a)
print('band64 per step', e.stats()['band64_steps']/30)
torch.cuda.synchronize()" > gpurun_out/ncu_dur.log 2>&1
