# ncu evidence for profiles/: launch list (C2) + full captures of the step kernel (C2, C5, C3)
set -x
B="python bench.py --steps 30 --warmup 3 --no-sweep --no-cpu"
$B > gpurun_out/plain_c2.log 2>&1 && $B --config c5 > gpurun_out/plain_c5.log 2>&1 && $B --config c3 > gpurun_out/plain_c3.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/launches_c2.csv $B > gpurun_out/ncu_l2.log 2>&1 ; \
ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/launches_c5.csv $B --config c5 > gpurun_out/ncu_l5.log 2>&1 ; \
ncu --set full --clock-control none --import-source on -k regex:k_step -s 3 -c 1 -o gpurun_out/prof_c2 -f $B > gpurun_out/ncu_c2.log 2>&1 ; \
ncu --set full --clock-control none --import-source on -k regex:k_step -s 3 -c 1 -o gpurun_out/prof_c5 -f $B --config c5 > gpurun_out/ncu_c5.log 2>&1 ; \
ncu --set full --clock-control none --import-source on -k regex:k_step -s 3 -c 1 -o gpurun_out/prof_c3 -f $B --config c3 > gpurun_out/ncu_c3.log 2>&1
ls -la gpurun_out | tail -12
