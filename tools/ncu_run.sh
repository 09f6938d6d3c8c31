set -x
B="python bench.py --steps 20 --warmup 3 --no-sweep --no-cpu"
$B > gpurun_out/plain_c2.log 2>&1 && $B --config c5 > gpurun_out/plain_c5.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches_c2.csv $B > gpurun_out/ncu_l2.log 2>&1 ; \
ncu --set full --clock-control none --import-source on -k regex:k_step -s 3 -c 1 -o gpurun_out/prof_c2 $B > gpurun_out/ncu_c2.log 2>&1 ; \
ncu --set full --clock-control none --import-source on -k regex:k_step -s 3 -c 1 -o gpurun_out/prof_c5 $B --config c5 > gpurun_out/ncu_c5.log 2>&1
ls -la gpurun_out; tail -3 gpurun_out/ncu_c5.log; tail -c 1500 gpurun_out/plain_c2.log
