B="python bench.py --steps 20 --warmup 3 --no-sweep --no-cpu --config c2"
$B > gpurun_out/plain_c2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_step -s 3 -c 1 -o gpurun_out/prof_c2_iter -f $B > gpurun_out/ncu_c2_iter.log 2>&1
tail -1 gpurun_out/ncu_c2_iter.log
