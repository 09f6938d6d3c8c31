# one iteration on the GPU box: parity tests, bench, ncu capture of the C5 step kernel
set -x
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -5
python bench.py --steps 2000 --warmup 10 --no-cpu > gpurun_out/bench_iter.log 2>&1; tail -c 2200 gpurun_out/bench_iter.log; timeout 300 python tools/parity_report.py 2>&1 | tail -8
B="python bench.py --steps 20 --warmup 3 --no-sweep --no-cpu --config c5"
$B > gpurun_out/plain_c5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_step -s 3 -c 1 -o gpurun_out/prof_c5_iter -f $B > gpurun_out/ncu_c5_iter.log 2>&1
tail -2 gpurun_out/ncu_c5_iter.log
