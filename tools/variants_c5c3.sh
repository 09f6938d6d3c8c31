# C5 and C3 per-step time for library variants (_variants/<name>/libuuvsim_core.so)
for v in default "$@"; do
  if [ "$v" = default ]; then unset UUVSIM_B200_LIB; else export UUVSIM_B200_LIB=_variants/$v/libuuvsim_core.so; fi
  for c in c5 c3; do
    python bench.py --steps 500 --warmup 10 --no-sweep --no-cpu --config $c 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v $c', round(d['ms_per_step']*1e3,2), 'us  frac', round(d['roofline']['frac'],4), 'regs', d['engine']['step_kernel_registers'])" 2>&1 | tail -1
  done
done
