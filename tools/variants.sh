# bench prebuilt library variants (_variants/<name>/libuuvsim_core.so)
for v in "$@"; do
  for c in "c5 --pair on"; do
    UUVSIM_B200_LIB=_variants/$v/libuuvsim_core.so python bench.py --steps 500 --warmup 5 --no-sweep --no-cpu --config $c 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v $c', round(d['ms_per_step']*1e3,2), round(d['steady_state']['ms_per_step']*1e3,2), round(d['roofline']['frac'],4), d['engine']['step_kernel_registers'])" 2>&1 | tail -1
  done
done
