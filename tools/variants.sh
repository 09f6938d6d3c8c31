# bench prebuilt library variants (_variants/<name>/libuuvsim_core.so) on C5/C2/C3
for v in "$@"; do
  for c in "c5 --pair on" "c5 --pair off" "c2 --pair off" "c3 --pair off"; do
    UUVSIM_B200_LIB=_variants/$v/libuuvsim_core.so python bench.py --steps 300 --warmup 5 --no-sweep --no-cpu --config $c 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v $c', round(d['ms_per_step']*1e3,2), round(d['steady_state']['ms_per_step']*1e3,2), round(d['roofline']['frac'],4), d['engine']['step_kernel_registers'])" 2>&1 | tail -1
  done
done
