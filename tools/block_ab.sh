# C2 device step + mapped e2e for block-size variants (_variants/<name>/libuuvsim_core.so)
for v in default "$@"; do
  if [ "$v" = default ]; then unset UUVSIM_B200_LIB; else export UUVSIM_B200_LIB=_variants/$v/libuuvsim_core.so; fi
  for c in c2 c4; do
    python bench.py --steps 2000 --warmup 20 --no-sweep --no-cpu --config $c 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v $c dev_us', round(d['ms_per_step']*1e3,2), 'b2b_us', round(d['steady_state']['ms_per_step']*1e3,2), 'e2e', round(d['e2e']['value']/1e6,1), 'M/s regs', d['engine']['step_kernel_registers'])" 2>&1 | tail -1
  done
done
