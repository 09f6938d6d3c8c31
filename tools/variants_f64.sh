for v in default "$@"; do
  if [ "$v" = default ]; then unset UUVSIM_B200_LIB; else export UUVSIM_B200_LIB=_variants/$v/libuuvsim_core.so; fi
  for c in c2 c3 c5; do
    python bench.py --steps 200 --warmup 10 --no-sweep --no-cpu --config $c --precision fp64 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v $c fp64', round(d['ms_per_step']*1e3,2), 'us regs', d['engine']['step_kernel_registers'])"
  done
done
