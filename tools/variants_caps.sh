# register-cap A/B: fp32 C4/C3/C2 and fp64 C2/C3/C5 for default vs variant libraries
for v in default "$@"; do
  if [ "$v" = default ]; then unset UUVSIM_B200_LIB; else export UUVSIM_B200_LIB=_variants/$v/libuuvsim_core.so; fi
  for cp in "c4 fp32" "c3 fp32" "c2 fp32" "c2 fp64" "c3 fp64" "c5 fp64"; do
    set -- $cp
    python bench.py --steps 300 --warmup 10 --no-sweep --no-cpu --config $1 --precision $2 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v $1 $2', round(d['ms_per_step']*1e3,2), 'us regs', d['engine']['step_kernel_registers'])"
  done
done
