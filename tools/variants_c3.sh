# C3 per-step time, alternating default and variant libraries (same box)
for rep in 1 2 3; do
  for v in default "$@"; do
    if [ "$v" = default ]; then unset UUVSIM_B200_LIB; else export UUVSIM_B200_LIB=_variants/$v/libuuvsim_core.so; fi
    python bench.py --steps 1000 --warmup 10 --no-sweep --no-cpu --config ${CFG:-c3} 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step']*1e3,2))"
  done
done
