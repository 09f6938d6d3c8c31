for c in c2 c5 c4 c3; do for so in on off; do
python bench.py --steps 500 --warmup 10 --no-cpu --no-sweep --config $c --stage-obs $so 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c stage=$so', round(d['ms_per_step']*1e3,2), round(d['steady_state']['ms_per_step']*1e3,2), round(d['roofline']['frac'],4))"
done; done
