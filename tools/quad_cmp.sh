b() { timeout 300 python bench.py "$@" --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('  ', d['config']['workload'], round(d['ms_per_step'],4), 'ms', round(d['roofline']['frac'],3), d['roofline']['kernel'])"; }
for K in 1 2 3 4; do
  b --problem diffreac --k $K --N 48
  DG_QUAD_CTA=1 b --problem diffreac --k $K --N 48
done
b --config 2 --quad 7
