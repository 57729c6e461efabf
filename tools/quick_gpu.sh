# quick correctness + timing sweep used during development
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q --timeout=120 2>&1 | tail -3
for C in 0 1 2 3 4; do
  timeout 120 python bench.py --config $C --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($C, round(d['ms_per_step'],4), 'ms', round(d['value']/1e9,2), 'GDOF/s', d['roofline']['bound'], round(d['roofline']['frac'],3), d['roofline']['kernel'])"
done
