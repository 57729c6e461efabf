for T in 2x4 4x4 4x2; do
  export DG_AX8_TILE=$T
  timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "axis8" 2>&1 | tail -1
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$T', d['ms_per_step'], d['value']/1e9, 'GDOF/s')"
done
