timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "axis8 or config_sampled" 2>&1 | tail -1
for T in 2x2 2x4; do for CL in 12 96; do
  DG_AX8_TILE=$T DG_AX8_CHUNK=$CL timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$T', $CL, round(d['ms_per_step'],4), round(d['value']/1e9,1), 'GDOF/s')"
done; done
DG_AX8_TILE=2x2 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "axis8" 2>&1 | tail -1
