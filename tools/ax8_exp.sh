# k_axis8 experiments: phase trace (DG_AX8_TRACE build) + tile/minBlocks variants
set -x
DG_BUILD_FLAGS=-DDG_AX8_TRACE python -c "from paper_1812_08075_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
python tools/trace_ax8.py 3 2>&1 | tail -12
python -c "from paper_1812_08075_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
for T in 2x4m2 2x4m1 4x4m1 2x2m3 2x2m2 4x2m2; do
  DG_AX8_TILE=$T timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$T', round(d['ms_per_step'],4), round(d['value']/1e9,1), 'GDOF/s')"
done
