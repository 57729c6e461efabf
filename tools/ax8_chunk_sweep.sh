# k_axis8 planes per work item (DG_AX8_CHUNK) on cfg3 after the table rewrite, interleaved rounds
O=gpurun_out/${1:-chunk}
mkdir -p $O
for i in 1 2; do
  for C in 16 8 12 24 32 48 96; do
    DG_AX8_CHUNK=$C timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('chunk $C', round(d['ms_per_step'],4), 'sustained', round(d['sustained']['ms_per_apply'],4), d['clocks']['sm_mhz'])" | tee -a $O/sweep.txt
  done
done
