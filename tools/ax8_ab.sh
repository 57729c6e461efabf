# interleaved A/B timing of k_axis8 library variants on cfg3: bash tools/ax8_ab.sh <out> <variant>...
# (variant "default" = lib/libdg.so, else lib/variants/libdg_<variant>.so)
O=gpurun_out/$1; shift
mkdir -p $O
for i in 1 2 3; do
  for V in "$@"; do
    if [ $V = default ]; then L=paper_1812_08075_b200/lib/libdg.so; else L=paper_1812_08075_b200/lib/variants/libdg_$V.so; fi
    DG_LIB=$L timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$V', round(d['ms_per_step'],4), 'sustained', round(d['sustained']['ms_per_apply'],4), d['clocks']['sm_mhz'])" | tee -a $O/ab.txt
  done
done
