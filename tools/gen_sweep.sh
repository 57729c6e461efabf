# k_gen tile / occupancy sweep: rebuild with -DGEN<n>_{T1,T2,MB} and time cfg1 (n=4), cfg2 (n=6), cfg4 (n=5)
b() { python bench.py --config $1 --steps ${2:-10} --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('   cfg$1', round(d['ms_per_step'],4), 'ms', round(d['roofline']['frac'],3))"; }
v() { echo "-DGEN4_T1=$1 -DGEN4_T2=$2 -DGEN4_MB=$3 -DGEN5_T1=$4 -DGEN5_T2=$5 -DGEN5_MB=$6 -DGEN6_T1=$7 -DGEN6_T2=$8 -DGEN6_MB=$9"; }
for V in "$(v 2 4 3 2 2 3 2 2 2)" "$(v 2 4 4 2 2 4 2 2 3)" "$(v 2 2 4 2 4 2 2 4 1)" "$(v 4 4 2 4 2 2 4 2 1)"; do
  echo "== $V"
  DG_BUILD_FLAGS="$V" python -c "from paper_1812_08075_b200 import build as b; b.build(force=True)" > /tmp/bl.log 2>&1 || { echo build failed; tail -3 /tmp/bl.log; continue; }
  b 1 20; b 2 10; b 4 5
done
python -c "from paper_1812_08075_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
