# k_gen tile / occupancy sweep: rebuild with -DGEN<n>_{T1,T2,MB} and time cfg4 (n=5) and cfg2 (n=6)
b() { python bench.py --config $1 --steps ${2:-10} --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('   cfg$1', round(d['ms_per_step'],4), 'ms', round(d['roofline']['frac'],3))"; }
v() { echo "-DGEN4_T1=2 -DGEN4_T2=4 -DGEN4_MB=4 -DGEN5_T1=$1 -DGEN5_T2=$2 -DGEN5_MB=$3 -DGEN6_T1=$4 -DGEN6_T2=$5 -DGEN6_MB=$6"; }
for V in "$(v 2 2 4 2 2 3)" "$(v 4 2 2 2 2 2)" "$(v 2 2 3 4 2 1)"; do
  echo "== $V"
  DG_BUILD_FLAGS="$V" python -c "from paper_1812_08075_b200 import build as b; b.build(force=True)" > /tmp/bl.log 2>&1 || { echo build failed; tail -3 /tmp/bl.log; continue; }
  b 4 5; b 2 10
done
python -c "from paper_1812_08075_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
