b() { python bench.py --config 1 --steps 30 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('   cfg1', round(d['ms_per_step']*1000,2), 'us', round(d['roofline']['frac'],3))"; }
for V in "2 4 4" "2 4 5" "2 4 6" "4 4 2" "4 4 3" "2 2 8"; do
  set -- $V
  echo "== n=4 tile $1x$2 minB $3"
  DG_BUILD_FLAGS="-DGEN4_T1=$1 -DGEN4_T2=$2 -DGEN4_MB=$3 -DGEN5_T1=2 -DGEN5_T2=4 -DGEN5_MB=2 -DGEN6_T1=2 -DGEN6_T2=2 -DGEN6_MB=2" python -c "from paper_1812_08075_b200 import build as b; b.build(force=True)" > /tmp/bl.log 2>&1 || { echo build failed; continue; }
  b; b
done
python -c "from paper_1812_08075_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
