# Evidence refresh for the k_gen rows (cfg2, cfg4) after a k_gen change: smoke, full GPU suite, bench lines, ncu
# launch lists, one --set full capture per config, ncu_counters merge, summaries.
#   bash tools/evidence_gen.sh <out-dir>
set -x
O=${1:-gpurun_out/ev_gen}
mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
for C in 2 4; do timeout 900 python bench.py --config $C --steps 20 --warmup 5 --cpu-seconds 8 > $O/bench_cfg$C.json 2> $O/bench_cfg$C.err; done
for C in 2 4; do
  ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file $O/launches_cfg$C.csv python bench.py --config $C --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:k_gen -s 3 -c 1 -o $O/prof_gen_cfg2 python bench.py --config 2 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_gen -s 3 -c 1 -o $O/prof_gen_cfg4 python bench.py --config 4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu4.log 2>&1
cp profiles/r02/ncu_counters.json $O/ncu_counters.json
python tools/ncu_counters.py $O/ncu_counters.json cfg2_diffusion_q5_64_affine:k_gen:$O/prof_gen_cfg2.ncu-rep cfg4_diffusion_q4_256_affine:k_gen:$O/prof_gen_cfg4.ncu-rep > $O/counters.log 2>&1
for R2 in gen_cfg2 gen_cfg4; do
  python tools/ncu_stalls.py $O/prof_$R2.ncu-rep > $O/stalls_$R2.txt 2>&1
  python tools/ncu_stalls.py $O/prof_$R2.ncu-rep --lines >> $O/stalls_$R2.txt 2>&1
done
python tools/ncu_summary.py --launches $O/launches_cfg2.csv --rep $O/prof_gen_cfg2.ncu-rep --out $O/ncu_gen_cfg2 --title "k_gen on cfg2 (N=1)" > /dev/null 2>&1
python tools/ncu_summary.py --launches $O/launches_cfg4.csv --rep $O/prof_gen_cfg4.ncu-rep --out $O/ncu_gen_cfg4 --title "k_gen on cfg4 (N=1)" > /dev/null 2>&1
rm -f $O/*.ncu-rep
tail -2 $O/pytest_gpu.log
