# Full evidence run for profiles/<round>: smoke, GPU tests, default bench (e2e + cpu baseline + clocks), reference
# arm, per-config bench lines, ncu launch lists of the timed region (--profile-from-start off), one --set full
# capture per hot kernel (k_axis8 cfg3, k_gen cfg1/cfg2/cfg4, k_quad, k_stokes), stall summaries, ncu_counters.json.
#   bash tools/round_evidence.sh r02
set -x
R=${1:-r02}
O=gpurun_out/ev_$R
mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > $O/clocks.csv &
SMI=$!
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err
kill $SMI
python tools/mb_pcie.py > $O/pcie.json 2>&1
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_ref.json 2> $O/bench_ref.err
for C in 0 1 2 4; do timeout 900 python bench.py --config $C --steps 20 --warmup 5 --cpu-seconds 8 > $O/bench_cfg$C.json 2> $O/bench_cfg$C.err; done
timeout 900 python bench.py --config 2 --quad 7 --steps 5 --warmup 3 --no-e2e --cpu-seconds 6 > $O/bench_cfg2_quad7.json 2> $O/bench_cfg2_quad7.err
timeout 900 python bench.py --problem diffreac --k 3 --N 64 --solve --steps 10 --warmup 3 --no-e2e --cpu-seconds 6 > $O/bench_diffreac_k3_64.json 2> $O/bench_diffreac.err
timeout 900 python bench.py --problem nlreac --k 3 --N 64 --jacobian --steps 10 --warmup 3 --no-e2e --cpu-seconds 6 > $O/bench_nljac_k3_64.json 2> $O/bench_nlreac.err
timeout 900 python bench.py --problem stokes --k 3 --N 48 --steps 10 --warmup 3 --no-e2e --cpu-seconds 6 > $O/bench_stokes_k3_48.json 2> $O/bench_stokes.err
timeout 900 python bench.py --config 2 --basis lobatto --steps 10 --warmup 3 --no-e2e --cpu-seconds 6 > $O/bench_cfg2_gll.json 2> $O/bench_cfg2_gll.err
for C in 3 4; do timeout 900 python bench.py --config $C --steps 10 --warmup 3 --dist-loopback --no-cpu-baseline > $O/bench_cfg${C}_distloop.json 2> $O/bench_cfg${C}_distloop.err; done
for C in 3 2 4 1; do
  B="python bench.py --config $C --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
  ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file $O/launches_cfg$C.csv $B > /dev/null 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:k_axis8 -s 3 -c 1 -o $O/prof_axis8_cfg3 python bench.py --config 3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_gen -s 3 -c 1 -o $O/prof_gen_cfg2 python bench.py --config 2 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_gen -s 3 -c 1 -o $O/prof_gen_cfg4 python bench.py --config 4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_line -s 3 -c 1 -o $O/prof_line_cfg1 python bench.py --config 1 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_quad -s 3 -c 1 -o $O/prof_quad_dr3 python bench.py --problem diffreac --k 3 --N 64 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu5.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_stokes -s 3 -c 1 -o $O/prof_stokes_k3 python bench.py --problem stokes --k 3 --N 48 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu7.log 2>&1
python tools/ncu_counters.py $O/ncu_counters.json cfg3_poisson_q7_96:k_axis8:$O/prof_axis8_cfg3.ncu-rep cfg2_diffusion_q5_64_affine:k_gen:$O/prof_gen_cfg2.ncu-rep cfg4_diffusion_q4_256_affine:k_gen:$O/prof_gen_cfg4.ncu-rep cfg1_poisson_q3_32:k_line:$O/prof_line_cfg1.ncu-rep > $O/counters.log 2>&1
for R2 in axis8_cfg3 gen_cfg2 gen_cfg4 line_cfg1 quad_dr3 stokes_k3; do
  python tools/ncu_stalls.py $O/prof_$R2.ncu-rep > $O/stalls_$R2.txt 2>&1
  python tools/ncu_stalls.py $O/prof_$R2.ncu-rep --lines >> $O/stalls_$R2.txt 2>&1
done
python tools/ncu_summary.py --launches $O/launches_cfg3.csv --rep $O/prof_axis8_cfg3.ncu-rep --out $O/ncu_axis8_cfg3 --title "k_axis8 on cfg3 (N=1)" > /dev/null 2>&1
python tools/ncu_summary.py --launches $O/launches_cfg2.csv --rep $O/prof_gen_cfg2.ncu-rep --out $O/ncu_gen_cfg2 --title "k_gen on cfg2 (N=1)" > /dev/null 2>&1
python tools/ncu_summary.py --launches $O/launches_cfg4.csv --rep $O/prof_gen_cfg4.ncu-rep --out $O/ncu_gen_cfg4 --title "k_gen on cfg4 (N=1)" > /dev/null 2>&1
python tools/ncu_summary.py --launches $O/launches_cfg1.csv --rep $O/prof_line_cfg1.ncu-rep --out $O/ncu_line_cfg1 --title "k_line on cfg1 (N=1)" > /dev/null 2>&1
python tools/ncu_summary.py --rep $O/prof_quad_dr3.ncu-rep --out $O/ncu_quad_dr3 --title "k_quad_diffreac, k=3 on 64^3 (SURVEY 8(f1))" > /dev/null 2>&1
python tools/ncu_summary.py --rep $O/prof_stokes_k3.ncu-rep --out $O/ncu_stokes_k3 --title "k_stokes, k=3 on 48^3 (SURVEY 8(f4))" > /dev/null 2>&1
mkdir -p $O/reps && mv $O/prof_gen_cfg4.ncu-rep $O/reps/ 2>/dev/null
rm -f $O/*.ncu-rep
tail -2 $O/pytest_gpu.log
cat $O/bench.json
