# Full evidence run for profiles/: tests, smoke, default bench (with e2e + cpu baseline), ncu launch list and full capture of the top kernel
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > gpurun_out/clocks.csv &
SMI=$!
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
kill $SMI
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
for C in 0 1 2 4; do timeout 600 python bench.py --config $C --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_cfg$C.json 2>&1; done
C="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline"
$C > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv $C > gpurun_out/ncu_launch.log 2>&1
C2="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$C2 > gpurun_out/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_axis8 -s 3 -c 1 -o gpurun_out/prof_top $C2 > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/pytest_gpu.log
