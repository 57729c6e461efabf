# Source-level ncu capture of k_stokes (k = 3, 48^3) (development)
O=gpurun_out/prof_${1:-s0}; mkdir -p $O
python bench.py --problem stokes --k 3 --N 48 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench.json 2> $O/bench.err
ncu --set full --clock-control none --import-source on -k regex:k_stokes -s 3 -c 1 -o $O/rep python bench.py --problem stokes --k 3 --N 48 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu.log 2>&1
ncu -i $O/rep.ncu-rep --page source --csv --print-source cuda,sass > $O/source.csv 2>/dev/null
gzip -f $O/source.csv; rm -f $O/rep.ncu-rep
