# Source-level ncu capture of k_quad (diffusion-reaction k = 3, 64^3) (development)
O=gpurun_out/prof_${1:-q0}; mkdir -p $O
ncu --set full --clock-control none --import-source on -k regex:k_quad -s 3 -c 1 -o $O/rep python bench.py --problem diffreac --k 3 --N 64 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu.log 2>&1
ncu -i $O/rep.ncu-rep --page source --csv --print-source cuda,sass > $O/source.csv 2>/dev/null
python tools/ncu_stalls.py $O/rep.ncu-rep > $O/stalls.txt 2>&1
gzip -f $O/source.csv; rm -f $O/rep.ncu-rep
