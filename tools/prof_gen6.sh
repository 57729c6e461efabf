O=gpurun_out/prof_g6; mkdir -p $O
ncu --set full --clock-control none --import-source on -k regex:k_gen -s 3 -c 1 -o $O/rep python tools/kbench.py --k 5 --N 64 --geom 1 --coeff 1 --R 1 > $O/ncu.log 2>&1
ncu -i $O/rep.ncu-rep --page source --csv --print-source cuda,sass > $O/source.csv 2>/dev/null
ncu -i $O/rep.ncu-rep --page details > $O/details.txt 2>/dev/null
python tools/ncu_stalls.py $O/rep.ncu-rep > $O/stalls.txt 2>&1
gzip -f $O/source.csv; rm -f $O/rep.ncu-rep
