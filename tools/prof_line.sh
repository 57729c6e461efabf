O=gpurun_out/prof_$1; mkdir -p $O
python tools/kbench.py --k 3 --N 32 --geom 0 --coeff 0 --R 50 --graph > $O/time.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_line|k_blk" -s 3 -c 1 -o $O/rep python tools/kbench.py --k 3 --N 32 --geom 0 --coeff 0 --R 5 > $O/ncu.log 2>&1
ncu -i $O/rep.ncu-rep --page raw --csv > $O/raw.csv 2>/dev/null
ncu -i $O/rep.ncu-rep --page details > $O/details.txt 2>/dev/null
python tools/ncu_stalls.py $O/rep.ncu-rep > $O/stalls.txt 2>&1
python tools/ncu_stalls.py $O/rep.ncu-rep --lines >> $O/stalls.txt 2>&1
rm -f $O/rep.ncu-rep
