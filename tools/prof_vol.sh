O=gpurun_out/prof_vol; mkdir -p $O
DG_LIB=paper_1812_08075_b200/lib/libdg_vol.so ncu --set full --clock-control none --import-source on -k regex:k_gen -s 3 -c 1 -o $O/rep python tools/kbench.py --k 4 --N 128 --geom 1 --coeff 1 --R 1 > $O/ncu.log 2>&1
ncu -i $O/rep.ncu-rep --page details > $O/details.txt 2>/dev/null
python tools/ncu_stalls.py $O/rep.ncu-rep > $O/stalls.txt 2>&1
python tools/ncu_stalls.py $O/rep.ncu-rep --lines >> $O/stalls.txt 2>&1
ncu --set full --clock-control none -k regex:k_slab -s 1 -c 1 -o $O/slab ./tools/proto_slab 128 > $O/ncu_slab.log 2>&1
ncu -i $O/slab.ncu-rep --page details > $O/details_slab.txt 2>/dev/null
python tools/ncu_stalls.py $O/slab.ncu-rep > $O/stalls_slab.txt 2>&1
rm -f $O/*.ncu-rep
