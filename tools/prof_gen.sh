# Source-level ncu capture of k_gen on an affine c(x) mesh (development): timing, then one --set full capture
# with source counters; exports the source page as CSV for tools/ncu_smem_regions.py / per-line analysis.
#   bash tools/prof_gen.sh <tag> <k> <N>
T=${1:-g}; K=${2:-4}; NN=${3:-128}
O=gpurun_out/prof_$T
mkdir -p $O
python tools/kbench.py --k $K --N $NN --geom 1 --coeff 1 --R 20 > $O/time.txt 2>&1
python tools/kbench.py --k $K --N 256 --geom 1 --coeff 1 --R 10 >> $O/time.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_gen -s 3 -c 1 -o $O/rep python tools/kbench.py --k $K --N $NN --geom 1 --coeff 1 --R 1 > $O/ncu.log 2>&1
ncu -i $O/rep.ncu-rep --page source --csv --print-source cuda,sass > $O/source.csv 2>/dev/null
ncu -i $O/rep.ncu-rep --page raw --csv > $O/raw.csv 2>/dev/null
python tools/ncu_stalls.py $O/rep.ncu-rep > $O/stalls.txt 2>&1
python tools/ncu_stalls.py $O/rep.ncu-rep --lines >> $O/stalls.txt 2>&1
gzip -f $O/source.csv
rm -f $O/rep.ncu-rep
