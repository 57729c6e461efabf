./tools/proto_slab 32
./tools/proto_slab 128
for rep in 1 2; do DG_LIB=paper_1812_08075_b200/lib/libdg_vol.so python tools/kbench.py --k 4 --N 128 --geom 1 --coeff 1 --R 20 2>&1 | tail -1; python tools/kbench.py --k 4 --N 128 --geom 1 --coeff 1 --R 20 2>&1 | tail -1; done
