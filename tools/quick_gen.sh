# k_gen development loop: GPU parity of the k_gen paths + timing of the affine c(x) configs (cfg4-like 128^3 / 256^3,
# cfg2) with tools/kbench.py
timeout 900 python -m pytest tests -m gpu -x -q -k "parity or varjac or halo or dist or slab" 2>&1 | tail -3
python tools/kbench.py --k 4 --N 128 --geom 1 --coeff 1 --R 20
python tools/kbench.py --k 4 --N 256 --geom 1 --coeff 1 --R 10
python tools/kbench.py --k 5 --N 64 --geom 1 --coeff 1 --R 50
python tools/kbench.py --k 3 --N 64 --geom 1 --coeff 1 --R 50
