"""B200-native matrix-free SIPG-DG operator with sum factorisation (arXiv 1812.08075 hot path).

Layout: csrc/ (CUDA kernels + C-ABI, built into lib/libdg.so), dg.py (ctypes binding with the
C names), slab.py (x0-slab domain decomposition with a torch.distributed/NCCL halo exchange).
"""
from .dg import (DgError, Operator, dg_alg_bytes, dg_alg_flops, dg_apply, dg_apply_host,  # noqa: F401
                 dg_apply_planes, dg_destroy, dg_kernel_name, dg_last_error, dg_launches_per_apply,
                 dg_local_ndofs, dg_local_offset, dg_plane_ndofs, dg_set_stream, dg_setup, load)
