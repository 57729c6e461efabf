"""Thin Python binding of libdg (include/dg.h) — argument marshalling only.

Every step of the operator runs in the CUDA kernels of libdg.so; this module only converts
torch tensors / numpy arrays into the C-ABI's plain pointers and sizes. There is no CPU
path: if libdg.so is missing or no CUDA device is present, the calls raise.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DG_LIB") or os.path.join(_HERE, "lib", "libdg.so")  # DG_LIB: experiment variants only

DG_OK = 0
DG_ERR_INVALID = -1
DG_ERR_UNSUPPORTED = -2
DG_ERR_CUDA = -3
DG_ERR_NCCL = -4
DG_ERR_OOM = -5
DG_GEOM_AXIS = 0
DG_GEOM_AFFINE = 1
DG_COEFF_ONE = 0
DG_COEFF_SINCOS = 1
DG_PROBLEM_PERIODIC = 0
DG_PROBLEM_DIFFREAC = 1
DG_PROBLEM_NLREAC = 2
DG_PROBLEM_STOKES = 3
DG_BASIS_GAUSS, DG_BASIS_LOBATTO, DG_BASIS_EQUIDISTANT = 0, 1, 2

_ERRNAMES = {-1: "DG_ERR_INVALID", -2: "DG_ERR_UNSUPPORTED", -3: "DG_ERR_CUDA", -4: "DG_ERR_NCCL", -5: "DG_ERR_OOM"}


class DgError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{_ERRNAMES.get(code, code)}: {msg}")
        self.code = code


class dg_mesh(ctypes.Structure):
    _fields_ = [
        ("N", ctypes.c_int32 * 3),
        ("plane_begin", ctypes.c_int32),
        ("nplanes", ctypes.c_int32),
        ("geom_kind", ctypes.c_int32),
        ("jac", ctypes.POINTER(ctypes.c_double)),
        ("coeff_kind", ctypes.c_int32),
        ("penalty_scale", ctypes.c_double),
        ("device", ctypes.c_int32),
        ("stream", ctypes.c_void_p),
        ("problem", ctypes.c_int32),
        ("basis", ctypes.c_int32),
    ]


EXPORTS = ["dg_setup", "dg_apply", "dg_apply_planes", "dg_apply_host", "dg_destroy", "dg_set_stream",
           "dg_local_ndofs", "dg_local_offset", "dg_plane_ndofs", "dg_alg_flops", "dg_alg_bytes",
           "dg_launches_per_apply", "dg_kernel_name", "dg_last_error", "dg_bench_fp64", "dg_line_ops", "dg_line_ops_axis8",
           "dg_apply_jacobian", "dg_apply_jacobian_planes", "dg_halo_ndofs", "dg_pack_halo", "dg_apply_planes_tr", "dg_slab_range", "dg_get_unique_id",
           "dg_setup_dist", "dg_apply_dist"]

_lib = None


def load(path: str = LIB_PATH):
    """dlopen libdg.so (raises if it has not been built — no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"libdg.so not built at {path}: run `python -m paper_1812_08075_b200.build` "
                          "or __graft_entry__.build() (there is no CPU fallback)")
    L = ctypes.CDLL(path)
    vp, dp = ctypes.c_void_p, ctypes.POINTER(ctypes.c_double)
    L.dg_setup.argtypes = [ctypes.POINTER(dg_mesh), ctypes.c_int, ctypes.c_int, ctypes.POINTER(vp)]
    L.dg_apply.argtypes = [vp, vp, vp]
    L.dg_apply_planes.argtypes = [vp, vp, vp, vp, vp, ctypes.c_int, ctypes.c_int]
    L.dg_apply_planes_tr.argtypes = [vp, vp, vp, vp, vp, ctypes.c_int, ctypes.c_int]
    L.dg_pack_halo.argtypes = [vp, vp, vp, vp]
    L.dg_slab_range.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int32),
                                ctypes.POINTER(ctypes.c_int32)]
    L.dg_get_unique_id.argtypes = [vp]
    L.dg_setup_dist.argtypes = [ctypes.POINTER(dg_mesh), ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, vp,
                                ctypes.POINTER(vp)]
    L.dg_apply_dist.argtypes = [vp, vp, vp]
    L.dg_apply_host.argtypes = [vp, vp, vp]
    L.dg_apply_jacobian.argtypes = [vp, vp, vp, vp]
    L.dg_apply_jacobian_planes.argtypes = [vp, vp, vp, vp, vp, vp, ctypes.c_int, ctypes.c_int]
    L.dg_destroy.argtypes = [vp]
    L.dg_set_stream.argtypes = [vp, vp]
    for f in ("dg_local_ndofs", "dg_local_offset", "dg_plane_ndofs", "dg_halo_ndofs"):
        getattr(L, f).argtypes = [vp]
        getattr(L, f).restype = ctypes.c_int64
    for f in ("dg_alg_flops", "dg_alg_bytes"):
        getattr(L, f).argtypes = [vp]
        getattr(L, f).restype = ctypes.c_double
    L.dg_launches_per_apply.argtypes = [vp]
    L.dg_kernel_name.argtypes = [vp]
    L.dg_kernel_name.restype = ctypes.c_char_p
    L.dg_last_error.restype = ctypes.c_char_p
    L.dg_bench_fp64.argtypes = [ctypes.c_int, ctypes.c_int, dp, dp]
    L.dg_line_ops.argtypes = [ctypes.c_int, ctypes.c_double, vp, vp, vp]
    L.dg_line_ops_axis8.argtypes = [ctypes.c_double, vp, vp, vp]
    _lib = L
    return L


def _check(rc: int):
    if rc != DG_OK:
        raise DgError(rc, load().dg_last_error().decode())


def _ptr(t) -> int:
    """Raw pointer of a torch tensor or numpy array."""
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


# ------------------------------------------------------------------ C-ABI with the same names
def dg_setup(N, k: int, quad: int, *, plane_begin: int = 0, nplanes: int | None = None, geom_kind: int = 0,
             jac: np.ndarray | None = None, coeff_kind: int = 0, penalty_scale: float = 10.0, device: int = 0,
             stream: int | None = None, problem: int = 0, basis: int = 0) -> int:
    """Returns an opaque context handle (int). jac: host float64 array [(L+2) N1 N2, 9] for affine; basis:
    DG_BASIS_GAUSS (0) or DG_BASIS_LOBATTO (1)."""
    m, _keep = _mesh(N, plane_begin, nplanes, geom_kind, jac, coeff_kind, penalty_scale, device, stream, problem, basis)
    h = ctypes.c_void_p()
    _check(load().dg_setup(ctypes.byref(m), k, quad, ctypes.byref(h)))
    return h.value


def _mesh(N, plane_begin, nplanes, geom_kind, jac, coeff_kind, penalty_scale, device, stream, problem, basis=0):
    """dg_mesh for the C-ABI (+ the contiguous jac array it points to, kept alive by the caller)."""
    m = dg_mesh()
    m.N[0], m.N[1], m.N[2] = int(N[0]), int(N[1]), int(N[2])
    m.plane_begin = plane_begin
    m.nplanes = int(N[0]) if nplanes is None else nplanes
    m.geom_kind = geom_kind
    keep = None
    if jac is not None:
        keep = np.ascontiguousarray(jac, dtype=np.float64)
        need = 9 * (m.nplanes + 2) * int(N[1]) * int(N[2])
        if keep.size != need:
            raise DgError(DG_ERR_INVALID, f"jac has {keep.size} doubles, the slab needs {need} (9 per cell of L+2 planes)")
        m.jac = keep.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    m.coeff_kind = coeff_kind
    m.penalty_scale = float(penalty_scale)
    m.device = device
    m.stream = stream
    m.problem = problem
    m.basis = basis
    return m, keep


def dg_slab_range(N0: int, rank: int, nranks: int):
    """(plane_begin, nplanes) of a rank in the collective form's x0-slab split."""
    b, n = ctypes.c_int32(), ctypes.c_int32()
    _check(load().dg_slab_range(int(N0), rank, nranks, ctypes.byref(b), ctypes.byref(n)))
    return b.value, n.value


def dg_get_unique_id() -> bytes:
    """A 128-byte ncclUniqueId for dg_setup_dist (create on one rank, broadcast)."""
    buf = ctypes.create_string_buffer(128)
    _check(load().dg_get_unique_id(buf))
    return buf.raw


def dg_setup_dist(N, k: int, quad: int, rank: int, nranks: int, nccl_id: bytes, *, geom_kind: int = 0,
                  jac: np.ndarray | None = None, coeff_kind: int = 0, penalty_scale: float = 10.0, device: int = 0,
                  stream: int | None = None, problem: int = 0, basis: int = 0) -> int:
    """Collective context for rank `rank` of `nranks` (include/dg.h): jac covers the rank's L+2 planes."""
    pb, npl = dg_slab_range(int(N[0]), rank, nranks)
    m, _keep = _mesh(N, pb, npl, geom_kind, jac, coeff_kind, penalty_scale, device, stream, problem, basis)
    if len(nccl_id) != 128:
        raise DgError(DG_ERR_INVALID, "nccl_id must be 128 bytes")
    idbuf = ctypes.create_string_buffer(nccl_id, 128)
    h = ctypes.c_void_p()
    _check(load().dg_setup_dist(ctypes.byref(m), k, quad, rank, nranks, idbuf, ctypes.byref(h)))
    return h.value


def dg_apply_dist(ctx: int, x, r):
    _check(load().dg_apply_dist(ctx, _ptr(x), _ptr(r)))


def dg_apply(ctx: int, x, r):
    _check(load().dg_apply(ctx, _ptr(x), _ptr(r)))


def dg_apply_planes(ctx: int, x, x_below, x_above, r, p_begin: int, p_end: int):
    _check(load().dg_apply_planes(ctx, _ptr(x), _ptr(x_below), _ptr(x_above), _ptr(r), p_begin, p_end))


def dg_apply_planes_tr(ctx: int, x, tr_below, tr_above, r, p_begin: int, p_end: int):
    _check(load().dg_apply_planes_tr(ctx, _ptr(x), _ptr(tr_below), _ptr(tr_above), _ptr(r), p_begin, p_end))


def dg_pack_halo(ctx: int, x, tr_lo, tr_hi):
    _check(load().dg_pack_halo(ctx, _ptr(x), _ptr(tr_lo), _ptr(tr_hi)))


def dg_halo_ndofs(ctx: int) -> int:
    return load().dg_halo_ndofs(ctx)


def dg_apply_jacobian(ctx: int, u0, z, r):
    _check(load().dg_apply_jacobian(ctx, _ptr(u0), _ptr(z), _ptr(r)))


def dg_apply_jacobian_planes(ctx: int, u0, z, z_below, z_above, r, p_begin: int, p_end: int):
    _check(load().dg_apply_jacobian_planes(ctx, _ptr(u0), _ptr(z), _ptr(z_below), _ptr(z_above), _ptr(r), p_begin,
                                           p_end))


def dg_apply_host(ctx: int, x_host, r_host):
    _check(load().dg_apply_host(ctx, _ptr(x_host), _ptr(r_host)))


def dg_destroy(ctx: int):
    _check(load().dg_destroy(ctx))


def dg_set_stream(ctx: int, stream: int | None):
    _check(load().dg_set_stream(ctx, stream))


def dg_local_ndofs(ctx: int) -> int:
    return load().dg_local_ndofs(ctx)


def dg_local_offset(ctx: int) -> int:
    return load().dg_local_offset(ctx)


def dg_plane_ndofs(ctx: int) -> int:
    return load().dg_plane_ndofs(ctx)


def dg_alg_flops(ctx: int) -> float:
    return load().dg_alg_flops(ctx)


def dg_alg_bytes(ctx: int) -> float:
    return load().dg_alg_bytes(ctx)


def dg_launches_per_apply(ctx: int) -> int:
    return load().dg_launches_per_apply(ctx)


def dg_kernel_name(ctx: int) -> str:
    return load().dg_kernel_name(ctx).decode()


def dg_bench_fp64(device: int = 0, iters: int = 4000):
    """(TFLOP/s, ms) of the DFMA microbenchmark."""
    tf, ms = ctypes.c_double(), ctypes.c_double()
    _check(load().dg_bench_fp64(device, iters, ctypes.byref(tf), ctypes.byref(ms)))
    return tf.value, ms.value


def dg_line_ops(k: int, penalty_scale: float, x, nb) -> np.ndarray:
    """The kernels' even/odd line algebra on the host (include/dg.h): returns [D x | D^T x + face terms |
    B^ x + neighbour terms | e0.x, d0.x, e1.x, d1.x] for one line x (n = k+1) and nb = 4 values."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    nb = np.ascontiguousarray(nb, dtype=np.float64)
    n = k + 1
    assert x.shape == (n,) and nb.shape == (4,)
    out = np.empty(3 * n + 4)
    _check(load().dg_line_ops(k, float(penalty_scale), x.ctypes.data, nb.ctypes.data, out.ctypes.data))
    return out


def dg_line_ops_axis8(penalty_scale: float, x, nb) -> np.ndarray:
    """k_axis8's line operator on the host (include/dg.h): [B^ x + neighbour terms | e0.x, d0.x, e1.x, d1.x] for
    one line x of 8 values (k = 7) and nb = 4 values."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    nb = np.ascontiguousarray(nb, dtype=np.float64)
    assert x.shape == (8,) and nb.shape == (4,)
    out = np.empty(12)
    _check(load().dg_line_ops_axis8(float(penalty_scale), x.ctypes.data, nb.ctypes.data, out.ctypes.data))
    return out


def dg_last_error() -> str:
    return load().dg_last_error().decode()


# ------------------------------------------------------------------ convenience wrapper
class Operator:
    """RAII wrapper: one context (whole mesh or one x0-slab) and tensor-checked applies."""

    def __init__(self, N, k: int, *, geom_kind: int = 0, coeff_kind: int = 0, penalty_scale: float = 10.0,
                 jac: np.ndarray | None = None, plane_begin: int = 0, nplanes: int | None = None, device: int = 0,
                 stream=None, quad: int | None = None, problem: int = 0, basis: int = 0):
        import torch
        self.N = tuple(int(v) for v in N)
        self.k = k
        self.n = k + 1
        if stream is None:
            stream = torch.cuda.current_stream(device)
        self._stream = stream
        self.ctx = dg_setup(self.N, k, k + 1 if quad is None else quad, plane_begin=plane_begin, nplanes=nplanes,
                            geom_kind=geom_kind, jac=jac, coeff_kind=coeff_kind, penalty_scale=penalty_scale,
                            device=device, stream=stream.cuda_stream, problem=problem, basis=basis)
        self.ndofs = dg_local_ndofs(self.ctx)
        self.offset = dg_local_offset(self.ctx)
        self.plane_ndofs = dg_plane_ndofs(self.ctx)
        self.halo_ndofs = dg_halo_ndofs(self.ctx)
        self.nplanes = self.ndofs // self.plane_ndofs

    def _chk(self, t, n=None):
        import torch
        if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
            raise DgError(DG_ERR_INVALID, "expected a contiguous float64 CUDA tensor")
        if t.numel() != (self.ndofs if n is None else n):
            raise DgError(DG_ERR_INVALID, f"expected {self.ndofs if n is None else n} entries, got {t.numel()}")

    def set_stream(self, stream):
        self._stream = stream
        dg_set_stream(self.ctx, stream.cuda_stream)

    def apply(self, x, r=None):
        import torch
        self._chk(x)
        if r is None:
            r = torch.empty_like(x)
        self._chk(r)
        dg_apply(self.ctx, x, r)
        return r

    def apply_jacobian(self, u0, z, r=None):
        """r = J(u0) z (DG_PROBLEM_NLREAC contexts; include/dg.h dg_apply_jacobian)."""
        import torch
        self._chk(u0)
        self._chk(z)
        if r is None:
            r = torch.empty_like(z)
        self._chk(r)
        dg_apply_jacobian(self.ctx, u0, z, r)
        return r

    def apply_jacobian_planes(self, u0, z, z_below, z_above, r, p_begin: int, p_end: int):
        self._chk(u0)
        self._chk(z)
        self._chk(r)
        self._chk(z_below, self.plane_ndofs)
        self._chk(z_above, self.plane_ndofs)
        dg_apply_jacobian_planes(self.ctx, u0, z, z_below, z_above, r, p_begin, p_end)
        return r

    def apply_planes(self, x, x_below, x_above, r, p_begin: int, p_end: int):
        self._chk(x)
        self._chk(r)
        self._chk(x_below, self.plane_ndofs)
        self._chk(x_above, self.plane_ndofs)
        dg_apply_planes(self.ctx, x, x_below, x_above, r, p_begin, p_end)
        return r

    def apply_planes_tr(self, x, tr_below, tr_above, r, p_begin: int, p_end: int):
        """dg_apply_planes with trace halos (include/dg.h)."""
        self._chk(x)
        self._chk(r)
        self._chk(tr_below, self.halo_ndofs)
        self._chk(tr_above, self.halo_ndofs)
        dg_apply_planes_tr(self.ctx, x, tr_below, tr_above, r, p_begin, p_end)
        return r

    def pack_halo(self, x, tr_lo, tr_hi):
        """The slab's boundary traces for the neighbours (dg_pack_halo)."""
        self._chk(x)
        self._chk(tr_lo, self.halo_ndofs)
        self._chk(tr_hi, self.halo_ndofs)
        dg_pack_halo(self.ctx, x, tr_lo, tr_hi)
        return tr_lo, tr_hi

    def apply_host(self, x_host, r_host):
        import torch
        for t in (x_host, r_host):
            if (t.is_cuda or t.dtype != torch.float64 or t.numel() != self.ndofs or not t.is_contiguous()
                    or t.data_ptr() % 16):
                raise DgError(DG_ERR_INVALID, "expected contiguous 16-B aligned float64 host tensors of local_ndofs entries")
        dg_apply_host(self.ctx, x_host, r_host)
        return r_host

    @property
    def alg_flops(self) -> float:
        return dg_alg_flops(self.ctx)

    @property
    def alg_bytes(self) -> float:
        return dg_alg_bytes(self.ctx)

    @property
    def kernel_name(self) -> str:
        return dg_kernel_name(self.ctx)

    @property
    def launches_per_apply(self) -> int:
        return dg_launches_per_apply(self.ctx)

    def close(self):
        if getattr(self, "ctx", None):
            dg_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DistOperator(Operator):
    """The collective form (dg_setup_dist / dg_apply_dist): this rank's x0-slab, the halo exchange done by libdg's own
    NCCL communicator. Every rank constructs it with the same nccl_id and calls apply in the same order."""

    def __init__(self, N, k: int, rank: int, nranks: int, nccl_id: bytes, *, geom_kind: int = 0, coeff_kind: int = 0,
                 penalty_scale: float = 10.0, jac: np.ndarray | None = None, device: int = 0, stream=None,
                 quad: int | None = None, problem: int = 0, basis: int = 0):
        import torch
        self.N = tuple(int(v) for v in N)
        self.k = k
        self.n = k + 1
        if stream is None:
            stream = torch.cuda.current_stream(device)
        self._stream = stream
        self.rank, self.nranks = rank, nranks
        self.ctx = dg_setup_dist(self.N, k, k + 1 if quad is None else quad, rank, nranks, nccl_id,
                                 geom_kind=geom_kind, jac=jac, coeff_kind=coeff_kind, penalty_scale=penalty_scale,
                                 device=device, stream=stream.cuda_stream, problem=problem, basis=basis)
        self.ndofs = dg_local_ndofs(self.ctx)
        self.offset = dg_local_offset(self.ctx)
        self.plane_ndofs = dg_plane_ndofs(self.ctx)
        self.halo_ndofs = dg_halo_ndofs(self.ctx)
        self.nplanes = self.ndofs // self.plane_ndofs

    def apply(self, x, r=None):
        import torch
        self._chk(x)
        if r is None:
            r = torch.empty_like(x)
        self._chk(r)
        dg_apply_dist(self.ctx, x, r)
        return r
