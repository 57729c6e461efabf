/*
 * dg.h — C-ABI of libdg: matrix-free application of the symmetric interior penalty DG
 * operator (SIPG, theta = -1) for -div(c grad u) on a structured periodic hexahedral mesh,
 * Q_k tensor-product Lagrange elements on Gauss-Legendre nodes, evaluated with sum
 * factorisation on sm_100a (B200).
 *
 * The operation (PAPER.md = /root/reference/PAPER.md, line numbers P:Lnnn):
 *   r = A x,  (A x)_I = R_I(x) = r_h(sum_J x_J phi_J, phi_I)
 *   r_h = sum_T (c grad u, grad v)_T
 *       + sum_F [ -(n_F.{c grad u}, [v])_F - ([u], n_F.{c grad v})_F + gamma_F([u],[v])_F ]
 *                                                         Eq. diffreac_weak, theta=-1 P:L995
 *   evaluated per cell with Alg. assembly (gradients by sum factorisation,
 *   pointwise flux, transposed contractions) and per facet with the normal-direction
 *   1-point tables.
 * Readings fixed in DESIGN.md §2 (R1-R20): periodic unit cube, no boundary facets, f = 0;
 * gamma_F = penalty_scale * k (k+1) / h_d with h_d = 1/N_d (BASELINE.json configs);
 * [v] = v|T- - v|T+, T- the lower cell along the face normal d (periodic wrap: cell N_d-1 is
 * T- of the face it shares with cell 0), n_F oriented T- -> T+ (P:L765); face geometry
 * (normal, surface element, quadrature points, c_F) taken from T-.
 *
 * Data layout (all fp64):
 *   cell (i0,i1,i2), canonical id c = (i0 N1 + i1) N2 + i2   (i0 slowest => x0-slabs contiguous)
 *   DOF  g = c n^3 + j0 + n j1 + n^2 j2, n = k+1 (vec convention, j0 fastest)
 *   A context owns the x0-planes [plane_begin, plane_begin + nplanes) (a "slab"); its local
 *   vectors hold those planes' blocks contiguously (local offset = plane_begin N1 N2 n^3).
 *
 * Error behaviour: every function returns DG_OK (0) or a negative DG_ERR_* code and never
 * aborts; dg_last_error() returns a thread-local message for the last failure. No function
 * falls back to a CPU path: without a usable CUDA device dg_setup returns DG_ERR_CUDA.
 * Thread safety: a context is not thread-safe; distinct contexts are independent.
 */
#ifndef DG_H
#define DG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DG_OK 0
#define DG_ERR_INVALID (-1)     /* bad argument (sizes, pointers, aliasing, unsupported k) */
#define DG_ERR_UNSUPPORTED (-2) /* valid request this build does not implement (e.g. quad outside k+1..k+3) */
#define DG_ERR_CUDA (-3)        /* CUDA runtime failure (no device, launch error, ...) */
#define DG_ERR_NCCL (-4)        /* NCCL unavailable or failed (collective entry points only) */
#define DG_ERR_OOM (-5)         /* device or pinned-host allocation failed */

#define DG_GEOM_AXIS 0   /* J_T = diag(1/N0, 1/N1, 1/N2) */
#define DG_GEOM_AFFINE 1 /* per-cell affine map x = o_T + J_T xi, J_T given per cell */
#define DG_COEFF_ONE 0   /* c = 1 (Poisson) */
#define DG_COEFF_SINCOS 1 /* c(x) = 1 + 0.5 sin(2 pi x0) cos(2 pi x1), at the mapped quadrature points */

#define DG_PROBLEM_PERIODIC 0 /* the configs: periodic cube, -div(c grad u), f = 0: r = A x */
#define DG_PROBLEM_DIFFREAC 1 /* the paper's problem: non-periodic (0,1)^3,
                                 -div(K grad u) + 10 u = -6, K = x x^T + I, u = |x|^2 on the boundary;
                                 r = R(x) = A x - b (Eq. diffreac_weak incl. the f and g terms); axiparallel
                                 (DG_GEOM_AXIS) only, coeff_kind ignored, quad = k+2 (k_quad);
                                 gamma_F = penalty_scale k (k+2) |F| / |T| (the paper: penalty_scale = alpha = 3) */
#define DG_PROBLEM_STOKES 3   /* the paper's Stokes problem (Eq. stokes_weak; DESIGN.md
                                 R27/R28): (0,1)^3, mu = 1, f = 0, Dirichlet g = (4 x_1 (1 - x_1), 0, 0) on the
                                 boundary without the face x_0 = 1 (Neumann there); velocity Q_k, pressure
                                 Q_{k-1}; per cell 3 n^3 + k^3 DOFs [u_0 | u_1 | u_2 | p] (every dg_local_ndofs /
                                 dg_plane_ndofs count uses this block); r = R(x) incl. the g terms; DG_GEOM_AXIS,
                                 DG_COEFF_ONE, quad = k+1 (k_stokes); gamma_F as DG_PROBLEM_DIFFREAC */
#define DG_PROBLEM_NLREAC 2   /* its nonlinear variant (reading R26): reaction 10 u^2 in
                                 place of 10 u, f = 10|x|^4 - 10|x|^2 - 6 (u = |x|^2 stays the exact solution),
                                 K, g, penalty, restrictions as DG_PROBLEM_DIFFREAC; dg_apply returns the
                                 nonlinear residual R(x), dg_apply_jacobian* the action J(u0) z of its Jacobian */

#define DG_BASIS_GAUSS 0   /* Lagrange basis on the n = k+1 Gauss-Legendre nodes (reading R8; the configs): collocated
                              with the k+1-point rule, A = I */
#define DG_BASIS_LOBATTO 1 /* Lagrange basis on the n Gauss-Lobatto nodes (the non-Gauss basis):
                              A^(i) = [l_j(xi_q)] != I at every Gauss rule, so stage 1 / 3 need the full sum
                              factorisation (Eq. lowcomplex); DG_PROBLEM_PERIODIC only, any
                              geometry / coefficient, quad = k+1 .. k+3 (k_quad); DOF j of a line is the value at the
                              j-th Gauss-Lobatto node */
#define DG_BASIS_EQUIDISTANT 2 /* Lagrange basis on the n equidistant nodes j / k (SPEC.md's CPU program); as
                              DG_BASIS_LOBATTO otherwise */

typedef struct dg_ctx dg_ctx;

typedef struct dg_mesh {
    int32_t N[3];          /* global cells per direction; the unit cube is periodic in all three; N[d] >= 2 */
    int32_t plane_begin;   /* first global x0-plane owned by this context, 0 <= plane_begin < N[0] */
    int32_t nplanes;       /* number of owned x0-planes L, 1 <= L <= N[0] (L == N[0]: whole mesh) */
    int32_t geom_kind;     /* DG_GEOM_AXIS or DG_GEOM_AFFINE */
    const double* jac;     /* HOST pointer, read during dg_setup only (caller keeps ownership).
                              DG_GEOM_AFFINE: row-major 3x3 J_T (9 doubles) for every cell of the
                              L+2 x0-planes plane_begin-1 .. plane_begin+L (global indices mod N0),
                              each plane in canonical (i1, i2) order. det J_T must be nonzero.
                              DG_GEOM_AXIS: must be NULL. */
    int32_t coeff_kind;    /* DG_COEFF_ONE or DG_COEFF_SINCOS */
    double penalty_scale;  /* gamma_F = penalty_scale * k (k+1) * N[d] on faces with normal d (> 0) */
    int32_t device;        /* CUDA device ordinal */
    void* stream;          /* cudaStream_t on which dg_apply* enqueue work (NULL: legacy default stream) */
    int32_t problem;       /* DG_PROBLEM_PERIODIC (default, 0), _DIFFREAC, _NLREAC or _STOKES */
    int32_t basis;         /* DG_BASIS_GAUSS (default, 0), DG_BASIS_LOBATTO or DG_BASIS_EQUIDISTANT */
} dg_mesh;

/* Create a context: 1D tables (Gauss-Legendre nodes/weights, Lagrange derivative matrix D,
 * boundary vectors e0,e1,d0,d1), device copy of the slab's
 * geometry, kernel selection. k in [1,7]; quad = Gauss points per direction: k+1 (collocation), k+2
 * (overintegration, A != I: k_quad), k+3 (periodic problem, k <= 6: k_quad); other values ->
 * DG_ERR_UNSUPPORTED (P:L604-616 raised quadrature counts). Allocates device memory for the L+2 planes
 * plane_begin-1 .. plane_begin+L: DG_GEOM_AFFINE: J (72 B/cell) and per-cell geometry records
 * (288 B/cell: |det J| J^-1 J^-T, rows of J, upper-face normals / surface elements);
 * DG_COEFF_SINCOS: c(x) factor tables (96 (n+1) B/cell) and c at the upper-face points
 * (8 (3n^2 rounded up to even) B/cell); DG_GEOM_AXIS + DG_COEFF_ONE: nothing. *out owned by
 * the caller, release with dg_destroy. Synchronous. Kernel selection is deterministic: k_axis8 for
 * axis-aligned Q7 with c = 1 and N1 % 2 == N2 % 4 == 0; k_line for other axis-aligned c = 1 slabs whose x
 * is at most 32 MB (L2-resident); k_gen when its (i1, i2) tile divides the mesh;
 * k_cell_general otherwise; k_quad / k_stokes for the other problems, and k_quad for the non-Gauss bases
 * (DG_BASIS_LOBATTO / DG_BASIS_EQUIDISTANT: A != I at every rule, quad = k+1 .. k+3). A failing kernel attribute
 * call or allocation returns DG_ERR_CUDA / DG_ERR_OOM (no silent switch to another kernel) and
 * releases everything allocated so far. */
int dg_setup(const dg_mesh* mesh, int k, int quad, dg_ctx** out);

/* r = A x for a context owning the WHOLE mesh (nplanes == N[0]).
 * x, r: caller-owned DEVICE pointers to dg_local_ndofs() doubles each, not overlapping (else
 * DG_ERR_INVALID). Alignment (else DG_ERR_INVALID, checked before any launch): every pointer
 * 8-byte aligned; x, r and the halo planes of dg_apply_planes 16-byte aligned when dg_kernel_name()
 * is "k_gen" or "k_axis8" (16-B vector / bulk-copy accesses; their plane sizes are multiples of
 * 16 B, so whole-mesh halos inside x qualify); x 128-byte aligned for "k_axis8" (the TMA tensor
 * map base). cudaMalloc / PyTorch allocations satisfy all of these. r is overwritten (every entry written exactly once).
 * Asynchronous on the context stream; the caller synchronises. */
int dg_apply(dg_ctx* ctx, const double* x, double* r);

/* Slab form used for x0 domain decomposition: overwrite the rows of r belonging to local
 * x0-planes [p_begin, p_end) (0 <= p_begin <= p_end <= L).
 *   x        DEVICE, the L owned planes (dg_local_ndofs() doubles)
 *   x_below  DEVICE, the DOF blocks of global plane plane_begin-1 (mod N0): N1 N2 n^3 doubles
 *            (the halo received from the lower neighbour; for a whole-mesh context this is
 *            x + (L-1) N1 N2 n^3)
 *   x_above  DEVICE, the blocks of global plane plane_begin+L (mod N0)
 *   r        DEVICE, dg_local_ndofs() doubles; rows outside [p_begin, p_end) are untouched.
 * Asynchronous on the context stream. */
int dg_apply_planes(dg_ctx* ctx, const double* x, const double* x_below, const double* x_above, double* r,
                    int p_begin, int p_end);

/* Traces-only halo exchange for the x0-slab decomposition (the "traces only" payload): the
 * face between slabs needs from the neighbour only u and d_0 u at the n^2 face points of each boundary cell
 * (the 1-point face tables e0/e1, d0/d1 of P:L143-146 applied along the d = 0 lines), 2 n^2 instead of
 * n^3 doubles per cell (cfg3: 4x less, cfg4: 2.5x less).
 * dg_halo_ndofs: doubles of one trace halo, N1 N2 2 n^2 (per cell u[n^2] then d_0 u[n^2], point j1 + n j2).
 * dg_pack_halo: from the slab's x (DEVICE, dg_local_ndofs doubles) write tr_lo = the lower-end traces (e0.x,
 *   d0.x) of the first local plane (the lower neighbour's tr_above) and tr_hi = the upper-end traces (e1.x,
 *   d1.x) of the last local plane (the upper neighbour's tr_below); DEVICE, dg_halo_ndofs doubles each, 16-byte
 *   aligned. Asynchronous on the context stream.
 * dg_apply_planes_tr: dg_apply_planes with the two halo planes replaced by trace halos as produced by the
 *   neighbours' dg_pack_halo (16-byte aligned). Interior plane ranges never read them.
 * Both return DG_ERR_UNSUPPORTED unless dg_kernel_name() is "k_gen", "k_axis8" or "k_line". */
int64_t dg_halo_ndofs(const dg_ctx* ctx);
int dg_pack_halo(dg_ctx* ctx, const double* x, double* tr_lo, double* tr_hi);
int dg_apply_planes_tr(dg_ctx* ctx, const double* x, const double* tr_below, const double* tr_above, double* r,
                       int p_begin, int p_end);

/* Collective form: the mesh split into x0-slabs over nranks processes (one GPU each),
 * rank q owning planes [q N0 / nranks, (q+1) N0 / nranks) — a contiguous range of the canonical vector, the
 * periodic wrap making the ranks a ring. The context owns an NCCL communicator (libnccl.so.2 is loaded at run
 * time); one application is ONE point-to-point exchange step (ncclSend / ncclRecv of the two boundary payloads
 * with ranks q -+ 1 on a high-priority stream) overlapped with the interior planes, then the two boundary planes.
 * Payload: the face traces of dg_pack_halo for k_gen / k_axis8 / k_line, the full boundary planes otherwise.
 * dg_slab_range: the planes of a rank (plane_begin, nplanes) — use it to fill the mesh (and its jac, L+2 planes).
 * dg_get_unique_id: a 128-byte ncclUniqueId (one rank creates it and broadcasts it by its own means).
 * dg_setup_dist: COLLECTIVE (every rank, same arguments but rank); mesh->plane_begin / nplanes must be the
 *   rank's slab. nranks = 1 is valid (the exchange is a send / receive to itself: a loopback of the same code).
 * dg_apply_dist: COLLECTIVE, every rank in the same order; x, r DEVICE, dg_local_ndofs doubles (the slab), as
 *   dg_apply. Asynchronous on the context stream (the exchange runs on the context's own comm stream).
 * DG_ERR_NCCL if NCCL is missing or fails. dg_destroy releases the communicator. */
int dg_slab_range(int N0, int rank, int nranks, int32_t* plane_begin, int32_t* nplanes);
int dg_get_unique_id(void* nccl_id_128);
int dg_setup_dist(const dg_mesh* mesh, int k, int quad, int rank, int nranks, const void* nccl_id_128, dg_ctx** out);
int dg_apply_dist(dg_ctx* ctx, const double* x, double* r);

/* The action of the Jacobian of a DG_PROBLEM_NLREAC residual at the linearization point u0
 * ("not only the solution needs to be evaluated in step 1 ... but also the given
 * linearization point"; A_i(c, z) = (J z)_i, depending on both c and z):
 *   r = J(u0) z = (K grad z, grad v) + (20 u0 z, v) + the SIPG face terms of z with g = 0.
 * u0 and z are evaluated at the quadrature points by the same sum-factorisation sweeps in one
 * kernel (k_quad mode 3). Arguments as dg_apply / dg_apply_planes (z takes x's place, z_below /
 * z_above its halo planes); u0: DEVICE, dg_local_ndofs() doubles of the owned planes only (the
 * Jacobian's u0-dependence is cell-local), 8-byte aligned, must not overlap r.
 * DG_ERR_UNSUPPORTED unless the context's problem is DG_PROBLEM_NLREAC. Asynchronous. */
int dg_apply_jacobian(dg_ctx* ctx, const double* u0, const double* z, double* r);
int dg_apply_jacobian_planes(dg_ctx* ctx, const double* u0, const double* z, const double* z_below,
                             const double* z_above, double* r, int p_begin, int p_end);

/* End-to-end form with HOST buffers (whole-mesh context): copies x host->device, applies A,
 * copies r device->host, pipelined over x0-plane chunks on three streams (H2D, compute, D2H)
 * so the PCIe transfers overlap the kernels. x_host, r_host: dg_local_ndofs() doubles
 * (page-locked memory gives full overlap; pageable memory works but serialises). Device
 * staging buffers are allocated on first use and kept in the context. Synchronous: returns
 * after r_host is complete. */
int dg_apply_host(dg_ctx* ctx, const double* x_host, double* r_host);

/* Release all device memory, streams and events of the context. NULL is accepted. */
int dg_destroy(dg_ctx* ctx);

int dg_set_stream(dg_ctx* ctx, void* stream);

int64_t dg_local_ndofs(const dg_ctx* ctx);  /* L N1 N2 n^3 */
int64_t dg_local_offset(const dg_ctx* ctx); /* plane_begin N1 N2 n^3: offset of the slab in the global vector */
int64_t dg_plane_ndofs(const dg_ctx* ctx);  /* N1 N2 n^3: size of one x0-plane (halo message) */

/* Algorithmic work of one application over the local slab:
 * flops = F_alg(n) * local DOFs, with F_alg the collocated sum-factorisation count with
 * each face once; bytes = 16 B per DOF (read x, write r) + 120 B per affine cell (J, G~). */
double dg_alg_flops(const dg_ctx* ctx);
double dg_alg_bytes(const dg_ctx* ctx);

/* Kernel launches enqueued by one dg_apply / dg_apply_planes call (dg_apply_dist: pack + interior + 2
 * boundary launches), and the name of the kernel. */
int dg_launches_per_apply(const dg_ctx* ctx);
const char* dg_kernel_name(const dg_ctx* ctx);

/* FP64 peak microbenchmark (measurement utility, not part of the operator): runs 8 independent
 * DFMA chains per thread on every SM for `iters` x 128 DFMAs per thread and returns the achieved
 * FP64 TFLOP/s (2 flops per DFMA) and the kernel time. Synchronous. */
int dg_bench_fp64(int device, int iters, double* tflops, double* ms);

/* The kernels' 1D line algebra evaluated on the HOST with the same code (no device needed; a
 * testing / inspection entry). For one line x[n], n = k+1, and four neighbour / face values
 * nb = (a, b, c, d) writes out[3n + 4]:
 *   out[0, n)     D x                                   (stage-1 sweep, D[q][j] = l_j'(xi_q))
 *   out[n, 2n)    D^T x + e0 a + d0 b + e1 c + d1 d     (stage-3 sweep with the face back-projection
 *                                                        at the two line ends)
 *   out[2n, 3n)   B^ x + aL a + bL b + aR c + bR d      (axis-aligned line operator, DESIGN.md §4.1:
 *                 B^ = D^T W D + (e0 d0^T + d0 e0^T - e1 d1^T - d1 e1^T)/2 + P (e0 e0^T + e1 e1^T),
 *                 aL = -d0/2 - P e0, bL = e0/2, aR = d1/2 - P e1, bR = -e1/2, P = penalty_scale k(k+1))
 *   out[3n, 3n+4) e0.x, d0.x, e1.x, d1.x                (face traces, 1-point tables)
 * computed in the even/odd (centro-(anti)symmetric) form the kernels use. k in [1,7]. */
int dg_line_ops(int k, double penalty_scale, const double* x, const double* nb, double* out);

/* The same for k_axis8's line operator (k = 7, n = 8; host build of kernel_axis8.cuh's algebra with the tables
 * dg_setup gives that kernel): B^ applied from the volume stiffness K = D^T W D and rank-2 trace
 * terms. For one line x[8] and nb = (a, b, c, d) writes out[12]:
 *   out[0, 8)   B^ x + aL a + bL b + aR c + bR d   (same B^, aL, bL, aR, bR as dg_line_ops, P = penalty_scale 56)
 *   out[8, 12)  e0.x, d0.x, e1.x, d1.x
 * Host pointers, caller-owned; returns DG_ERR_INVALID for NULL arguments. */
int dg_line_ops_axis8(double penalty_scale, const double* x, const double* nb, double* out);

/* Thread-local description of the last error ("" if none). */
const char* dg_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* DG_H */
