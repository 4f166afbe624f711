/*
 * pmg_b200.h — C-ABI of the B200-native vertex-patch multigrid hot path.
 *
 * Drop-in boundary for the reference library `pmg` (/root/reference/proj).
 * Every entry point below replaces one reference function; the citation is the
 * reference declaration it stands in for. Plain C types only: opaque handles,
 * device or host pointers, int64 sizes, a cudaStream_t passed as void*.
 * No exceptions cross this boundary; every call returns a pmg_status.
 *
 * Vectors use the reference layout unchanged (mesh.cpp:42-57): a flat array of
 * N = m^d values of the level's interior nodes, lexicographic with direction 0
 * fastest, homogeneous Dirichlet nodes eliminated. T is double (PMG_F64) or
 * float (PMG_F32), fixed per context like the reference's explicit
 * instantiations (smoother.cpp:153-158, multigrid.cpp:46-51).
 *
 * Device-pointer entry points enqueue on `stream` and return without
 * synchronising. *_host entry points take host pointers and are synchronous
 * (H2D, compute, D2H) — the reference's std::span calling convention.
 */
#ifndef PMG_B200_H
#define PMG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum
{
  PMG_OK = 0,
  PMG_ERR_INVALID = 1,    /* std::invalid_argument in the reference        */
  PMG_ERR_RUNTIME = 2,    /* std::runtime_error / std::logic_error          */
  PMG_ERR_DIVERGENCE = 3, /* pmg::DivergenceError (multigrid.hpp:22-29)     */
  PMG_ERR_CUDA = 4        /* CUDA launch / allocation failure               */
} pmg_status;

typedef enum
{
  PMG_F64 = 0,
  PMG_F32 = 1
} pmg_dtype;

/* SmootherVariant, smoother.hpp:21-27 (same numbering). */
typedef enum
{
  PMG_GLOBAL = 0,
  PMG_SEPARATE = 1,
  PMG_FUSED = 2,
  PMG_BOUNDARY = 3,
  PMG_NAIVE = 100 /* straightforward global-memory fused kernel (the "≥2×"
                     comparator of the north star); same result as FUSED */
} pmg_variant;

typedef struct pmg_level_s *pmg_level; /* ~ LevelContext<T>     (level_context.hpp:17-26) */
typedef struct pmg_mg_s *pmg_mg;       /* ~ MultigridContext<T> (multigrid.hpp:34-49)     */

/* Last error message of the calling thread (static storage, never NULL). */
const char *pmg_last_error(void);

/* Library / device facts used by the bench and the tests. */
int pmg_version(void);
int pmg_device_info(int device, int *sm_count, int *sm_clock_khz, int *cc_major,
                    int *cc_minor);

/* ---- level context ------------------------------------------------------
 * ~ make_level_context<T>(build_hierarchy(dim, degree, level).back())
 *   (level_context.cpp:9-36, mesh.cpp:12-40). Setup (1D matrices, generalized
 *   eigenpairs, prolongation matrix) runs on the host in f64, is cast to T
 *   and uploaded once. */
int pmg_level_create(int dim, int degree, int level, int dtype, int device, pmg_level *out);
int pmg_level_destroy(pmg_level h);
/* m (dofs per dim), N (total dofs), patches (n-1)^d */
int pmg_level_info(pmg_level h, int64_t *dofs_per_dim, int64_t *total_dofs,
                   int64_t *patches);

/* ~ smooth<T>(ctx, x, b, variant, threads, ws)   smoother.hpp:45-47
 *   One colourised multiplicative vertex-patch step, colours in ascending
 *   parity code; x updated in place. */
int pmg_smooth(pmg_level h, int variant, void *x, const void *b, void *stream);
int pmg_smooth_host(pmg_level h, int variant, void *x, const void *b);

/* One colour of the step only (for the multi-GPU slab driver and tests). */
int pmg_smooth_color(pmg_level h, int variant, int color, void *x, const void *b,
                     void *stream);

/* One colour restricted to a slab of a (possibly stacked) 3D box, for the
 * multi-GPU domain decomposition (paper_2405_19004_b200/dd.py): the box has
 * the level's n cells along x, y and nz_cells along z; only patches whose
 * vertex z-coordinate lies in [vz_lo, vz_hi] are smoothed; x_local / b_local
 * hold the global dof planes z >= z_offset (m*m values per plane). fused or
 * boundary variant. */
int pmg_smooth_color_slab(pmg_level h, int variant, int color, void *x_local,
                          const void *b_local, int64_t z_offset, int64_t nz_cells, int vz_lo,
                          int vz_hi, void *stream);

/* ~ apply_laplacian<T>(level, cell_mass, cell_stiffness, x, y, mode, threads)
 *   operator.hpp:47-50 — y = A_l x. */
int pmg_apply_laplacian(pmg_level h, const void *x, void *y, void *stream);
int pmg_apply_laplacian_host(pmg_level h, const void *x, void *y);

/* ~ compute_residual<T>(lev, x, b, r, threads)   multigrid.hpp:90-92 */
int pmg_compute_residual(pmg_level h, const void *x, const void *b, void *r, void *stream);
int pmg_compute_residual_host(pmg_level h, const void *x, const void *b, void *r);

/* ~ prolongate<T>(coarse, fine, x_coarse, x_fine)   multigrid.hpp:56-58
 *   (accumulate != 0 gives x_fine += P x_coarse, the V-cycle's correction) */
int pmg_prolongate(pmg_level coarse, pmg_level fine, const void *xc, void *xf, int accumulate,
                   void *stream);
int pmg_prolongate_host(pmg_level coarse, pmg_level fine, const void *xc, void *xf);

/* ~ restrict_vector<T>(coarse, fine, r_fine, r_coarse)   multigrid.hpp:61-63 */
int pmg_restrict_vector(pmg_level coarse, pmg_level fine, const void *rf, void *rc,
                        void *stream);
int pmg_restrict_vector_host(pmg_level coarse, pmg_level fine, const void *rf, void *rc);

/* ~ vector_norm(v)   multigrid.hpp:89 — deterministic two-pass reduction in
 *   f64 (also for f32 vectors); synchronises `stream`. */
int pmg_vector_norm(pmg_level h, const void *v, double *out, void *stream);
/* Same for an arbitrary device vector of n entries of `dtype` on `device`. */
int pmg_norm2(const void *v, int64_t n, int dtype, int device, double *out, void *stream);

/* ---- multigrid context --------------------------------------------------
 * ~ make_multigrid_context<T>(dim, degree, finest_level, variant, kind,
 *   threads)   multigrid.hpp:51-54 (kind = vertex_patch). */
int pmg_mg_create(int dim, int degree, int finest_level, int dtype, int variant, int device,
                  pmg_mg *out);
/* SmootherKind, multigrid.hpp:16-20 (same numbering). */
enum
{
  PMG_VERTEX_PATCH = 0,
  PMG_POINT_GS = 1
};
/* ~ make_multigrid_context<T>(dim, degree, finest_level, variant, kind,
 *   threads)   multigrid.hpp:51-54 with the smoother kind: PMG_POINT_GS makes
 *   the V-cycle smooth with one lexicographic point Gauss-Seidel sweep
 *   (multigrid.cpp:286-300; f64 only -> PMG_ERR_INVALID; a level beyond the
 *   reference's 1e7-nonzero CSR budget -> PMG_ERR_RUNTIME, operator.cpp:209-227).
 *   The coarse solve stays the patch smoother's exact step, as in the reference. */
int pmg_mg_create_kind(int dim, int degree, int finest_level, int dtype, int variant, int kind,
                       int device, pmg_mg *out);
int pmg_mg_destroy(pmg_mg h);
int pmg_mg_num_levels(pmg_mg h);
pmg_level pmg_mg_level(pmg_mg h, int li); /* borrowed; index 0 = mesh level 1 */
int pmg_mg_set_smoothing(pmg_mg h, int pre_smooth, int post_smooth);
int pmg_mg_set_variant(pmg_mg h, int variant);

/* ~ v_cycle<T>(ctx, li, x, b)   multigrid.hpp:68-69. use_graph != 0 replays a
 *   CUDA graph of the whole cycle (captured on first use for this (li, x, b)). */
int pmg_v_cycle(pmg_mg h, int li, void *x, const void *b, int use_graph, void *stream);
int pmg_v_cycle_host(pmg_mg h, int li, void *x, const void *b);

/* ~ full_multigrid(ctx, rhs_per_level, x, tol, max_iterations)
 *   multigrid.hpp:80-86 (f64 contexts only, like the reference). rhs[li] are
 *   device pointers, one per level; x (device) receives the solution.
 *   history (capacity history_cap) receives ||b|| then ||r|| per V-cycle.
 *   Returns PMG_ERR_DIVERGENCE after max_iterations, like DivergenceError. */
int pmg_full_multigrid(pmg_mg h, const void *const *rhs_per_level, void *x, double tol,
                       int max_iterations, int *iterations, double *history, int history_cap,
                       void *stream);

/* Host-vector forms (the reference's std::span calls): rhs_host[li] and x
 * are host arrays; x receives the solution. */
int pmg_full_multigrid_host(pmg_mg h, const double *const *rhs_host, double *x, double tol,
                            int max_iterations, int *iterations, double *history,
                            int history_cap);
/* ~ vector_norm(v)   multigrid.hpp:89 on a host vector (reduced on the device). */
int pmg_vector_norm_host(const void *v, int64_t n, int dtype, int device, double *out);

/* ~ compute_rhs(level, f)   operator.hpp:58-59, for f = 1 (kind 0) and
 *   f = d pi^2 prod sin(pi x_a) (kind 1); host output in f64. */
int pmg_compute_rhs_host(int dim, int degree, int level, int kind, double *out);
/* ~ l2_error(level, x, u)   operator.hpp:62-64 for u = prod sin(pi x_a). */
int pmg_l2_error_sin_host(int dim, int degree, int level, const double *x, double *out);

/* Device versions (same kinds / quadrature; no reference counterpart on the
 * device): b (device, the level's dtype, N entries) = compute_rhs of the
 * level, formed as the tensor power of the 1D load vector (exact on the
 * uniform level); l2_error evaluates u_h - u pointwise at the (k+2)^d Gauss
 * points of every cell (x: device, the level's dtype). */
int pmg_compute_rhs(pmg_level h, int kind, void *b, void *stream);
int pmg_l2_error_sin(pmg_level h, const void *x, double *out, void *stream);

/* ~ point_gauss_seidel(a, x, b)   smoother.hpp / smoother.cpp:160-166 with
 *   a = assemble_sparse(level): one forward lexicographic Gauss-Seidel sweep
 *   (sparse.cpp:31-47) of an f64 level, x in place. The device sweep uses the
 *   Kronecker-sum structure of the level operator (no CSR) and the reference's
 *   row order exactly (wavefronts of independent rows, csrc/gs.cu). */
int pmg_point_gauss_seidel(pmg_level h, void *x, const void *b, void *stream);
int pmg_point_gauss_seidel_host(pmg_level h, double *x, const double *b);
/* ~ assemble_sparse(level)   operator.hpp / operator.cpp:194-281: the CSR
 *   matrix of the level operator, rows and columns in the reference's order.
 *   Host only. With row_ptr = cols = vals = NULL only *nnz is set; otherwise
 *   the arrays hold N + 1, nnz and nnz entries. */
int pmg_assemble_sparse_host(int dim, int degree, int level, int64_t *row_ptr, int32_t *cols,
                             double *vals, int64_t *nnz);

/* General fields (compute_rhs / l2_error with any ScalarField,
 * operator.hpp:55-64): the caller evaluates f (or u_exact) at the reference's
 * quadrature points — (k+2)^d Gauss points per cell, pmg_quadrature_rule
 * gives the k+2 points / weights on [0,1] — into a DEVICE array
 * fq[cell * (k+2)^d + q] (cells and q lexicographic, direction 0 fastest;
 * the point of (cell c, q) is x_a = (c_a + xi_{q_a}) h, h = 2^-level), f64.
 * pmg_compute_rhs_q: b (device, the level's dtype) = the reference's b_i =
 * sum over cells of (w f) against phi_i; pmg_l2_error_q: ||u_h - u||_L2 with
 * the same rule (synchronises `stream`). */
int pmg_quadrature_rule(int degree, double *points, double *weights);
int pmg_compute_rhs_q(pmg_level h, const double *fq, void *b, void *stream);
int pmg_l2_error_q(pmg_level h, const void *x, const double *uq, double *out, void *stream);

/* ---- mixed precision / Krylov (krylov.hpp:30-39) -------------------------
 * Right-preconditioned GMRES(restart) in f64 on the device with the V-cycle
 * of `prec` (an f32 context: mixed precision; an f64 context: double) as the
 * preconditioner; operator = f64 level operator of `op`'s finest level. */
int pmg_gmres(pmg_mg op, pmg_mg prec, const void *b, void *x, double tol, int restart,
              int max_iterations, int *iterations, double *history, int history_cap,
              void *stream);

/* ~ gmres(apply_A, apply_P, b, x, tol, restart, max_iterations)   krylov.hpp:30-39
 *   with host vectors b, x (x: initial guess in, solution out). */
int pmg_gmres_host(pmg_mg op, pmg_mg prec, const double *b, double *x, double tol, int restart,
                   int max_iterations, int *iterations, double *history, int history_cap);

/* ---- raw kernels (tests / bench) ----------------------------------------- */
/* Setup data of a level as uploaded (f64 copies), for parity tests:
 * S (ni*ni row-major), lambda (ni), mass_if, stiff_if (ni*nc), prolongation
 * ((2k+1)*(k+1)), cell mass/stiffness ((k+1)^2). Any pointer may be NULL. */
int pmg_level_setup_data(pmg_level h, double *S, double *lambda, double *mass_if,
                         double *stiff_if, double *prolongation, double *cell_mass,
                         double *cell_stiffness);

/* Host-only, no device needed: the f64 setup of one level exactly as the
 * library computes it (~ make_level_context, level_context.cpp:9-36, plus the
 * derived band / even-odd data). Any pointer may be NULL. Sizes: S, ni*ni;
 * lambda, ni; mass_if / stiff_if, ni*nc; prolongation, nc*(k+1); cell_*,
 * (k+1)^2; band_*, k*(2k+1); eo_perm, ni (ni = 2k-1, nc = 2k+1). */
int pmg_host_level_setup(int dim, int degree, int level, double *S, double *lambda,
                         double *mass_if, double *stiff_if, double *prolongation,
                         double *cell_mass, double *cell_stiffness, double *band_mass,
                         double *band_stiff, int *eo_perm);

/* Slab domain decomposition (3D, along direction 2; paper_2405_19004_b200/dd.py).
 * Device arrays hold the GLOBAL dof planes [zoff, zoff + nplanes) of a level
 * vector (m*m words per plane, the reference layout otherwise). Each call
 * computes only the requested global output planes and fails with
 * PMG_ERR_INVALID if the slab does not hold the planes they depend on. Every
 * output value is computed exactly as by the full-domain call, so slabs
 * reproduce the single-GPU V-cycle bitwise.
 *   residual r = b - A x on planes [p0, p1)            (multigrid.cpp:268-276)
 *   restriction to coarse planes [q0, q1)              (multigrid.cpp:162-248)
 *   prolongation (accumulate != 0: +=) on fine [f0, f1) (multigrid.cpp:71-160) */
int pmg_compute_residual_slab(pmg_level h, const void *x, const void *b, void *r, int64_t zoff, int64_t nplanes,
                              int64_t p0, int64_t p1, void *stream);
int pmg_restrict_slab(pmg_level coarse, pmg_level fine, const void *rf, int64_t zoff_f, int64_t np_f, void *rc,
                      int64_t zoff_c, int64_t np_c, int64_t q0, int64_t q1, void *stream);
int pmg_prolongate_slab(pmg_level coarse, pmg_level fine, const void *xc, int64_t zoff_c, int64_t np_c, void *xf,
                        int64_t zoff_f, int64_t np_f, int64_t f0, int64_t f1, int accumulate, void *stream);

/* ---- multi-GPU: slab domain decomposition behind the C-ABI ----------------
 * ~ make_multigrid_context / smooth / v_cycle / full_multigrid
 *   (multigrid.hpp:51-86, smoother.hpp:45-47) on `world` ranks, one device
 *   per rank. 3D only (dim must be 3 when world > 1). Rank g owns a
 *   contiguous range of patch-vertex planes along z:
 *   per colour one one-directional k-plane message per interface, posted after
 *   the boundary-layer patches and overlapped with the interior ones; the
 *   V-cycle adds one halo exchange per residual / restriction / coarse
 *   correction, and levels too thin to split are agglomerated on rank 0
 *   (coarse right-hand side gathered, coarse V-cycle as one CUDA graph,
 *   correction broadcast). Colour order and per-patch arithmetic are those of
 *   one device, so smoother and V-cycle results equal the single-device ones
 *   bitwise; norms are all-reduced (rank-ordered partial sums).
 *
 * Transports: PMG_DD_COPY — all ranks in this process, plane messages as
 *   device-to-device / peer copies (cudaMemcpyPeerAsync, NVLink when the
 *   devices are peers); device ids may repeat ("virtual ranks" on one GPU).
 *   PMG_DD_NCCL — grouped ncclSend/ncclRecv, ncclBroadcast, ncclAllReduce
 *   (libnccl.so.2 loaded at first use): pmg_dd_create with distinct devices
 *   (ncclCommInitAll), or pmg_dd_create_rank in one process per GPU
 *   (ncclCommInitRank with the id rank 0 got from pmg_dd_nccl_id).
 *
 * stack > 1 builds a box of `stack` unit cubes along z (weak scaling: one
 * cube per rank); only pmg_dd_smooth is defined on such a box.
 * Vectors: the handle owns x and b of the finest level, as per-rank slabs of
 * GLOBAL dof planes [z0, z0 + nplanes) (m*m values per plane, the reference
 * layout otherwise); a rank owns planes [own_lo, own_hi]. Operations enqueue
 * on the ranks' streams (pmg_dd_stream) and return; pmg_dd_synchronize waits. */
typedef struct pmg_dd_s *pmg_dd;
enum
{
  PMG_DD_COPY = 0,
  PMG_DD_NCCL = 1
};
enum
{
  PMG_DD_X = 0,
  PMG_DD_B = 1
};
int pmg_dd_create(int ndev, const int *devices, int dim, int degree, int finest_level, int stack,
                  int dtype, int variant, int transport, pmg_dd *out);
/* NCCL unique id (NCCL_UNIQUE_ID_BYTES = 128 bytes), made once on rank 0 and
 * shared with the other processes by the caller. */
int pmg_dd_nccl_id(void *id_out);
int pmg_dd_create_rank(int world, int rank, int device, const void *nccl_id, int dim, int degree,
                       int finest_level, int stack, int dtype, int variant, pmg_dd *out);
int pmg_dd_destroy(pmg_dd h);
/* world size, ranks held by this process, number of decomposed levels
 * (finest first; 0 = every level is agglomerated on rank 0). */
int pmg_dd_info(pmg_dd h, int *world, int *local_ranks, int *decomposed_levels);
/* Local rank i's slab of the finest-level vector `which` (PMG_DD_X / _B). */
int pmg_dd_slab(pmg_dd h, int local, int which, void **ptr, int64_t *z0, int64_t *nplanes,
                int64_t *own_lo, int64_t *own_hi);
/* The compute stream of local rank i (cudaStream_t) and its global rank. */
int pmg_dd_stream(pmg_dd h, int local, void **stream, int *rank);
/* Global host vector (N = m*m*mz values) <-> the local ranks' slabs:
 * scatter fills each slab completely, gather writes the owned planes. */
int pmg_dd_scatter_host(pmg_dd h, int which, const void *global);
int pmg_dd_gather_host(pmg_dd h, int which, void *global);
int pmg_dd_set_smoothing(pmg_dd h, int pre_smooth, int post_smooth);
/* One smoothing step of the finest level (x in place). With
 * pmg_dd_set_graph(h, 1) (all local ranks on one device: virtual ranks, or
 * one process per GPU) the step is captured once as a CUDA graph (launches,
 * events, plane copies / NCCL calls) and replayed on the first local rank's
 * stream. */
int pmg_dd_smooth(pmg_dd h);
int pmg_dd_set_graph(pmg_dd h, int enable);
/* One V-cycle from the finest level (x in place, b right-hand side). */
int pmg_dd_v_cycle(pmg_dd h);
/* ||b - A x|| of the finest level (all-reduced; synchronises). */
int pmg_dd_residual_norm(pmg_dd h, double *out);
/* ~ full_multigrid (multigrid.cpp:355-400), f64 only: rhs_host[li] is the
 * global host right-hand side of level index li (li = 0 .. finest-1; every
 * process passes all of them); the solution is left in the x slabs. */
int pmg_dd_full_multigrid(pmg_dd h, const double *const *rhs_host, double tol, int max_iterations,
                          int *iterations, double *history, int history_cap);
int pmg_dd_synchronize(pmg_dd h);
/* Host-only: the decomposition plan of one rank (owned vertex / dof planes,
 * whether the level is split, the per-colour boundary-layer planes and plane
 * messages), for tests and tools; see csrc/dd.cu. Returns the number of
 * int64 written, or minus a pmg_status. */
int64_t pmg_dd_plan(int world, int rank, int degree, int level, int stack, int64_t *out, int64_t cap);

/* Number of kernel launches issued by this library since load (counter). */
int64_t pmg_launch_count(void);

/* Smoother kernel organisation for subsequent calls (process-wide; no
 * reference counterpart, the reference has one CPU loop): 0 = per-degree
 * default, 1 = line-per-thread kernel everywhere, 2 = plane-streaming kernel
 * where it exists (3D, degree <= 2, fused / boundary) with one launch per
 * colour (the default for degree 2), 3 = the same with all colours of a step
 * in one persistent launch, 4 = one thread per patch (3D degree 2). Results agree to rounding (2 and 3 bitwise);
 * used for A/B measurement. Returns PMG_ERR_INVALID otherwise. */
int pmg_set_smoother_impl(int impl);
int pmg_get_smoother_impl(void);

/* Kernel organisation a colour launch of pmg_smooth runs on this level under
 * the current implementation choice (introspection for the parity tests and
 * the bench's roofline label): writes one of PMG_KERNEL_* to *kernel. */
enum
{
  PMG_KERNEL_LINE = 0,    /* vp_smooth_kernel: seven 1D line stages, in place */
  PMG_KERNEL_POINT = 1,   /* vp_point_kernel: degree 1, 3^d-point stencil */
  PMG_KERNEL_PATCH2D = 2, /* vp_patch2d_kernel: 2D, one thread per patch */
  PMG_KERNEL_PATCH3D = 3, /* vp_patch3d_kernel: 3D degree 2, one thread per patch */
  PMG_KERNEL_PLANE = 4,   /* vp_smooth_plane_kernel: 3D degree <= 2, plane streaming */
  PMG_KERNEL_PP = 5,      /* vp_smooth_pp_kernel: 3D, ping-pong conflict-free layouts */
  PMG_KERNEL_NAIVE = 6    /* naive_smooth_kernel: the straightforward comparator */
};
int pmg_smoother_kernel(pmg_level h, int variant, int color, int *kernel);

#ifdef __cplusplus
}
#endif

#endif /* PMG_B200_H */
