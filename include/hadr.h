/*
 * hadr.h — C ABI of the B200-native amplitude solve (libhadr.so).
 *
 * Drop-in boundary for the hot path of the reference package `helmadr`
 * (arXiv 1712.06091; /root/reference/pkg/src/helmadr).  The reference is pure
 * Python and has no FFI of its own: these entry points are what its duck-typed
 * solver API binds to through the Python shim in
 * paper_1712_06091_b200/ (ctypes).  Each function cites
 * the reference callable it replaces.
 *
 * Conventions
 *   - complex vectors are interleaved (re, im) doubles, numpy complex128 layout,
 *     flattened row-major over (n1, n2[, n3]): k = (i1*n2 + i2)*n3 + i3, the last
 *     axis (depth) fastest (helmadr/grid.py:5-9); 2D grids pass n3 = 1;
 *   - `on_device` = 0: pointers are host memory (copied in/out inside the call);
 *     `on_device` = 1: pointers are device memory on the current CUDA device;
 *   - inputs are never modified (helmadr/krylov.py:93, 138);
 *   - return 0 on success; HADR_EVALUE maps to Python ValueError,
 *     HADR_ERUNTIME / HADR_ECUDA to RuntimeError; hadr_last_error() has the text.
 *   - levels are 1-based, level 1 = finest (helmadr/multigrid.py:132).
 */
#ifndef HADR_H
#define HADR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HADR_OK 0
#define HADR_EVALUE 1
#define HADR_ERUNTIME 2
#define HADR_ECUDA 3

typedef struct hadr_op_s* hadr_op;     /* structured 2D stencil operator (device) */
typedef struct hadr_hier_s* hadr_hier; /* multigrid hierarchy + K-cycle workspace (device) */

/* Mirrors helmadr/krylov.py:34-53 SolveReport (history returned separately). */
typedef struct {
  int iterations;
  int converged;
  int note;          /* 0 = "", 1 = "numerical breakdown: non-finite Arnoldi vector" */
  int history_len;   /* entries written to the caller's history buffer */
  double bnorm;
  double final_relres;
  double wall_time;   /* seconds, host clock around the device solve */
  double device_time; /* seconds, CUDA events on the library stream around the solve */
  double ortho_max;   /* max |<v_i, v_j>| (i != j) of the Arnoldi basis over the restart cycles; computed
                         only with HADR_FG_DIAGNOSTICS (helmadr/krylov.py:214-217), else 0 */
} hadr_report;

const char* hadr_last_error(void);
int hadr_init(int device);
int hadr_device_sync(void);
int hadr_device_malloc(void** ptr, size_t bytes);
int hadr_device_free(void* ptr);
/* kind: 1 host->device, 2 device->host, 3 device->device */
int hadr_memcpy(void* dst, const void* src, size_t bytes, int kind);
/* device memset (byte value), stream-ordered and synchronised like hadr_memcpy */
int hadr_memset(void* dst, int value, size_t bytes);

/* ---- operators (helmadr/operators.py CSR matrices, as structured stencils) ---- */
/* From a canonical CSR matrix on the (n1, n2) grid; replaces the scipy CSR consumed by
 * helmadr/krylov.py:60-65 spmv and helmadr/multigrid.py:113 build_hierarchy. */
int hadr_op_from_csr(int n1, int n2, int n3, int64_t nnz, const int64_t* indptr, const int32_t* indices,
                     const double* data, hadr_op* out);
/* From coefficient planes coef[o*N + k] for offsets (d1, d2, d3) strictly ascending (2D: d3 = 0). */
int hadr_op_from_planes(int n1, int n2, int n3, int n_offsets, const int* offsets, const double* coef, hadr_op* out);
int hadr_op_info(hadr_op op, int* n1, int* n2, int* n3, int* n_offsets, int* offsets /* 3*125 */);
int hadr_op_export(hadr_op op, double* coef /* n_offsets*N complex */);
/* storage of the operator's stencil kernel: *n_slots = coefficient planes stored in the pair-compressed
 * copy (fine upwind operators: 2D 7, 3D 10) or the class-compressed copy (coarse upwind Galerkin
 * operators: the largest class present; interior rows read 2D 15, 3D 54), 0 = union planes (n_offsets).  Built lazily by the first apply /
 * solve (options "pair_compress", "class_compress"); no reference counterpart (layout only). */
int hadr_op_storage(hadr_op op, int* n_slots, long long* mixed_rows /* class-compressed rows whose class
                                                                        holds both +-2 sides of an axis */);
/* y = A x  (helmadr/krylov.py:60-65 spmv; scipy csr_matvec order, bit-exact) */
int hadr_op_apply(hadr_op op, const double* x, double* y, int on_device);
/* z = r / diag(A)  (helmadr/krylov.py:68-73 jacobi_apply) */
int hadr_op_jacobi(hadr_op op, const double* r, double* z, int on_device);
/* alpha*A + beta*B on the union pattern (helmadr/drivers.py:156 blend) */
int hadr_op_axpby(double ar, double ai, hadr_op A, double br, double bi, hadr_op B, hadr_op* out);
/* A + diag(s * field), field real (helmadr/operators.py:237-244 shift_operator) */
int hadr_op_add_diag(hadr_op A, double sr, double si, const double* field, hadr_op* out);
/* diag(left) A diag(right) (helmadr/operators.py:252-266 similarity_conjugate) */
int hadr_op_similarity(hadr_op A, const double* left, const double* right, hadr_op* out);
/* P^T A P for bilinear P (helmadr/multigrid.py:49-55 galerkin_coarsen) */
int hadr_op_galerkin(hadr_op A, hadr_op* out);
/* On-device assembly (helmadr/operators.py:190-234; 3D: the per-axis restatement):
 * scheme 0 central, 1 upwind1, 2 upwind2 ADR (assemble_adr), 3 Helmholtz (assemble_helmholtz;
 * grad/lap ignored).  dim 2 or 3; bc = (top, bottom, left, right, front, back) face kinds,
 * 0 neumann / 1 sommerfeld (front/back unused in 2D).  src = node of the point source
 * (near-source central stencil), src1 = -1 for none.  Fields are arrays of n1*n2*n3 doubles
 * (host, or device with on_device = 1); grad3 unused in 2D. */
int hadr_assemble(int dim, int n1, int n2, int n3, double h1, double h2, double h3, double omega, int scheme,
                  const int* bc, int src1, int src2, int src3, const double* kappa_sq, const double* gamma,
                  const double* grad1, const double* grad2, const double* grad3, const double* lap_tau, int on_device,
                  hadr_op* out);
/* solve_adr_upwind (helmadr/drivers.py:136-168) minus the host-side phase transforms:
 * assemble H2up, H1up, blend (1-beta)H2up + beta H1up, build the hierarchy, FGMRES on H2up
 * with the K-cycle on the blend.  qhat is the transformed source (to_adr).  *t_setup gets the
 * device time of assembly + hierarchy; rep->device_time the FGMRES time. */
int hadr_solve_adr_upwind(int dim, int n1, int n2, int n3, double h1, double h2, double h3, double omega,
                          const int* bc, int src1, int src2, int src3, const double* kappa_sq, const double* gamma,
                          const double* grad1, const double* grad2, const double* grad3, const double* lap_tau,
                          const double* qhat, double beta, int levels, int restart, int maxiter, double tol,
                          double* a_out, hadr_report* rep, double* history, int history_cap, double* t_setup,
                          int on_device);
/* release recycled hierarchies and cached device blocks */
int hadr_pool_trim(void);
void hadr_op_destroy(hadr_op op);

/* ---- transfer operators (helmadr/multigrid.py:19-46) ---- */
/* rc = P^T r (direction 0) or y = P e (direction 1) for the fine grid (n1, n2, n3); P is the
 * bilinear (2D, n3 = 1) / trilinear (3D) interpolation of helmadr/multigrid.py:19-46. */
int hadr_transfer(int n1, int n2, int n3, int direction, const double* in, double* out, int on_device);

/* ---- multigrid (helmadr/multigrid.py) ---- */
/* build_hierarchy(A0, grid, max_levels) with Galerkin coarse operators built on the device.
 * The hierarchy keeps a reference to `fine` (do not destroy it first). */
int hadr_hier_create(hadr_op fine, int max_levels, int coarse_steps, double coarse_tol, hadr_hier* out);
/* MGHierarchy(ops=...) from given per-level operators (finest first; borrowed). */
int hadr_hier_from_ops(int n_levels, const hadr_op* ops, int coarse_steps, double coarse_tol, hadr_hier* out);
int hadr_hier_info(hadr_hier h, int* n_levels, int* shapes /* 3*n_levels */);
/* borrowed handle to level `level` (1-based) operator */
int hadr_hier_level_op(hadr_hier h, int level, hadr_op* out);
/* k_cycle(hier, level, b, x) (helmadr/multigrid.py:132-171); x may be NULL (zero);
 * visits (nullable, n_levels ints) mirrors the `stats` dict */
int hadr_kcycle(hadr_hier h, int level, const double* b, const double* x, double* x_out, int* visits,
                int on_device);
/* make_kcycle_preconditioner(hier)(r) (helmadr/multigrid.py:174-184): graph-captured K-cycle */
int hadr_precond_apply(hadr_hier h, const double* r, double* z, int on_device);
void hadr_hier_destroy(hadr_hier h);
/* runtime options: "dist_min_planes" / "dist_levels" = slab levels policy (multi-GPU);
 * "ce_max_n" = levels with at most this many points run their coarse part inside
 * the single-cluster engine (default 32768; 0 = every operation is its own kernel);
 * "kcycle_c64" = 1: hierarchies built afterwards apply their operators from complex64 storage
 * (mixed precision: K-cycle operators c64, vectors / reductions / outer FGMRES c128) */
int hadr_set_option(const char* name, double value);
/* cluster-engine phase counters (enable with hadr_set_option("ce_profile", 1)): cycles seen by CTA 0,
 * 48 entries: [total, allreduce, n, relaxation control, n, stencil, n, launches, vector ops, n, barriers,
 * n, transfers, n, relaxation update, n, stencil on levels > 8192 points, n, shared-memory relaxation
 * staging (> 8192), n, its stencil rows (> 8192), n, staging (small levels), n, stencil rows (small), n,
 * all-reduce cluster-barrier wait, n, inner-FGMRES control, n, CGS2 step, n, then the CGS2 phases: dots 1, n,
 * all-reduce 1, n, update 1, n, dots 2, n, all-reduce 2, n, update 2, n, final barrier, n, 0, 0] */
int hadr_ce_profile(unsigned long long* out48, int reset);
/* Measurement hook (bench.py roofline): launch the cluster engine `reps` times back to back at
 * hierarchy level `level` (1-based, 2 <= level < n_levels) in its inner-FGMRES(2) entry — one
 * launch = the coarse part of the K-cycle from that level down (helmadr/multigrid.py:153-167)
 * on the level's current right-hand side — and return the mean launch time (CUDA events). */
int hadr_ce_bench(hadr_hier h, int level, int reps, double* avg_ms);
/* microbenchmark of the stencil kernel K1 on device vectors x, y: `reps` back-to-back launches timed
 * with CUDA events on the library stream; variant 0 = y = A x, 1 = the relaxation's fused
 * y = A(D^-1 s x) + basis write + <V0, y>, 2 = y = A x + <u, y>, 3 = the split relaxation step of large
 * 3D levels (V = s x, z = D^-1 V in one kernel, then y = A z + <u, y>).  *avg_ms = mean duration of one
 * such step (incl. any finalize). */
int hadr_op_bench(hadr_op op, const double* x, double* y, int reps, int variant, double* avg_ms);
/* number of kernels this library has launched so far (graph launches add their kernel nodes) */
long long hadr_launch_count(void);
/* CUDA-event timer on the library stream: start=1 records the start event (returns 0);
 * start=0 records the stop event, waits for it and returns the elapsed milliseconds (-1 on error) */
double hadr_stream_timer(int start);

/* ---- multi-GPU slab decomposition (the reference is single-process) ----
 * One process per GPU.  After hadr_dist_init_*, hadr_solve_adr_upwind runs collectively: every rank
 * passes the same global inputs, assembles and solves the axis-0 slab it owns (coarse levels below
 * "dist_min_planes" planes per rank are agglomerated = replicated), and receives the global amplitude. */
/* NCCL (one GPU per rank): rank 0 creates the id, the caller broadcasts its 128 bytes */
int hadr_dist_nccl_id(char* unique_id /* 128 bytes */);
int hadr_dist_init_nccl(int rank, int size, const char* unique_id);
/* Host communicator: blocking callbacks on host buffers (e.g. torch.distributed gloo); ranks may
 * share a GPU.  allgather: recv = size x nbytes in rank order; sendrecv: dst/src = -1 for none. */
typedef int (*hadr_host_allgather)(const void* send, void* recv, long long nbytes);
typedef int (*hadr_host_sendrecv)(const void* send, long long sbytes, int dst, void* recv, long long rbytes, int src);
typedef int (*hadr_host_bcast)(void* buf, long long nbytes, int root);
int hadr_dist_init_host(int rank, int size, hadr_host_allgather ag, hadr_host_sendrecv sr, hadr_host_bcast bc);
int hadr_dist_finalize(void);
/* kind: 0 none, 1 NCCL, 2 host callbacks */
int hadr_dist_info(int* rank, int* size, int* kind);
/* slab plan of a global grid under the active communicator: bounds[size + 1] fine-axis slab starts,
 * *n_dist_levels leading slab levels out of *n_levels */
int hadr_dist_plan(int n1, int n2, int n3, int max_levels, int* bounds, int* n_dist_levels, int* n_levels);
/* pure host helper: split n1 planes into `size` slabs with interior bounds multiples of `align` */
/* the slab plan hadr_dist_plan would make for `size` ranks (host logic only, no device or
 * communicator): fine slab bounds (size + 1), levels split in slabs, levels in total */
int hadr_slab_plan(int n1, int n2, int n3, int max_levels, int size, int* bounds, int* n_dist_levels, int* n_levels);
int hadr_slab_bounds(int n1, int size, int align, int* bounds /* size + 1 */);
/* pure host helper: the tiling the plane-marching stencil kernel (k_stencil_march; replaces csr_matvec on
 * large 3D fine levels, helmadr/krylov.py:60-65) uses for an owned slab of n1own x n2 x n3 points (n3 = 1:
 * 2D, marched row by row): out10 = {tiles along axis 1, tiles along axis 2, plane chunks, planes per chunk,
 * shared-memory row pitch, slot elements, halo rows, thread blocks, dynamic shared-memory bytes (jac: with
 * the D^-1 ring), points-per-tile cap}.  Tile t of n along an axis covers [t*n/nt, (t+1)*n/nt). */
int hadr_march_plan(int n1own, int n2, int n3, int jac, int* out10);

/* tau_derivatives (helmadr/eikonal.py:180-226) with AnalyticBase's distance factor
 * (helmadr/eikonal.py:15-36; 3D: the per-axis generalisation, lap(tau0) = 2/r): from tau1 on the
 * n[0] x .. x n[dim-1] grid over [0, L[a]] with the source node src[], writes tau = tau0 tau1 (may be
 * NULL), grads (dim planes of N doubles, axis-major) and lap.  Bit-identical to the reference's
 * numpy expressions (np.hypot = glibc's hypot).  on_device: every array is a device pointer. */
int hadr_tau_derivatives(int dim, const int* n, const double* L, const int* src, const double* tau1, double* tau,
                         double* grads, double* lap, int on_device);
/* out = q (.) exp(sign * i * omega * tau), sign = +1 (to_adr) / -1 (to_helmholtz): the phase transforms
 * of helmadr/operators.py:269-278 (rhs_transform) and compose_waveform (helmadr/drivers.py:171-173) on the
 * device; tau real.  cos/sin are the device's (within an ulp of numpy's). */
int hadr_phase_transform(long long n, const double* q, const double* tau, double omega, int sign, double* out,
                         int on_device);

/* ---- travel time (setup, host; the amplitude solve takes tau as an input) ----
 * Factored-eikonal fast marching (helmadr/_fmm.py:22-331 via helmadr/eikonal.py:72-99): tau = tau0 * tau1
 * with tau0 = |x - x0| and its gradient g0 (AnalyticBase), kappa = slowness; order 1 or 2.
 * Writes tau1 (N doubles); *n_accepted = N on success (fewer: disconnected / heap overflow).
 * dim 2 reproduces the reference; dim 3 is this build's extension (g03 used). No device needed. */
int hadr_fast_march(int dim, const int* n, const double* h, const double* tau0, const double* g01,
                    const double* g02, const double* g03, const double* kappa, const int* src, int order,
                    double* tau1, long long* n_accepted);

/* ---- accuracy workflow (helmadr/grid.py:175-191 relative_error_map; helmadr/drivers.py:176-196
 * accuracy_compare) ----
 * err = |u - u_ref| / max(|u_ref|, floor) over n complex points (err may be NULL); floor < 0 selects the
 * reference default 1e-12 * max|u_ref|, written back to *floor_used.  The nodes with |u_ref| >= floor are
 * the statistics mask: *count receives their number and vals[q] the idx[q]-th smallest masked error
 * (ascending order, idx clipped to [0, count-1]) for q < nidx, from which the host shim forms numpy's
 * median / linear-interpolated percentile.  on_device: u, u_ref, err are device pointers. */
int hadr_relative_error(long long n, const double* u, const double* u_ref, double floor, double* err,
                        double* floor_used, long long* count, const long long* idx, int nidx, double* vals,
                        int on_device);

/* ---- Krylov (helmadr/krylov.py) ---- */
/* _gmres_relax_pre / gmres_relax (helmadr/krylov.py:82-119) */
int hadr_gmres_relax(hadr_op A, const double* b, const double* x, int steps, double* x_out, int on_device);
/* fgmres(A, b, x0, precond=make_kcycle_preconditioner(M) or None, cfg) (helmadr/krylov.py:122-242).
 * M may be NULL (identity preconditioner); x0 may be NULL (zero). */
int hadr_fgmres(hadr_op A, hadr_hier M, const double* b, const double* x0, int restart, int maxiter, double tol,
                double* x_out, hadr_report* rep, double* history, int history_cap, int on_device);
/* fgmres with KrylovConfig's switches (helmadr/krylov.py:16-31): flags HADR_FG_NONFLEXIBLE = cfg.flexible
 * False (x += M(V[:k]^T y) at the end of each cycle, helmadr/krylov.py:222-223; identical to the flexible
 * update when M is NULL), HADR_FG_DIAGNOSTICS = cfg.collect_diagnostics (rep->ortho_max,
 * helmadr/krylov.py:214-217). */
#define HADR_FG_NONFLEXIBLE 1
#define HADR_FG_DIAGNOSTICS 2
int hadr_fgmres_ex(hadr_op A, hadr_hier M, const double* b, const double* x0, int restart, int maxiter, double tol,
                   int flags, double* x_out, hadr_report* rep, double* history, int history_cap, int on_device);

#ifdef __cplusplus
}
#endif
#endif /* HADR_H */
