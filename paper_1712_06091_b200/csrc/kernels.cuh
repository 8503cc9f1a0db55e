// Launch interface of the sm_100a kernels (kernels.cu) used by the host engine.
#pragma once
#include "ctl.cuh"

namespace hadr {

extern long long g_launch_count;
extern int g_pdl;
extern int g_mid_ppt;    // points per thread of a 2D level's kernels with mid_min_n < N <= mid_max_n
extern long g_mid_max_n;
extern long g_mid_min_n;  // programmatic dependent launch of the solve-phase kernels
extern int g_stencil_tile;
extern int g_stencil_march;   // plane-marching bulk-copy kernel on 3D pair-compressed fine levels
extern long g_march_min_n, g_march_min_n2d;
struct StencilDev;
bool march_takes(const StencilDev& A);
// the marching kernel's tiling of an (n1own, n2, n3) slab (n3 = 1: 2D): out[10] = {nty, ntx, nch, pc, pitch,
// slot, hy, blocks, smem bytes, points per tile cap}; false when the kernel declines the shape
bool march_plan(int n1own, int n2, int n3, int jac, int* out);  // launch_stencil runs the marching kernel on this operator
extern long g_cl_max_n;  // single-cluster reductions (in-kernel epilogue) up to this many points  // shared-memory tiled stencil kernel on the graph path

// Structured 2D/3D stencil in union-offset, plane-major layout (2D: n3 = 1, d3 = 0):
//   k = (i1*n2 + i2)*n3 + i3,  coef[o*N + k] multiplies x[k + (d1*n2 + d2)*n3 + d3],
//   offsets sorted by (d1, d2, d3) == ascending column index of the reference
//   CSR row for every in-grid entry, so the accumulation order equals scipy
//   csr_matvec's.
// Multi-GPU slabs along axis 0: a rank owns global planes [p0, p0 + n1own) of the
// n1 global planes; every pointer handed to a kernel points at the first OWNED
// point, halo planes sit at negative / past-the-end offsets, and coefficient
// planes are `pstride` apart.  Single GPU: p0 = 0, n1own = n1, pstride = N.
// Standard 2D offset sets in ascending (d1, d2) order, known at compile time to the
// cluster engine's fast stencil loops (StencilDev::std2d names the set an operator has).
// 21: the 5x5 box minus its corners (coarse Galerkin operators of upwind fine operators);
// 9: the plus of radius 2 (fine upwind/blend operators); 5: the plus of radius 1.
struct Std2D {
  template <int NO>
  __host__ __device__ static constexpr int d1(int o) {
    constexpr int a21[21] = {-2, -2, -2, -1, -1, -1, -1, -1, 0, 0, 0, 0, 0, 1, 1, 1, 1, 1, 2, 2, 2};
    constexpr int a9[9] = {-2, -1, 0, 0, 0, 0, 0, 1, 2};
    constexpr int a5[5] = {-1, 0, 0, 0, 1};
    return NO == 21 ? a21[o] : NO == 9 ? a9[o] : a5[o];
  }
  template <int NO>
  __host__ __device__ static constexpr int d2(int o) {
    constexpr int a21[21] = {-1, 0, 1, -2, -1, 0, 1, 2, -2, -1, 0, 1, 2, -2, -1, 0, 1, 2, -1, 0, 1};
    constexpr int a9[9] = {0, 0, -2, -1, 0, 1, 2, 0, 0};
    constexpr int a5[5] = {0, -1, 0, 1, 0};
    return NO == 21 ? a21[o] : NO == 9 ? a9[o] : a5[o];
  }
};

struct StencilDev {
  int n1, n2, n3;
  int nofs;
  int p0, n1own;
  int std2d;  // 2D operator whose offsets are exactly the Std2D set of this size (21 / 9 / 5), else 0
  int halo;   // max |linear displacement| of the offsets (the engine's point-partition halo)
  long pstride;
  int8_t d1[HADR_MAX_OFS];
  int8_t d2[HADR_MAX_OFS];
  int8_t d3[HADR_MAX_OFS];
  const cplx* coef;
  const float2* coef32;  // non-null: apply with complex64-stored coefficients (mixed-precision K-cycle)
  // Pair-compressed copy (fine upwind operators, plus-radius-2 union): the offsets +-2
  // along one axis are never both non-zero in a row (the upwind side), so they share
  // one plane; bit d of pcode[k] is set when row k holds the +2 member of axis d.
  // Slot planes (kernels.cu PcLayout) are pstr apart and cover the owned points only.
  const uint8_t* pcode;
  const cplx* pcoef;
  const float2* pcoef32;
  long pstr;
  // Class-compressed copy (coarse Galerkin operators of upwind fine operators): a row's
  // class fixes, per axis, which +-2 offsets it may hold (the upwind side '-' or '+',
  // or both where the upwind direction changes) — 3^dim classes.  Class c lists its
  // cnsl[c] live union offsets in ascending order (ctab[c * nsl + q] = {linear
  // displacement, d1, d2, d3}); a row reads only its class's slots, planes cstr apart
  // (owned points only), so a row in an interior class streams 15 (2D) / 54 (3D)
  // planes instead of the union's 21 / 81.
  const uint16_t* ccode;  // class | (slots of the class << 8)
  const cplx* ccoef;
  const float2* ccoef32;
  const int4* ctab;
  const int* cnsl;
  long cstr;
  int nsl;  // table row stride = slot planes stored
};

// coefficient from complex64 storage, widened to complex128 for the arithmetic
__device__ __forceinline__ cplx ld_c64(const StencilDev& A, long idx) {
  const float2 c = __ldg(A.coef32 + idx);
  return make_double2((double)c.x, (double)c.y);
}

// 125 offset slots of the 5x5x5 box, ascending == lexicographic (d1, d2, d3)
__host__ __device__ __forceinline__ int slot125(int d1, int d2, int d3) { return ((d1 + 2) * 5 + (d2 + 2)) * 5 + (d3 + 2); }
struct Mask125 {
  unsigned long long w[2];
};

enum : int { IN_PLAIN = 0, IN_SCALE = 1, IN_JAC = 2, IN_WRITEV = 4 };
enum : int { OUT_APPLY = 0, OUT_RESID = 1 };
enum : int { RED_NONE = 0, RED_NORM = 1, RED_DOT = 2, RED_DOT_CENTER = 4 };

enum EpiCode : int {
  EPI_NONE = 0,
  EPI_STORE,        // out[0..nv) = totals
  EPI_RELAX_BETA,   // beta = sqrt(t0)
  EPI_RELAX_H,      // H[i][j] = dot
  EPI_RELAX_STEP,   // H[j+1][j] = sqrt(t0); Givens; stop/continue
  EPI_FG_INIT,      // bnorm
  EPI_FG_S,         // w0 = sqrt(t0), H[0][j] = (t1, t2)
  EPI_FG_H,         // H[i][j] = dot
  EPI_FG_CORR,      // corr[i] = dot; H[i][j] += corr
  EPI_FG_N,         // wn; reo decision; inner: post if no reorth
  EPI_FG_N2,        // wn after reorth; inner: post
  EPI_FG_RES,       // inner early-exit residual -> restart decision
};

struct Epi {
  int code;
  int i, j;
  int inner;   // FG_N / FG_N2: run the device-side FGMRES post-step
  void* ctl;
  double* out;
};
inline Epi epi_none() { return Epi{EPI_NONE, 0, 0, 0, nullptr, nullptr}; }
inline Epi epi_store(double* out) { return Epi{EPI_STORE, 0, 0, 0, nullptr, out}; }
inline Epi epi(int code, void* ctl, int i = 0, int j = 0, int inner = 0) { return Epi{code, i, j, inner, ctl, nullptr}; }

struct StencilArgs {
  StencilDev A;
  const cplx* x;       // input vector (neighbours read)
  const double* scale; // IN_SCALE: x*(*scale)
  const cplx* dinv;    // IN_JAC: dinv (.) x
  cplx* vout;          // IN_WRITEV: transformed-but-unjacobied centre value
  const cplx* b;       // OUT_RESID
  cplx* y;             // output
  const cplx* u;       // RED_DOT partner (conjugated)
  Gate gate;
  RedScratch rs;
  Epi epi;
};

// Multi-GPU reductions: local totals -> `buf` (4 doubles), `gather` all-gathers every rank's
// buf into `all` (size x 4) on the stream, a 1-thread kernel sums them in rank order and
// runs the scalar epilogue (identical control state on every rank).
struct DistRed {
  int size;
  double* buf;
  double* all;
  void (*gather)(void* ctx, cudaStream_t s);
  void* ctx;
};

struct LaunchCfg {
  cudaStream_t stream;
  int max_blocks;                  // grid cap (multiple of the SM count)
  const DistRed* dist = nullptr;   // non-null: reductions are completed across the slab ranks
  int ppt = 1;                     // points per thread of the level's grid-stride kernels
  long cl_max_n = -1;              // >= 0: the level's own single-cluster limit (min with option cl_max_n)
};

void launch_stencil(const LaunchCfg& lc, int inm, int outm, int red, const StencilArgs& a);

// A 2-value (complex dot) reduction whose 1-block finalize was not launched: its consumer
// (the next MGS axpy of the chain) sums the producer's per-block partials itself, with the
// finalize kernel's exact summation (same thread layout, same order: bit-identical totals
// in every block), block 0 running the deferred epilogue.  Saves one kernel per link.
struct Pend {
  const double* partials = nullptr;  // producer's per-block partials (2 per block); null: none
  int nblocks = 0;
  Epi e{};
};
// While *g_defer_out is non-null, a 2-value finalize on a plain grid (no cluster, no
// multi-GPU communicator) is recorded there instead of launched.
extern Pend* g_defer_out;

// w -= (*h) * v ; then reduce: RED_DOT -> <u, w>, RED_NORM -> ||w||^2
void launch_axpy_red(const LaunchCfg& lc, long n, cplx* w, const cplx* h, const cplx* v, int red, const cplx* u,
                     Gate g, RedScratch rs, Epi e, Pend in = Pend{});
// reduce <u, w>
void launch_dot(const LaunchCfg& lc, long n, const cplx* u, const cplx* w, Gate g, RedScratch rs, Epi e);
// out = in * (*s) (s may be null: copy); red: RED_NORM of out ; out may be null (reduction only)
void launch_scale(const LaunchCfg& lc, long n, const cplx* in, const double* s, cplx* out, int red, Gate g,
                  RedScratch rs, Epi e);
void launch_zero(const LaunchCfg& lc, long n, cplx* out, Gate g);
// v = (*s) in ; z = dinv (.) v   (the relaxation step's input, split out of the stencil)
void launch_scale_jac(const LaunchCfg& lc, long n, const cplx* in, const double* s, const cplx* dinv, cplx* v,
                      cplx* z, Gate g);

// out = base + [dinv (.)] sum_{i<k} v_i * y_i ; k = *kptr if kptr else kfix ; base may be null (zero)
struct LinComb {
  const cplx* v[MMAX];
  const cplx* y;       // device coefficients (ctl) or null -> yv
  cplx yv[MMAX];       // by-value coefficients
  const int* kptr;
  int kfix;
  const cplx* base;
  const cplx* dinv;    // optional Jacobi on the sum
  cplx* out;
};
void launch_lincomb(const LaunchCfg& lc, long n, const LinComb& c, Gate g);

// Inner FGMRES finalisation, branches on the device path/cycle (helmadr/krylov.py:218-223).
void launch_fg_finalize(const LaunchCfg& lc, long n, FgCtl* f, const cplx* Z0, const cplx* Z1, cplx* x, Gate g,
                        int brk_stage);

// Restriction rc = P^T r and prolongation x += P e (bilinear P, helmadr/multigrid.py:19-46).
// (tri)linear P = kron(P1(n1), P1(n2), P1(n3)); an axis of size 1 is not coarsened.
// Slabs: restriction writes coarse planes [q0, q0 + nq) (nq < 0: all) from the fine slab starting at global
// plane p0f (one halo plane below it is read); prolongation updates fine planes [p0f, p0f + nf) (nf < 0: all)
// from a coarse vector whose index 0 is global coarse plane q0c.
void launch_restrict(const LaunchCfg& lc, int n1f, int n2f, int n3f, const cplx* r, cplx* rc, Gate g, int p0f = 0,
                     int q0 = 0, int nq = -1);
void launch_prolong_add(const LaunchCfg& lc, int n1f, int n2f, int n3f, const cplx* ec, cplx* x, Gate g,
                        int p0f = 0, int nf = -1, int q0c = 0);

void launch_set_gate(cudaStream_t s, int* dst, Gate g);
void launch_relax_init(cudaStream_t s, RelaxCtl* c, int steps, Gate g);
void launch_fg_setup(cudaStream_t s, FgCtl* f, double tol, Gate g);

// ---- operator construction (setup) ----
// mask: 2 x u64 offset bitset + 1 u64 "reach beyond the box" flag
void launch_csr_mask(cudaStream_t s, int n1, int n2, int n3, const int64_t* indptr, const int32_t* indices,
                     unsigned long long* mask);
void launch_csr_scatter(cudaStream_t s, int n1, int n2, int n3, const int64_t* indptr, const int32_t* indices,
                        const cplx* data, const int* slot_of, cplx* coef);
void launch_cdiv(cudaStream_t s, long n, const cplx* r, const cplx* d, cplx* z);
void launch_inv_diag(cudaStream_t s, long n, const cplx* diag, cplx* dinv, int* zero_flag);
void launch_remap_planes(cudaStream_t s, long n, const cplx* src, int nsrc, const int* dst_slot, cplx* dst,
                         cplx alpha, int accumulate);
void launch_add_diag_real(cudaStream_t s, long n, cplx* center, cplx sc, const double* field);
void launch_similarity(cudaStream_t s, const StencilDev& A, cplx* out, const cplx* left, const cplx* right);
// ADR/Helmholtz assembly into the plus-radius-2 planes of `dim` axes (2D: 9, 3D: 13 planes);
// bc[6] = (top, bottom, left, right, front, back) face kinds (0 neumann, 1 sommerfeld)
void launch_assemble(cudaStream_t s, int dim, int n1, int n2, int n3, double h1, double h2, double h3, double omega,
                     int scheme, const int* bc, int src1, int src2, int src3, const double* ksq, const double* gam,
                     const double* g1, const double* g2, const double* g3, const double* lap, cplx* coefp,
                     unsigned* mask, int r0 = 0, int nr = -1, long pstride = -1);
void launch_to_c64(cudaStream_t s, long n, const cplx* in, float2* out);
// pair compression of the owned rows of a plus-radius-2 union (kernels.cu PcLayout):
// pair_layout fills the slot table (returns the slot count, 0 if nofs is not 9 / 13);
// *conflict |= 1 where a row holds both members of a pair
int pair_layout(int nofs, int* pos_a, int* pos_b, int* bit);
void launch_pair_compress(cudaStream_t s, const StencilDev& A, int nslot, const int* pos_a, const int* pos_b,
                          const int* bit, cplx* pcoef, long pstr, uint8_t* pcode, int* conflict);
// class compression of the owned rows (Op::class_compress): pass 1 classifies every row into
// the first class (ascending size) whose live bitset (live[2c], live[2c+1]) covers its
// non-zeros, ccode[k] = c, and accumulates stats[0] += slots read, stats[1] = max class size,
// stats[2] += rows of mixed classes; pass 2 fills slot q < cnsl[c] of row k from union
// plane otab[c * nsl + q]
void launch_class_classify(cudaStream_t s, const StencilDev& A, int ncls, const unsigned long long* live_dev,
                           const int* cnsl_dev, const int* mixed_dev, uint16_t* ccode, unsigned long long* stats);
void launch_class_fill(cudaStream_t s, const StencilDev& A, const uint16_t* ccode, const int* cnsl_dev,
                       const int* otab_dev, int nsl, cplx* ccoef, long cstr);
void launch_phase(cudaStream_t s, long n, const cplx* q, const double* tau, double omega, int sign, cplx* out);
// tau = tau0 tau1, grad(tau) (dim planes), lap(tau) from tau1 (helmadr/eikonal.py:15-36, 180-226); tau may be null
void launch_tau_derivs(cudaStream_t s, int dim, const int* n, const double* h, const double* L, const int* src,
                       const double* tau1, double* tau, double* const* grads, double* lap);
void launch_galerkin(cudaStream_t s, const StencilDev& Af, int n1c, int n2c, int n3c, unsigned long long* mask,
                     const int* slot_of, cplx* coef_c, int q0 = 0, int nq = -1, long cstride = -1);

}  // namespace hadr
