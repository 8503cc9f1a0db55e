// Host-side engine: device operators, multigrid hierarchy, K-cycle emission
// (captured once as a CUDA graph per input/output pair) and the outer FGMRES.
#pragma once
#include <cuda_runtime.h>

#include <map>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "cluster_engine.h"
#include "kernels.cuh"

namespace hadr {

struct CudaError : std::runtime_error {
  CudaError(cudaError_t e, const char* what, const char* file, int line)
      : std::runtime_error(std::string("CUDA error ") + cudaGetErrorString(e) + " at " + file + ":" +
                           std::to_string(line) + " (" + what + ")") {}
};
struct ValueError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// Process-wide device context: one stream, one reduction scratch.
struct Ctx {
  int device = 0;
  int nsm = 148;
  cudaStream_t stream = nullptr;
  RedScratch rs{};
  RedScratch rs2{};          // second partials buffer: a deferred reduction's consumer writes its own here
  double* dscal = nullptr;   // device scalars for host readback
  double* hscal = nullptr;   // pinned mirror
  LaunchCfg lc{};
  static Ctx& get();
  void sync() { HADR_CUDA(cudaStreamSynchronize(stream)); }
};

// Caching device allocator (exact-size free lists): repeated solves of one
// configuration reuse their buffers instead of cudaMalloc/cudaFree per solve.
void* pool_alloc(size_t bytes);
void pool_free(void* p);
size_t pool_trim();  // release cached blocks; returns bytes freed
template <class T>
T* dalloc(size_t n) {
  return (T*)pool_alloc((n == 0 ? 1 : n) * sizeof(T));
}
inline void dfree(void* p) {
  if (p) pool_free(p);
}

// Structured 2D/3D operator (owns its coefficient planes).
// Slab operators (multi-GPU, dist.h) hold the rows of global axis-0 planes
// [p0, p0 + nown) plus `hal` halo planes on each side; `coef` points at the
// first owned row and coefficient planes are `pstride` apart.
struct Op {
  int n1 = 0, n2 = 0, n3 = 1;  // 2D: n3 = 1 (global shape)
  long N = 0;                  // global points
  int p0 = 0, nown = 0, hal = 0;
  long pstride = 0;
  int nofs = 0;
  int8_t d1[HADR_MAX_OFS] = {0}, d2[HADR_MAX_OFS] = {0}, d3[HADR_MAX_OFS] = {0};
  cplx* coef = nullptr;
  float2* coef32 = nullptr;  // complex64 copy used by the K-cycle in mixed precision (null: c128)
  cplx* dinv = nullptr;      // lazily computed inverse diagonal
  // pair-compressed copy of the owned rows (StencilDev::pcode), read by the flat stencil kernel
  uint8_t* pcode = nullptr;
  cplx* pcoef = nullptr;
  float2* pcoef32 = nullptr;
  int nslot = 0;
  bool pc_tried = false;
  // class-compressed copy of the owned rows (StencilDev::ccode), coarse upwind Galerkin operators
  uint16_t* ccode = nullptr;
  cplx* ccoef = nullptr;
  float2* ccoef32 = nullptr;
  int4* ctab = nullptr;
  int* cnsl = nullptr;
  int nsl = 0;
  long mixed_rows = 0;  // rows whose class holds both +-2 sides of some axis
  bool cc_tried = false;
  ~Op();
  void make_c64();           // (re)build coef32 (and pcoef32) from coef (pcoef)
  // (re)build the pair-compressed copy from coef; false (and no copy) when no +-2 pair
  // exists or a row holds both members.  Reuses its buffers when refreshing.
  bool pair_compress();
  // (re)build the class-compressed copy; false (and no copy) when the union is not an upwind
  // reach-2 set or the rows would read more than 85% of the union's planes on average
  bool class_compress();
  StencilDev dev() const;
  int center() const;
  const cplx* inv_diag();  // computes on first use; throws ValueError on a zero diagonal
  void refresh_inv_diag();  // recompute into the existing buffer (coefficients changed)
  bool slab() const { return nown > 0; }
  int own() const { return nown > 0 ? nown : n1; }
  long n23() const { return (long)n2 * n3; }
  long nloc() const { return (long)own() * n2 * n3; }      // owned points
  long stride() const { return pstride > 0 ? pstride : N; }
  long alloc_len() const { return (long)nofs * stride(); }  // coefficient entries incl. halos
  long base_off() const { return (long)hal * n23(); }       // coef - base
};
Op* op_copy(const Op& A);

Op* op_from_csr(int n1, int n2, int n3, long nnz, const int64_t* indptr, const int32_t* indices, const cplx* data);
Op* op_from_planes(int n1, int n2, int n3, int nofs, const int* offsets /* 3 per offset */, const cplx* coef_host);
Op* op_axpby(cplx alpha, const Op& A, cplx beta, const Op& B);       // alpha*A + beta*B on the union pattern
Op* op_add_diag_real(const Op& A, cplx sc, const double* field_host);  // A + diag(sc*field)
Op* op_similarity(const Op& A, const cplx* left_host, const cplx* right_host);
Op* op_galerkin(const Op& A);                                          // P^T A P
// ADR (scheme 0 central, 1 upwind1, 2 upwind2) or Helmholtz (scheme 3) operator, fields host (n1*n2)
Op* op_assemble(int dim, int n1, int n2, int n3, double h1, double h2, double h3, double omega, int scheme,
                const int* bc /* top,bottom,left,right,front,back */, int src1, int src2, int src3, const double* ksq,
                const double* gam, const double* g1, const double* g2, const double* g3, const double* lap,
                bool fields_on_device = false);
void op_apply(const Op& A, const cplx* x, cplx* y);                    // device pointers, async

struct Shape3 {
  int n1, n2, n3;
};

struct Level {
  Op* A = nullptr;
  bool own = false;
  int n1 = 0, n2 = 0, n3 = 1;
  long N = 0;                // points this rank computes (slab levels: owned points)
  bool dist = false;         // slab level (vectors carry kHalo halo planes each side)
  int p0 = 0, nown = 0;      // owned global planes [p0, p0 + nown)
  std::vector<int> bounds;   // slab level: every rank's first plane (size + 1 entries)
  const cplx* dinv = nullptr;
  int s = 0;                 // relaxation length at this level
  bool smr = false;          // its engine relaxation runs out of shared memory (fixed at allocation)
  LaunchCfg lc{};            // single-GPU launch config of the level's kernels (points per thread)
  bool smc = false;          // ... with its coefficient rows staged there too
  // K-cycle workspace
  cplx* r = nullptr;
  cplx* V[RMAX + 1] = {nullptr};
  cplx* w[2] = {nullptr, nullptr};
  cplx* z = nullptr;         // split relaxation input D^-1 (s w) (large 3D levels, g_relax_split)
  RelaxCtl* rctl = nullptr;
  // inner-FGMRES workspace (levels >= 2)
  cplx *fb = nullptr, *fx = nullptr, *fV0 = nullptr, *fu = nullptr, *fZ0 = nullptr, *fZ1 = nullptr,
       *fw = nullptr, *fr = nullptr;
  FgCtl* fctl = nullptr;
};

// The runtime options a hierarchy's structure and captured graphs depend on (engine
// split, shared-memory relaxations, stencil paths, launch attributes, profiling).
std::vector<long long> hier_option_signature();

struct Hier {
  std::vector<Level> lv;
  std::vector<long long> opt_sig = hier_option_signature();  // options at construction
  bool poolable = false;     // owns copies of every level operator: may be recycled
  bool c64 = false;          // K-cycle operators applied from complex64 storage (mixed precision)
  int coarse_steps = 10;
  double coarse_tol = 0.1;
  int* kact = nullptr;      // device: K-cycle-active flag per level
  CEDesc* ce_desc = nullptr;  // device: level descriptors for the cluster engine
  bool use_ce(int li) const;  // level li's coarse part runs in the cluster engine
  size_t ce_tile(int li) const;  // engine dynamic shared memory when entered at level li
  int* visits = nullptr;    // device: visit counters (stats mode)
  std::map<std::pair<const void*, void*>, cudaGraphExec_t> graphs;
  std::map<std::pair<const void*, void*>, long long> graph_kernels;  // kernel nodes per graph
  int ndist = 0;             // leading slab-distributed levels (multi-GPU)
  LaunchCfg dlc{};           // launch config of slab levels (reductions across ranks)
  const LaunchCfg& lcf(const Level& L) const;
  void xchg(const Level& L, const cplx* v) const;  // halo exchange of a slab-level vector
  cplx* valloc(const Level& L) const;              // level vector (with halos on slab levels)
  ~Hier();
  void alloc_workspace();
  // emit the kernels of k_cycle(level li, b, x0 -> xo) onto the context stream
  void emit_kcycle(int li, const cplx* b, const cplx* x0, cplx* xo, Gate g, bool count);
  void emit_relax(Level& L, const cplx* b, const cplx* x, cplx* xo, int s, Gate g);
  void emit_inner(int ci, Gate g, bool count);
  // precond application z = K(v) from level 1 with x = 0, via a cached CUDA graph
  void apply(const cplx* v, cplx* z);
  void kcycle_direct(int li, const cplx* b, const cplx* x0, cplx* xo, int* visits_host);
};

// runtime options (hadr_set_option)
extern long g_small_max_work;  // engine / cluster-kernel levels also need N x offsets <= this (option "small_max_work")
extern long g_ce_max_n;  // levels with N <= this run inside the cluster engine (0 disables)
extern int g_kcycle_c64; // build hierarchies with complex64 operator storage (mixed-precision K-cycle)
extern int g_ce_smem_relax;  // engine relaxations out of shared memory where they fit
extern int g_pair_compress;  // pair-compress fine operators (outer A, hierarchy level 0)
extern int g_ce_smem_coef;   // option "ce_smem_coef"
extern int g_defer_mgs;     // MGS dot finalizes folded into the next axpy (option "defer_mgs")
extern long g_relax_split;   // 3D levels with at least this many points form D^-1 (s w) once per point
extern int g_class_compress;  // class-compress coarse graph-path levels: 0 off, 1 3D, 2 2D and 3D

Hier* hier_build(Op* fine, int max_levels, int coarse_steps, double coarse_tol);
void hier_release(Hier* h);  // recycle (workspace + captured graphs) or delete
Hier* hier_pool_pop();       // take one recycled hierarchy (or null)
Hier* hier_from_ops(int nlev, Op** ops, int coarse_steps, double coarse_tol);
// Multi-GPU: slab plan of a global grid (fine slab bounds + number of distributed levels)
struct SlabPlan {
  std::vector<int> bounds;  // fine axis-0 slab starts, size + 1 entries
  int ndist = 0;            // levels 0 .. ndist-1 are slab-distributed, the rest replicated
  int nlev = 0;
};
SlabPlan slab_plan(int n1, int n2, int n3, int max_levels);
SlabPlan slab_plan_for(int n1, int n2, int n3, int max_levels, int ranks);  // host logic only
// hierarchy over a slab fine operator (every rank calls it collectively)
Hier* hier_build_dist(Op* fine_slab, const SlabPlan& plan, int coarse_steps, double coarse_tol);
// slab assembly: rows of this rank's slab (+1 halo row each side) from global host/device fields
Op* op_assemble_slab(int dim, int n1, int n2, int n3, double h1, double h2, double h3, double omega, int scheme,
                     const int* bc, int src1, int src2, int src3, const double* ksq, const double* gam,
                     const double* g1, const double* g2, const double* g3, const double* lap, bool fields_on_device,
                     int p0, int nown);
std::vector<Shape3> coarsenable_levels(int n1, int n2, int n3, int max_levels);

struct Report {
  int iterations = 0;
  int converged = 0;
  int note = 0;
  double bnorm = 0, final_relres = 0, wall_time = 0;
  double device_time = 0;  // CUDA events on the library stream around the solve
  double ortho_max = 0;    // max |<v_i, v_j>|, i != j, over the restart cycles (collect_diagnostics)
  std::vector<double> history;
};

enum : int { FG_NONFLEXIBLE = 1, FG_DIAGNOSTICS = 2 };

// x = fgmres(A, b, x0, M) on device pointers (x0 may be null)
// flags: FG_NONFLEXIBLE (x += M(V[:k]^T y), helmadr/krylov.py:222-223), FG_DIAGNOSTICS (ortho_max,
// helmadr/krylov.py:214-217)
void fgmres(Op& A, Hier* M, const cplx* b, const cplx* x0, cplx* x, int restart, int maxiter, double tol,
            Report& rep, int flags = 0);
// Jacobi-GMRES relaxation of arbitrary length on one operator (public gmres_relax)
void gmres_relax(Op& A, const cplx* b, const cplx* x, cplx* xo, int steps);

}  // namespace hadr
