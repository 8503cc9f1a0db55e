// sm_100a kernels of the amplitude solve (FGMRES + multigrid K-cycle).
//
// Memory-bound complex128 stencil / BLAS-1 work: no tensor cores (nothing is a
// dense contraction).  Every streaming kernel is a grid-stride loop over a grid
// capped at a multiple of the SM count; reductions finish in the last block
// (deterministic order) which also runs the scalar control epilogue, so no
// separate "small" kernel and no host round trip is needed per Krylov step.
#include "kernels.cuh"
#include "krylov_ctl.cuh"

#include <set>
#include <stdexcept>
#include <utility>

namespace hadr {

long long g_launch_count = 0;  // kernels launched directly on the stream (graphs add their node count)

__device__ __noinline__ void run_epi(const Epi& e, const double* t, int nv) {
  switch (e.code) {
    case EPI_STORE:
      for (int q = 0; q < nv; ++q) e.out[q] = t[q];
      break;
    case EPI_RELAX_BETA: {  // the relaxation's start: steps (e.j), k, cur, then beta (helmadr/krylov.py:95-97)
      RelaxCtl* c = (RelaxCtl*)e.ctl;
      c->steps = e.j;
      c->k = 0;
      c->cur = kStopped;
      relax_beta(c, t[0]);
      break;
    }
    case EPI_RELAX_H:
      ((RelaxCtl*)e.ctl)->H[e.i * RMAX + e.j] = mk(t[0], t[1]);
      break;
    case EPI_RELAX_STEP:
      relax_step((RelaxCtl*)e.ctl, e.j, t[0]);
      break;
    case EPI_FG_INIT:
      fg_init((FgCtl*)e.ctl, t[0]);
      break;
    case EPI_FG_S: {
      FgCtl* f = (FgCtl*)e.ctl;
      f->w0 = sqrt(t[0]);
      f->H[0 * MMAX + e.j] = mk(t[1], t[2]);
      break;
    }
    case EPI_FG_H:
      ((FgCtl*)e.ctl)->H[e.i * MMAX + e.j] = mk(t[0], t[1]);
      break;
    case EPI_FG_CORR: {
      FgCtl* f = (FgCtl*)e.ctl;
      f->corr[e.i] = mk(t[0], t[1]);
      f->H[e.i * MMAX + e.j] = cadd(f->H[e.i * MMAX + e.j], f->corr[e.i]);
      break;
    }
    case EPI_FG_N: {
      FgCtl* f = (FgCtl*)e.ctl;
      f->wn = sqrt(t[0]);
      f->reo = (f->wn < kReorthRatio * f->w0) ? 1 : 0;  // helmadr/krylov.py:178-179
      if (!f->reo && e.inner) fg_post(f, e.j);
      break;
    }
    case EPI_FG_N2: {
      FgCtl* f = (FgCtl*)e.ctl;
      f->wn = sqrt(t[0]);
      if (e.inner) fg_post(f, e.j);
      break;
    }
    case EPI_FG_RES:
      fg_res((FgCtl*)e.ctl, t[0]);
      break;
    default:
      break;
  }
}

// ---------------------------------------------------------------------------
// Reductions without same-address atomics (the last-block ticket pattern
// serialises in L2: 31.7 us at 1184 blocks, measured in tools/sync_microbench.cu).
//   CL = 0 : every block writes its partial sums; a 1-block k_finalize follows
//            (fixed summation order, then the scalar epilogue).
//   CL = 1 : the whole grid is ONE thread-block cluster (<= 16 CTAs): partials
//            are summed through distributed shared memory and CTA 0 runs the
//            epilogue inside the same kernel (~0.55 us, measured).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ const double* cluster_map(const double* p, unsigned rank) {
  unsigned long long in = reinterpret_cast<unsigned long long>(p), out;
  asm volatile("mapa.u64 %0, %1, %2;" : "=l"(out) : "l"(in), "r"(rank));
  return reinterpret_cast<const double*>(out);
}

template <int NV, int CL>
__device__ __forceinline__ void finish(double (&v)[NV], const RedScratch& rs, const Epi& e) {
  __shared__ double sm[NV * 32];
  block_sum<NV>(v, sm);
  if constexpr (CL == 0) {
    if (threadIdx.x == 0) {
#pragma unroll
      for (int q = 0; q < NV; ++q) rs.partials[blockIdx.x * NV + q] = v[q];
    }
  } else {
    __shared__ double cp[NV];
    if (threadIdx.x == 0) {
#pragma unroll
      for (int q = 0; q < NV; ++q) cp[q] = v[q];
    }
    cluster_sync_all();
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      double tot[NV];
#pragma unroll
      for (int q = 0; q < NV; ++q) tot[q] = 0.0;
      for (unsigned r = 0; r < gridDim.x; ++r) {
        const double* rp = cluster_map(cp, r);
#pragma unroll
        for (int q = 0; q < NV; ++q) tot[q] += rp[q];
      }
      run_epi(e, tot, NV);
    }
    cluster_sync_all();  // keep every CTA's shared memory alive until CTA 0 has read it
  }
}

template <int NV>
__global__ void __launch_bounds__(kThreads) k_finalize(RedScratch rs, int nblocks, Gate g, Epi e) {
  pdl_enter();
  if (!gate_open(g)) return;
  __shared__ double sm[NV * 32];
  double acc[NV];
#pragma unroll
  for (int q = 0; q < NV; ++q) acc[q] = 0.0;
  for (int b = threadIdx.x; b < nblocks; b += blockDim.x) {
#pragma unroll
    for (int q = 0; q < NV; ++q) acc[q] += rs.partials[b * NV + q];
  }
  block_sum<NV>(acc, sm);
  if (threadIdx.x == 0) run_epi(e, acc, NV);
}

__device__ __forceinline__ cplx ldc(const cplx* p, long i) { return __ldg(p + i); }

// Launch geometry of one vector op: a single cluster for small levels, else a
// grid capped at a multiple of the SM count (+ a finalize kernel when reducing).
long g_cl_max_n = 32768;  // option "cl_max_n": vector ops up to this size reduce inside one cluster
constexpr int kClusterMaxCTAs = 16;

struct Geo {
  int blocks;
  int cluster;  // 0: plain grid
};

// Points per thread of the grid-stride vector / stencil kernels (LaunchCfg::ppt, set per
// hierarchy level): 2 on 2D levels of 70k-300k points (config 2's 513^2: -3% per solve;
// 257^2, the fine level and 3D levels lose or break even, 3-8 points per thread lose).
int g_mid_ppt = 2;          // option "mid_ppt"
long g_mid_min_n = 70000;   // option "mid_min_n"
long g_mid_max_n = 300000;  // option "mid_max_n"

static long blocks_of(const LaunchCfg& lc, long n) {
  const long ppt = lc.ppt > 1 ? lc.ppt : 1;
  return (n + kThreads * ppt - 1) / (kThreads * ppt);
}

static Geo geo_for(const LaunchCfg& lc, long n) {
  long b = (n + kThreads - 1) / kThreads;
  const long clmax = lc.cl_max_n >= 0 && lc.cl_max_n < g_cl_max_n ? lc.cl_max_n : g_cl_max_n;  // per-level cap
  if (n <= clmax && !lc.dist) {  // distributed sums finish through the communicator
    if (b > kClusterMaxCTAs) b = kClusterMaxCTAs;
    if (b < 1) b = 1;
    return Geo{(int)b, (int)b};
  }
  b = blocks_of(lc, n);
  if (b > lc.max_blocks) b = lc.max_blocks;
  return Geo{(int)b, 0};
}

static int blocks_for(const LaunchCfg& lc, long n) {
  long b = blocks_of(lc, n);
  if (b > lc.max_blocks) b = lc.max_blocks;
  if (b < 1) b = 1;
  return (int)b;
}

int g_pdl = 1;  // programmatic dependent launch of the solve-phase kernels (option "pdl")

static inline int pdl_attr(cudaLaunchAttribute* at) {
  if (!g_pdl) return 0;
  at->id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at->val.programmaticStreamSerializationAllowed = 1;
  return 1;
}

template <typename... KArgs, typename... Args>
static void launch_k(void (*kern)(KArgs...), int blocks, int threads, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(threads);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  cfg.numAttrs = pdl_attr(at);
  cfg.attrs = at;
  cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

template <typename... KArgs, typename... Args>
static void launch_geo(void (*kern)(KArgs...), const Geo& geo, cudaStream_t s, Args&&... args) {
  if (!geo.cluster) {
    launch_k(kern, geo.blocks, kThreads, s, std::forward<Args>(args)...);
    return;
  }
  if (geo.cluster > 8) {  // non-portable cluster sizes must be enabled per kernel
    static std::set<const void*> enabled;
    if (!enabled.count((const void*)kern)) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      enabled.insert((const void*)kern);
    }
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(geo.blocks);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = geo.cluster;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1 + pdl_attr(at + 1);
  cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// Distributed reduction: every rank's local totals are all-gathered and summed in
// rank order (so every rank holds bit-identical control state), then the epilogue.
template <int NV>
__global__ void k_epi_gathered(const double* all, int size, Gate g, Epi e) {
  pdl_enter();
  if (!gate_open(g)) return;
  double t[NV];
#pragma unroll
  for (int q = 0; q < NV; ++q) t[q] = 0.0;
  for (int r = 0; r < size; ++r) {
#pragma unroll
    for (int q = 0; q < NV; ++q) t[q] += all[r * 4 + q];
  }
  run_epi(e, t, NV);
}

Pend* g_defer_out = nullptr;

template <int NV>
static void launch_finalize(const LaunchCfg& lc, const Geo& geo, Gate g, RedScratch rs, Epi e) {
  if (geo.cluster) return;
  if (NV == 2 && g_defer_out && !lc.dist) {  // the consumer finishes it (Pend)
    *g_defer_out = Pend{rs.partials, geo.blocks, e};
    return;
  }
  ++g_launch_count;
  if (!lc.dist) {
    launch_k(k_finalize<NV>, 1, kThreads, lc.stream, rs, geo.blocks, g, e);
    return;
  }
  const DistRed& d = *lc.dist;
  launch_k(k_finalize<NV>, 1, kThreads, lc.stream, rs, geo.blocks, g, epi_store(d.buf));
  d.gather(d.ctx, lc.stream);
  ++g_launch_count;
  launch_k(k_epi_gathered<NV>, 1, 1, lc.stream, (const double*)d.all, d.size, g, e);
}

// ---------------------------------------------------------------------------
// K1: stencil apply   y = A x   |   y = b - A x      (2D: n3 = 1)
//   input transform per neighbour: v = x*s (IN_SCALE), v = dinv (.) v (IN_JAC)
//   IN_WRITEV stores the centre's scaled input (the new Krylov basis vector).
//   reductions: ||y||^2, <u, y> (u = array, or the centre input with RED_DOT_CENTER)
// NO > 0: all NO offsets unrolled with batched loads; NO == 0: runtime chunks of
// 9 offsets (3D coarse unions of 27..81 offsets).
// ---------------------------------------------------------------------------
template <int CH, int INM, bool C32>
__device__ __forceinline__ void stencil_chunk(const StencilArgs& a, int o0, int nofs, long k, int i1, int i2, int i3,
                                              int n1, int n2, int n3, long N, double s, cplx& acc) {
  // All loads are unconditional (out-of-grid neighbours read the centre, dead
  // offsets read plane 0) so the compiler can batch them; out-of-grid terms are
  // then skipped, which keeps scipy csr_matvec's exact accumulation.
  cplx cv[CH], xv[CH], dv[CH];
  bool ok[CH];
#pragma unroll
  for (int q = 0; q < CH; ++q) {
    const int o = o0 + q;
    const bool live = o < nofs;
    const int oo = live ? o : 0;
    const int d1 = a.A.d1[oo], d2 = a.A.d2[oo], d3 = a.A.d3[oo];
    const int j1 = i1 + d1, j2 = i2 + d2, j3 = i3 + d3;  // j1: global plane (i1 global)
    ok[q] = live && j1 >= 0 && j1 < n1 && j2 >= 0 && j2 < n2 && j3 >= 0 && j3 < n3;
    const long jj = ok[q] ? k + ((long)d1 * n2 + d2) * n3 + d3 : k;  // owned-relative (halos at < 0)
    cv[q] = C32 ? ld_c64(a.A, live ? (long)o * N + k : k) : ldc(a.A.coef, live ? (long)o * N + k : k);
    xv[q] = ldc(a.x, jj);
    if (INM & IN_JAC) dv[q] = ldc(a.dinv, jj);
  }
#pragma unroll
  for (int q = 0; q < CH; ++q) {
    cplx v = xv[q];
    if (INM & IN_SCALE) v = cscale(v, s);
    if (INM & IN_JAC) v = cmul_np(dv[q], v);
    const cplx t = cadd(acc, cmul_sp(cv[q], v));
    acc = ok[q] ? t : acc;
  }
}

// Pair-compressed fine operator (StencilDev::pcode): the union is exactly the
// plus-radius-2 set (centre, +-1 and +-2 along each of D axes; 2D 9, 3D 13 offsets
// in sorted order) and the two +-2 offsets of an axis share one coefficient plane.
// One load per slot (2D 7, 3D 10 instead of 9 / 13); the far term of axis d is
// computed once and added at the position of whichever member the row holds, so
// the accumulation order (ascending column) and rounding equal the union kernel's.
//   2D union positions: 0 (-2,0) 1 (-1,0) 2 (0,-2) 3 (0,-1) 4 centre 5 (0,1) 6 (0,2) 7 (1,0) 8 (2,0)
//   3D: 0 (-2,0,0) 1 (-1,0,0) 2 (0,-2,0) 3 (0,-1,0) 4 (0,0,-2) 5 (0,0,-1) 6 centre
//       7 (0,0,1) 8 (0,0,2) 9 (0,1,0) 10 (0,2,0) 11 (1,0,0) 12 (2,0,0)
template <int NO>
struct PcLayout;
template <>
struct PcLayout<9> {
  static constexpr int NS = 7;
  // slot of each union position; pair (axis) of a position or -1; member: 0 minus, 1 plus
  __host__ __device__ static constexpr int slot(int p) {
    constexpr int t[9] = {0, 1, 2, 3, 4, 5, 2, 6, 0};
    return t[p];
  }
  __host__ __device__ static constexpr int pair(int p) {
    constexpr int t[9] = {0, -1, 1, -1, -1, -1, 1, -1, 0};
    return t[p];
  }
  __host__ __device__ static constexpr int plus_pos(int q) {  // slot -> union position of its plus member
    constexpr int t[7] = {8, -1, 6, -1, -1, -1, -1};
    return t[q];
  }
  __host__ __device__ static constexpr int first_pos(int q) {  // slot -> union position (minus member)
    constexpr int t[7] = {0, 1, 2, 3, 4, 5, 7};
    return t[q];
  }
  __host__ __device__ static constexpr int axis(int q) {  // slot -> axis of its offset (-1: centre)
    constexpr int t[7] = {0, 0, 1, 1, -1, 1, 0};
    return t[q];
  }
  __host__ __device__ static constexpr int delta(int q) {  // slot -> offset along that axis (pairs: -2)
    constexpr int t[7] = {-2, -1, -2, -1, 0, 1, 1};
    return t[q];
  }
};
template <>
struct PcLayout<13> {
  static constexpr int NS = 10;
  __host__ __device__ static constexpr int slot(int p) {
    constexpr int t[13] = {0, 1, 2, 3, 4, 5, 6, 7, 4, 8, 2, 9, 0};
    return t[p];
  }
  __host__ __device__ static constexpr int pair(int p) {
    constexpr int t[13] = {0, -1, 1, -1, 2, -1, -1, -1, 2, -1, 1, -1, 0};
    return t[p];
  }
  __host__ __device__ static constexpr int plus_pos(int q) {
    constexpr int t[10] = {12, -1, 10, -1, 8, -1, -1, -1, -1, -1};
    return t[q];
  }
  __host__ __device__ static constexpr int first_pos(int q) {
    constexpr int t[10] = {0, 1, 2, 3, 4, 5, 6, 7, 9, 11};
    return t[q];
  }
  __host__ __device__ static constexpr int axis(int q) {
    constexpr int t[10] = {0, 0, 1, 1, 2, 2, -1, 2, 1, 0};
    return t[q];
  }
  __host__ __device__ static constexpr int delta(int q) {
    constexpr int t[10] = {-2, -1, -2, -1, -2, -1, 0, 1, 1, 1};
    return t[q];
  }
};

// The 3D plus of radius 1 (7 offsets in sorted order: (-1,0,0) (0,-1,0) (0,0,-1) centre (0,0,1) (0,1,0)
// (1,0,0)) in the same terms, for the marching kernel: one slot per offset, no pairs, union planes.
template <>
struct PcLayout<7> {
  static constexpr int NS = 7;
  __host__ __device__ static constexpr int slot(int p) { return p; }
  __host__ __device__ static constexpr int pair(int) { return -1; }
  __host__ __device__ static constexpr int plus_pos(int) { return -1; }
  __host__ __device__ static constexpr int first_pos(int q) { return q; }
  __host__ __device__ static constexpr int axis(int q) {
    constexpr int t[7] = {0, 1, 2, -1, 2, 1, 0};
    return t[q];
  }
  __host__ __device__ static constexpr int delta(int q) {
    constexpr int t[7] = {-1, -1, -1, 0, 1, 1, 1};
    return t[q];
  }
};

// Coefficient planes are read exactly once per sweep: stream them with an L2
// evict-first policy (and no L1 allocation) so they do not push the stencil input's
// neighbour rows (x, D^-1) out of L2.  Measured on B200: the 2D fine sweep gains
// (K1 44.1 -> 41.5 us, apply 26.5 -> 21.4 us); the 3D fine and the class-compressed
// coarse sweeps lose 3-20%, so only the 2D pair-compressed path uses it.
#ifndef HADR_COEF_EVICT_FIRST
#define HADR_COEF_EVICT_FIRST 1
#endif
__device__ __forceinline__ unsigned long long coef_policy() {
  unsigned long long pol = 0;
#if HADR_COEF_EVICT_FIRST
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
#endif
  return pol;
}
__device__ __forceinline__ cplx ld_stream(const cplx* p, unsigned long long pol) {
#if HADR_COEF_EVICT_FIRST
  cplx r;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(r.x), "=d"(r.y) : "l"(p), "l"(pol));
  return r;
#else
  (void)pol;
  return __ldg(p);
#endif
}

template <int NO, int INM, bool C32>
__device__ __forceinline__ void stencil_pc(const StencilArgs& a, long k, int i1, int i2, int i3, int n1, int n2,
                                           int n3, double s, unsigned code, cplx& acc) {
  // Branch-free: the slot geometry is compile-time (PcLayout, verified on the host by
  // Op::pair_compress), so every load is in one basic block and issues back to back.
  using Lay = PcLayout<NO>;
  constexpr int NS = Lay::NS;
  const unsigned long long pol = NO == 9 ? coef_policy() : 0ull;
  const int crd[3] = {i1, i2, i3};
  const int ext[3] = {n1, n2, n3};
  const long str[3] = {(long)n2 * n3, (long)n3, 1};
  cplx cv[NS], xv[NS], dv[NS];
  bool ok[NS];
  const long ps = a.A.pstr;
#pragma unroll
  for (int q = 0; q < NS; ++q) {
    const int ax = Lay::axis(q);
    int dl = Lay::delta(q);
    if (Lay::plus_pos(q) >= 0) dl = ((code >> Lay::pair(Lay::first_pos(q))) & 1u) ? 2 : -2;
    long jj = k;
    ok[q] = true;
    if (ax >= 0) {
      ok[q] = (unsigned)(crd[ax] + dl) < (unsigned)ext[ax];
      jj = ok[q] ? k + dl * str[ax] : k;  // owned-relative (slab halos at < 0)
    }
    if constexpr (C32) {
      const float2 c = __ldg(a.A.pcoef32 + (long)q * ps + k);
      cv[q] = make_double2((double)c.x, (double)c.y);
    } else {
      cv[q] = NO == 9 ? ld_stream(a.A.pcoef + (long)q * ps + k, pol) : ldc(a.A.pcoef, (long)q * ps + k);
    }
    xv[q] = ldc(a.x, jj);
    if (INM & IN_JAC) dv[q] = ldc(a.dinv, jj);
  }
  cplx tv[NS];
#pragma unroll
  for (int q = 0; q < NS; ++q) {
    cplx v = xv[q];
    if (INM & IN_SCALE) v = cscale(v, s);
    if (INM & IN_JAC) v = cmul_np(dv[q], v);
    tv[q] = cmul_sp(cv[q], v);
  }
#pragma unroll
  for (int p = 0; p < NO; ++p) {
    const int q = Lay::slot(p);
    bool live = ok[q];
    if (Lay::pair(p) >= 0) {
      const unsigned member = (Lay::plus_pos(q) == p) ? 1u : 0u;
      live = live && ((code >> Lay::pair(p)) & 1u) == member;
    }
    const cplx t = cadd(acc, tv[q]);
    acc = live ? t : acc;
  }
}

// Class-compressed coarse operator: slots of the row's class in ascending union order,
// chunks of CH slots, every load of a chunk independent (table -> coefficient, x, D^-1).
// Class-compressed coarse operator: the row's class slots in ascending union order, chunks
// of CH slots, every load of a chunk independent (table -> coefficient, x, D^-1).
template <int CH, int INM, bool C32>
__device__ __forceinline__ void stencil_cc(const StencilArgs& a, int cls, int nslc, long k, int i1, int i2, int i3,
                                           int n1, int n2, int n3, double s, cplx& acc) {
  // warp-uniform trip count (the warp's largest class); slots past a row's own class are dead
  const int nsw = __reduce_max_sync(__activemask(), (unsigned)nslc);
  const long cs = a.A.cstr;
  const int4* tab = a.A.ctab + (long)cls * a.A.nsl;
  for (int q0 = 0; q0 < nsw; q0 += CH) {
    int4 t[CH];
#pragma unroll
    for (int q = 0; q < CH; ++q) t[q] = __ldg(tab + (q0 + q < nslc ? q0 + q : 0));
    cplx cv[CH], xv[CH], dv[CH];
    bool ok[CH];
#pragma unroll
    for (int q = 0; q < CH; ++q) {
      const bool live = q0 + q < nslc;
      const int j1 = i1 + t[q].y, j2 = i2 + t[q].z, j3 = i3 + t[q].w;
      ok[q] = live && j1 >= 0 && j1 < n1 && j2 >= 0 && j2 < n2 && j3 >= 0 && j3 < n3;
      const long jj = ok[q] ? k + t[q].x : k;
      const long ci = (long)(live ? q0 + q : 0) * cs + k;
      if constexpr (C32) {
        const float2 c = __ldg(a.A.ccoef32 + ci);
        cv[q] = make_double2((double)c.x, (double)c.y);
      } else {
        cv[q] = ldc(a.A.ccoef, ci);
      }
      xv[q] = ldc(a.x, jj);
      if (INM & IN_JAC) dv[q] = ldc(a.dinv, jj);
    }
#pragma unroll
    for (int q = 0; q < CH; ++q) {
      cplx v = xv[q];
      if (INM & IN_SCALE) v = cscale(v, s);
      if (INM & IN_JAC) v = cmul_np(dv[q], v);
      const cplx tt = cadd(acc, cmul_sp(cv[q], v));
      acc = ok[q] ? tt : acc;
    }
  }
}

// Resident CTAs per SM: the pair-compressed relaxation variant (IN_JAC: 21 loads per
// point in 2D) gets 128 registers so all of a point's loads issue back to back
// (B200, 1025^2 fine sweep: 50.6 us union / 44.1 us at 4 CTAs / 41.4 us at 2 CTAs);
// plain applies keep 4 CTAs (26.3 us vs 30.6 us at 2).
// (the class-compressed kernel measured fastest at 4 CTAs/SM in every variant)
// Class-compressed chunk (slots whose loads are issued together): measured on B200 at
// 4 CTAs/SM, the Jacobi variant (coefficient, x, D^-1 per slot) is fastest at 9, the
// plain apply (coefficient, x) at 6 (3D level-2 apply 1524 -> 1309 us); 3 CTAs/SM and
// chunks of 12 were slower in every variant.
template <int INM>
__host__ __device__ constexpr int cc_chunk() {
  return (INM & IN_JAC) ? 9 : 6;
}
template <int INM, bool PC, bool CC>
constexpr int stencil_min_blocks() {
  return (PC && (INM & IN_JAC)) ? 2 : 4;
}
template <int INM, int OUTM, int RED, int NO, int CL, bool PC = false, bool CC = false>
__global__ void __launch_bounds__(kThreads, stencil_min_blocks<INM, PC, CC>()) k_stencil(StencilArgs a) {
  pdl_enter();
  if (!gate_open(a.gate)) return;
  const int n1 = a.A.n1, n2 = a.A.n2, n3 = a.A.n3, nofs = a.A.nofs;
  const int n23 = n2 * n3;
  const long N = a.A.pstride;                    // coefficient plane stride
  const long Nown = (long)a.A.n1own * n23;       // points computed (owned slab)
  const int p0 = a.A.p0;
  const double s = (INM & IN_SCALE) ? *a.scale : 1.0;
  const bool c32 = a.A.coef32 != nullptr;
  constexpr int NV = ((RED & RED_NORM) ? 1 : 0) + ((RED & (RED_DOT | RED_DOT_CENTER)) ? 2 : 0);
  double red[NV > 0 ? NV : 1];
#pragma unroll
  for (int q = 0; q < (NV > 0 ? NV : 1); ++q) red[q] = 0.0;
  const long stride = (long)gridDim.x * blockDim.x;
  for (long k = (long)blockIdx.x * blockDim.x + threadIdx.x; k < Nown; k += stride) {
    const int il = (int)(k / n23);
    const int i1 = il + p0;  // global plane
    const int rem = (int)(k - (long)il * n23);
    const int i2 = rem / n3;
    const int i3 = rem - i2 * n3;
    cplx acc = mk(0.0, 0.0);
    // the point's own streams (centre, residual rhs, dot partner) are loaded up front with
    // the stencil's loads rather than after the accumulation (one memory round trip less)
    cplx xc = mk(0.0, 0.0), bk = mk(0.0, 0.0), uk = mk(0.0, 0.0);
    if ((INM & IN_WRITEV) || (RED & RED_DOT_CENTER)) xc = ldc(a.x, k);
    if (OUTM == OUT_RESID) bk = ldc(a.b, k);
    if (RED & RED_DOT) uk = ldc(a.u, k);
    if constexpr (PC) {
      const unsigned code = __ldg(a.A.pcode + k);
      if (a.A.pcoef32)
        stencil_pc<NO, INM, true>(a, k, i1, i2, i3, n1, n2, n3, s, code, acc);
      else
        stencil_pc<NO, INM, false>(a, k, i1, i2, i3, n1, n2, n3, s, code, acc);
    } else if constexpr (CC) {
      const unsigned cw = __ldg(a.A.ccode + k);
      const int cls = (int)(cw & 0xFFu);
      if (a.A.ccoef32)
        stencil_cc<cc_chunk<INM>(), INM, true>(a, cls, (int)(cw >> 8), k, i1, i2, i3, n1, n2, n3, s, acc);
      else
        stencil_cc<cc_chunk<INM>(), INM, false>(a, cls, (int)(cw >> 8), k, i1, i2, i3, n1, n2, n3, s, acc);
    } else if constexpr (NO > 0) {
      if (c32)
        stencil_chunk<NO, INM, true>(a, 0, nofs, k, i1, i2, i3, n1, n2, n3, N, s, acc);
      else
        stencil_chunk<NO, INM, false>(a, 0, nofs, k, i1, i2, i3, n1, n2, n3, N, s, acc);
    } else {
      for (int o0 = 0; o0 < nofs; o0 += 9) {
        if (c32)
          stencil_chunk<9, INM, true>(a, o0, nofs, k, i1, i2, i3, n1, n2, n3, N, s, acc);
        else
          stencil_chunk<9, INM, false>(a, o0, nofs, k, i1, i2, i3, n1, n2, n3, N, s, acc);
      }
    }
    cplx vc = mk(0.0, 0.0);
    if ((INM & IN_WRITEV) || (RED & RED_DOT_CENTER)) {
      vc = xc;
      if (INM & IN_SCALE) vc = cscale(vc, s);
      if (INM & IN_WRITEV) a.vout[k] = vc;
    }
    cplx y = (OUTM == OUT_RESID) ? csub(bk, acc) : acc;
    a.y[k] = y;
    if (RED & RED_NORM) red[0] += y.x * y.x + y.y * y.y;
    if (RED & (RED_DOT | RED_DOT_CENTER)) {
      const cplx u = (RED & RED_DOT_CENTER) ? vc : uk;
      constexpr int o = (RED & RED_NORM) ? 1 : 0;
      red[o] += u.x * y.x + u.y * y.y;
      red[o + 1] += u.x * y.y - u.y * y.x;
    }
  }
  if constexpr (NV > 0) {
    double v[NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) v[q] = red[q];
    finish<NV, CL>(v, a.rs, a.epi);
  }
}

// ---------------------------------------------------------------------------
// K1 tiled: the same stencil with the (transformed) input staged in shared memory.
// A block owns a tile of tp planes x ty rows x tx columns (3D: 2 x 4 x 32, 2D:
// 8 x 32) and stages it with a 2-point halo on every stencilled axis, applying
// the scale / D^-1 transform once per staged point.  Neighbour reads are LDS;
// the coefficient planes stream from HBM exactly once.  Arithmetic and
// accumulation order are identical to k_stencil (bit-identical outputs).
// ---------------------------------------------------------------------------
struct TileCfg {
  int tp, ty, tx, hy;    // tile extents, halo rows (2 in 3D, 0 in 2D)
  int ntp, nty, ntx;     // tile counts per axis
};

template <int CH, bool C32>
__device__ __forceinline__ void tile_chunk(const StencilArgs& a, const cplx* tl, int o0, int nofs, long k, int i1,
                                           int i2, int i3, int n1, int n2, int n3, long N, int tidx, int sP, int sY,
                                           bool d3, cplx& acc) {
  cplx cv[CH];
  int ti[CH];
  bool ok[CH];
#pragma unroll
  for (int q = 0; q < CH; ++q) {
    const int o = o0 + q;
    const bool live = o < nofs;
    const int oo = live ? o : 0;
    const int d1 = a.A.d1[oo], d2 = a.A.d2[oo], dd3 = a.A.d3[oo];
    const int j1 = i1 + d1, j2 = i2 + d2, j3 = i3 + dd3;
    ok[q] = live && j1 >= 0 && j1 < n1 && j2 >= 0 && j2 < n2 && j3 >= 0 && j3 < n3;
    ti[q] = ok[q] ? tidx + d1 * sP + (d3 ? d2 * sY + dd3 : d2) : tidx;
    cv[q] = C32 ? ld_c64(a.A, live ? (long)o * N + k : k) : ldc(a.A.coef, live ? (long)o * N + k : k);
  }
#pragma unroll
  for (int q = 0; q < CH; ++q) {
    const cplx t = cadd(acc, cmul_sp(cv[q], tl[ti[q]]));
    acc = ok[q] ? t : acc;
  }
}

template <int INM, int OUTM, int RED, int NO>
__global__ void __launch_bounds__(kThreads, 4) k_stencil_tile(StencilArgs a, TileCfg t) {
  pdl_enter();
  if (!gate_open(a.gate)) return;
  extern __shared__ cplx tl[];
  const int n1 = a.A.n1, n2 = a.A.n2, n3 = a.A.n3, nofs = a.A.nofs;
  const long N = a.A.pstride;
  const int n1own = a.A.n1own, p0 = a.A.p0;
  const bool d3 = n3 > 1;
  const int nY = d3 ? n2 : 1, nX = d3 ? n3 : n2;
  const double s = (INM & IN_SCALE) ? *a.scale : 1.0;
  const bool c32 = a.A.coef32 != nullptr;
  const int sY = t.tx + 4, sP = (t.ty + 2 * t.hy) * sY, tsize = (t.tp + 4) * sP;
  const long ntiles = (long)t.ntp * t.nty * t.ntx;
  const int px = threadIdx.x % t.tx, py = (threadIdx.x / t.tx) % t.ty, pp = threadIdx.x / (t.tx * t.ty);
  constexpr int NV = ((RED & RED_NORM) ? 1 : 0) + ((RED & (RED_DOT | RED_DOT_CENTER)) ? 2 : 0);
  double red[NV > 0 ? NV : 1];
#pragma unroll
  for (int q = 0; q < (NV > 0 ? NV : 1); ++q) red[q] = 0.0;
  for (long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int bx = (int)(tile % t.ntx), by = (int)((tile / t.ntx) % t.nty), bp = (int)(tile / ((long)t.ntx * t.nty));
    const int P0 = bp * t.tp, Y0 = by * t.ty, X0 = bx * t.tx;
    for (int e = threadIdx.x; e < tsize; e += blockDim.x) {
      const int ep = e / sP, r = e - ep * sP, ey = r / sY, ex = r - ey * sY;
      const int gp = P0 - 2 + ep, gy = Y0 - t.hy + ey, gx = X0 - 2 + ex;
      cplx v = mk(0.0, 0.0);
      if (gp + p0 >= 0 && gp + p0 < n1 && gp < n1own + 2 && gy >= 0 && gy < nY && gx >= 0 && gx < nX) {
        const long kk = ((long)gp * nY + gy) * nX + gx;
        v = ldc(a.x, kk);
        if (INM & IN_SCALE) v = cscale(v, s);
        if (INM & IN_JAC) v = cmul_np(ldc(a.dinv, kk), v);
      }
      tl[e] = v;
    }
    __syncthreads();
    const int il = P0 + pp, y = Y0 + py, x = X0 + px;
    if (pp < t.tp && il < n1own && y < nY && x < nX) {
      const long k = ((long)il * nY + y) * nX + x;
      const int i1 = il + p0, i2 = d3 ? y : x, i3 = d3 ? x : 0;
      const int tidx = (pp + 2) * sP + (py + t.hy) * sY + (px + 2);
      cplx acc = mk(0.0, 0.0);
      cplx xc = mk(0.0, 0.0), bk = mk(0.0, 0.0), uk = mk(0.0, 0.0);  // issued with the stencil's loads
      if ((INM & IN_WRITEV) || (RED & RED_DOT_CENTER)) xc = ldc(a.x, k);
      if (OUTM == OUT_RESID) bk = ldc(a.b, k);
      if (RED & RED_DOT) uk = ldc(a.u, k);
      if constexpr (NO > 0) {
        if (c32)
          tile_chunk<NO, true>(a, tl, 0, nofs, k, i1, i2, i3, n1, n2, n3, N, tidx, sP, sY, d3, acc);
        else
          tile_chunk<NO, false>(a, tl, 0, nofs, k, i1, i2, i3, n1, n2, n3, N, tidx, sP, sY, d3, acc);
      } else {
        for (int o0 = 0; o0 < nofs; o0 += 9) {
          if (c32)
            tile_chunk<9, true>(a, tl, o0, nofs, k, i1, i2, i3, n1, n2, n3, N, tidx, sP, sY, d3, acc);
          else
            tile_chunk<9, false>(a, tl, o0, nofs, k, i1, i2, i3, n1, n2, n3, N, tidx, sP, sY, d3, acc);
        }
      }
      cplx vc = mk(0.0, 0.0);
      if ((INM & IN_WRITEV) || (RED & RED_DOT_CENTER)) {
        vc = xc;
        if (INM & IN_SCALE) vc = cscale(vc, s);
        if (INM & IN_WRITEV) a.vout[k] = vc;
      }
      cplx yv = (OUTM == OUT_RESID) ? csub(bk, acc) : acc;
      a.y[k] = yv;
      if (RED & RED_NORM) red[0] += yv.x * yv.x + yv.y * yv.y;
      if (RED & (RED_DOT | RED_DOT_CENTER)) {
        const cplx u = (RED & RED_DOT_CENTER) ? vc : uk;
        constexpr int o = (RED & RED_NORM) ? 1 : 0;
        red[o] += u.x * yv.x + u.y * yv.y;
        red[o + 1] += u.x * yv.y - u.y * yv.x;
      }
    }
    __syncthreads();  // the tile is restaged for the next tile
  }
  if constexpr (NV > 0) {
    double v[NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) v[q] = red[q];
    finish<NV, 0>(v, a.rs, a.epi);
  }
}


// ---------------------------------------------------------------------------
// K1 marching (3D fine levels: the pair-compressed plus-radius-2 operator — 13 offsets, 10 slot
// planes — and the 7-point plus of radius 1 from its union planes; every variant of K1: plain
// input or the relaxation's D^-1 (s x) from a second ring of D^-1 tiles, apply / residual,
// fused dot / norm; a 2D instantiation marches a grid row by row):
// a block owns a column tile of ty x tx points of the (axis 1, axis 2) plane and
// marches along axis 0 through a chunk of planes.  The input's plane tiles (2-point
// halo on axes 1 and 2) land in a ring of 6 shared-memory slots by row-wise bulk
// asynchronous copies (cp.async.bulk -> UBLKCP; one "full" mbarrier per slot counts the
// bytes), issued by a dedicated producer warp that runs ahead of the arithmetic as far
// as the ring allows; the compute warps hand a slot back through its "empty" mbarrier
// (one arrival per warp), so there is no block-wide barrier in the loop.  Every input
// element comes from DRAM once per sweep (plus the tile halo, ~1.4x of 16 of the ~210 B
// per point) instead of once per axis-0 neighbour plane that has left L2 (ncu: 20.2 GB
// per 513^2 x 257 sweep for the flat kernel, 15.2 GB here; layout 14.1 GB).  The ten
// coefficient planes stream from HBM straight into registers, once.  Arithmetic and
// accumulation order are stencil_pc's: bit-identical outputs.
// ---------------------------------------------------------------------------
struct MarchCfg {
  int nty, ntx, nch;  // tiles along axis 1 / axis 2, chunks of planes
  int pc;             // planes per chunk
  int pitch, slot;    // shared-memory row pitch and slot size (elements)
  int hy;             // halo rows of a slot along axis 1 (3D: 2; 2D, where a plane is one grid row: 0)
};
#ifndef HADR_MARCH_THREADS
#define HADR_MARCH_THREADS 480  // compute threads (one point of the tile each); + 1 producer warp
#endif
#ifndef HADR_MARCH_PPT
#define HADR_MARCH_PPT 1
#endif
#ifndef HADR_MARCH_MIN_BLOCKS
#define HADR_MARCH_MIN_BLOCKS 1
#endif
constexpr int kMarchRing = 6;
constexpr int kMarchPpt = HADR_MARCH_PPT;
constexpr int kMarchThreads = HADR_MARCH_THREADS;
constexpr int kMarchBlock = kMarchThreads + 32;
constexpr int kMarchWarps = kMarchThreads / 32;

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
  unsigned done;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void bulk_g2s(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

// NO = 13: 3D (planes along axis 0, tiles over axes 1 x 2).  NO = 9: 2D — the grid (n1, n2) is marched as
// (n1, 1, n2): a plane is one grid row, a tile a row segment of up to one point per compute thread.
template <int NO, int INM, int OUTM, int RED, bool C32>
__global__ void __launch_bounds__(kMarchBlock, HADR_MARCH_MIN_BLOCKS) k_stencil_march(StencilArgs a, MarchCfg m) {
  pdl_enter();
  if (!gate_open(a.gate)) return;
  extern __shared__ __align__(128) unsigned char march_smem[];
  __shared__ __align__(8) unsigned long long full[kMarchRing], empty[kMarchRing];
  cplx* ring = reinterpret_cast<cplx*>(march_smem);
  // relaxation input (IN_JAC): D^-1 tiles in a second ring, the transform D^-1 (.) (s x) applied per read
  constexpr bool JAC = (INM & IN_JAC) != 0;
  const long dofs = (long)kMarchRing * m.slot;  // D^-1 ring offset (elements)
  using Lay = PcLayout<NO>;
  constexpr int NS = Lay::NS;
  constexpr bool D2 = NO == 9;
  constexpr int NV = ((RED & RED_NORM) ? 1 : 0) + ((RED & (RED_DOT | RED_DOT_CENTER)) ? 2 : 0);
  const int n1 = a.A.n1, n2 = D2 ? 1 : a.A.n2, n3 = D2 ? a.A.n2 : a.A.n3, n1own = a.A.n1own, p0 = a.A.p0;
  const long n23 = (long)n2 * n3;
  int item = blockIdx.x;
  const int bx = item % m.ntx;
  item /= m.ntx;
  const int by = item % m.nty;
  const int bc = item / m.nty;
  const int Y0 = (int)((long)by * n2 / m.nty), Y1 = (int)((long)(by + 1) * n2 / m.nty);
  const int X0 = (int)((long)bx * n3 / m.ntx), X1 = (int)((long)(bx + 1) * n3 / m.ntx);
  const int P0 = bc * m.pc, P1 = (P0 + m.pc < n1own) ? P0 + m.pc : n1own;
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < kMarchRing; ++s) {
      mbar_init(smem_u32(&full[s]), 1u);
      mbar_init(smem_u32(&empty[s]), (unsigned)kMarchWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  double red[NV > 0 ? NV : 1];
#pragma unroll
  for (int q = 0; q < (NV > 0 ? NV : 1); ++q) red[q] = 0.0;
  if (wid == kMarchWarps) {
    // ---- producer warp: plane q (owned-relative; halo planes at q < 0 and q >= n1own) -> slot
    // (q - (P0 - 2)) % ring; a slot's barriers complete one phase per plane it carries ----
    const int ys = Y0 - m.hy > 0 ? Y0 - m.hy : 0, ye = Y1 + m.hy < n2 ? Y1 + m.hy : n2;
    const int xs = X0 - 2 > 0 ? X0 - 2 : 0, xe = X1 + 2 < n3 ? X1 + 2 : n3;
    const int nrows = ye - ys;
    const unsigned rowbytes = (unsigned)(xe - xs) * (unsigned)sizeof(cplx);
    for (int q = P0 - 2; q <= P1 + 1; ++q) {
      const int r = q - (P0 - 2), s = r % kMarchRing, use = r / kMarchRing;
      if (use > 0) mbar_wait(smem_u32(&empty[s]), (unsigned)(use - 1) & 1u);  // the compute warps left the slot
      const bool valid = q + p0 >= 0 && q + p0 < n1;
      const unsigned bar = smem_u32(&full[s]);
      if (lane == 0) {
        if (valid)
          mbar_expect_tx(bar, (unsigned)nrows * rowbytes * (JAC ? 2u : 1u));
        else
          mbar_arrive(bar);
      }
      __syncwarp();
      if (valid) {
        const cplx* src = a.x + (long)q * n23 + xs;
        const unsigned dst = smem_u32(ring + (long)s * m.slot + (xs - (X0 - 2)));
        for (int rr = lane; rr < nrows; rr += 32)
          bulk_g2s(dst + (unsigned)((ys + rr - (Y0 - m.hy)) * m.pitch) * (unsigned)sizeof(cplx),
                   src + (long)(ys + rr) * n3, rowbytes, bar);
        if constexpr (JAC) {
          const cplx* dsrc = a.dinv + (long)q * n23 + xs;
          const unsigned ddst = dst + (unsigned)dofs * (unsigned)sizeof(cplx);
          for (int rr = lane; rr < nrows; rr += 32)
            bulk_g2s(ddst + (unsigned)((ys + rr - (Y0 - m.hy)) * m.pitch) * (unsigned)sizeof(cplx),
                     dsrc + (long)(ys + rr) * n3, rowbytes, bar);
        }
      }
    }
  } else {
    // ---- compute warps ----
    constexpr bool UNION = NO == 7;  // the 7-point operator streams its union planes (nothing to compress)
    const long ps = UNION ? a.A.pstride : a.A.pstr;
    const double sc = (INM & IN_SCALE) ? *a.scale : 1.0;
    const int ty = Y1 - Y0, tx = X1 - X0;
    int sidx[kMarchPpt];
    int krel[kMarchPpt];
    bool act[kMarchPpt];
    unsigned okm[kMarchPpt];  // bit (axis - 1) * 5 + (delta + 2): in-grid neighbour along axes 1, 2
#pragma unroll
    for (int t = 0; t < kMarchPpt; ++t) {
      const int e = threadIdx.x + t * kMarchThreads;
      act[t] = e < ty * tx;
      const int py = act[t] ? e / tx : 0, px = act[t] ? e - py * tx : 0;
      const int i2 = Y0 + py, i3 = X0 + px;
      sidx[t] = (py + m.hy) * m.pitch + (px + 2);
      krel[t] = i2 * n3 + i3;
      unsigned mk_ = 0;
#pragma unroll
      for (int d = -2; d <= 2; ++d) {
        if ((unsigned)(i2 + d) < (unsigned)n2) mk_ |= 1u << (d + 2);
        if ((unsigned)(i3 + d) < (unsigned)n3) mk_ |= 1u << (5 + d + 2);
      }
      okm[t] = mk_;
    }
    for (int r = 0; r < 4; ++r) mbar_wait(smem_u32(&full[r]), 0u);  // planes P0 - 2 .. P0 + 1
    for (int p = P0; p < P1; ++p) {
      // the unit's global loads (10 coefficients, pair code, rhs / dot partner) go out first
      cplx cv[kMarchPpt][NS], bk[kMarchPpt], uk[kMarchPpt];
      unsigned code[kMarchPpt];
#pragma unroll
      for (int t = 0; t < kMarchPpt; ++t) {
        if (!act[t]) continue;
        const long k = (long)p * n23 + krel[t];
        code[t] = UNION ? 0u : (unsigned)__ldg(a.A.pcode + k);
#pragma unroll
        for (int q = 0; q < NS; ++q) {
          if constexpr (C32) {
            const float2 c = __ldg((UNION ? a.A.coef32 : a.A.pcoef32) + (long)q * ps + k);
            cv[t][q] = make_double2((double)c.x, (double)c.y);
          } else {
            cv[t][q] = ldc(UNION ? a.A.coef : a.A.pcoef, (long)q * ps + k);
          }
        }
        if (OUTM == OUT_RESID) bk[t] = ldc(a.b, k);
        if (RED & RED_DOT) uk[t] = ldc(a.u, k);
      }
      const int r2 = p - P0 + 4;  // plane p + 2
      mbar_wait(smem_u32(&full[r2 % kMarchRing]), (unsigned)(r2 / kMarchRing) & 1u);
      const cplx* pl[5];  // slots of planes p - 2 .. p + 2
#pragma unroll
      for (int d = 0; d < 5; ++d) pl[d] = ring + (long)((p - P0 + d) % kMarchRing) * m.slot;
      unsigned ok0 = 0;  // bit (delta + 2): in-grid plane along axis 0
#pragma unroll
      for (int d = -2; d <= 2; ++d)
        if ((unsigned)(p + p0 + d) < (unsigned)n1) ok0 |= 1u << (d + 2);
#pragma unroll
      for (int t = 0; t < kMarchPpt; ++t) {
        if (!act[t]) continue;
        const long k = (long)p * n23 + krel[t];
        cplx tv[NS];
        bool ok[NS];
        cplx xc[kMarchPpt];  // the centre's raw input
#pragma unroll
        for (int q = 0; q < NS; ++q) {
          const int ax = (D2 && Lay::axis(q) == 1) ? 2 : Lay::axis(q);  // 2D: the in-row axis is the tile's x
          int dl = Lay::delta(q);
          if (Lay::plus_pos(q) >= 0) dl = ((code[t] >> Lay::pair(Lay::first_pos(q))) & 1u) ? 2 : -2;
          const cplx* src;
          if (ax < 0) {
            ok[q] = true;
            src = pl[2] + sidx[t];
          } else if (ax == 0) {
            ok[q] = (ok0 >> (dl + 2)) & 1u;
            // (a select between the two candidate slots, not a runtime index into pl[])
            src = (Lay::plus_pos(q) >= 0 ? (dl > 0 ? pl[4] : pl[0]) : pl[Lay::delta(q) + 2]) + sidx[t];
          } else if (ax == 1) {
            ok[q] = (okm[t] >> (dl + 2)) & 1u;
            src = pl[2] + sidx[t] + dl * m.pitch;
          } else {
            ok[q] = (okm[t] >> (5 + dl + 2)) & 1u;
            src = pl[2] + sidx[t] + dl;
          }
          cplx v = *src;
          if (INM & IN_SCALE) v = cscale(v, sc);
          if constexpr (JAC) v = cmul_np(src[dofs], v);
          if (ax < 0) xc[t] = *src;
          tv[q] = cmul_sp(cv[t][q], v);
        }
        cplx acc = mk(0.0, 0.0);
#pragma unroll
        for (int pp = 0; pp < NO; ++pp) {
          const int q = Lay::slot(pp);
          bool live = ok[q];
          if (Lay::pair(pp) >= 0) {
            const unsigned member = (Lay::plus_pos(q) == pp) ? 1u : 0u;
            live = live && ((code[t] >> Lay::pair(pp)) & 1u) == member;
          }
          const cplx tt = cadd(acc, tv[q]);
          acc = live ? tt : acc;
        }
        cplx vc = mk(0.0, 0.0);
        if ((INM & IN_WRITEV) || (RED & RED_DOT_CENTER)) {
          vc = xc[t];
          if (INM & IN_SCALE) vc = cscale(vc, sc);
          if (INM & IN_WRITEV) a.vout[k] = vc;
        }
        const cplx y = (OUTM == OUT_RESID) ? csub(bk[t], acc) : acc;
        a.y[k] = y;
        if (RED & RED_NORM) red[0] += y.x * y.x + y.y * y.y;
        if (RED & (RED_DOT | RED_DOT_CENTER)) {
          const cplx u = (RED & RED_DOT_CENTER) ? vc : uk[t];
          constexpr int o = (RED & RED_NORM) ? 1 : 0;
          red[o] += u.x * y.x + u.y * y.y;
          red[o + 1] += u.x * y.y - u.y * y.x;
        }
      }
      __syncwarp();  // every lane's reads of plane p - 2 are done: hand its slot back
      if (lane == 0) mbar_arrive(smem_u32(&empty[(p - P0) % kMarchRing]));
    }
  }
  if constexpr (NV > 0) {
    double v[NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) v[q] = red[q];
    finish<NV, 0>(v, a.rs, a.epi);
  }
}

int g_stencil_march = 1;          // option "stencil_march": 0 off, 1 policy (large fine levels), 2 always
long g_march_min_n = 2000000;     // option "march_min_n": policy threshold, 3D (owned points)
long g_march_min_n2d = 1L << 40;  // option "march_min_n2d": policy threshold, 2D

// the marching kernel's policy: a pair-compressed plus-radius-2 operator (3D 13 / 2D 9 offsets) of at least
// march_min_n / march_min_n2d owned points
static bool is_plus1_3d(const StencilDev& A) {  // exactly the 3D plus of radius 1, in PcLayout<7>'s order
  if (A.nofs != 7 || A.n3 < 2) return false;
  using Lay = PcLayout<7>;
  for (int q = 0; q < 7; ++q) {
    const int d[3] = {A.d1[q], A.d2[q], A.d3[q]};
    for (int ax = 0; ax < 3; ++ax)
      if (d[ax] != (Lay::axis(q) == ax ? Lay::delta(q) : 0)) return false;
  }
  return true;
}

bool march_takes(const StencilDev& A) {
  if (!g_stencil_march) return false;
  const bool d7 = is_plus1_3d(A);
  const bool d3 = (A.pcode && A.nofs == 13 && A.n3 >= 2) || d7, d2 = A.pcode && A.nofs == 9 && A.n3 == 1;
  if (!d3 && !d2) return false;
  return g_stencil_march > 1 || (long)A.n1own * A.n2 * A.n3 >= (d3 ? g_march_min_n : g_march_min_n2d);
}

// Tiling of the marching kernel (host logic; hadr_march_plan exposes it to the CPU tests): the
// (axis 1, axis 2) plane in nty x ntx near-equal tiles of at most one point per compute thread,
// axis 0 in nch chunks of pc planes.  d3 = false: a 2D grid marched as (n1, 1, n2).
static bool march_dims(bool d3, int n1own, int nY, int nX, bool jac, MarchCfg& m, int& blocks, size_t& smem) {
  if (n1own < 1 || nY < 1 || nX < 1) return false;
  const int txcap = d3 ? 34 : kMarchThreads * kMarchPpt;
  m.hy = d3 ? 2 : 0;
  m.ntx = (nX + txcap - 1) / txcap;
  const int txmax = (nX + m.ntx - 1) / m.ntx;
  int tymax = (kMarchThreads * kMarchPpt) / txmax;
  if (tymax > nY) tymax = nY;
  m.nty = (nY + tymax - 1) / tymax;
  tymax = (nY + m.nty - 1) / m.nty;
  const long cols = (long)m.ntx * m.nty;
  long nch = (148L * HADR_MARCH_MIN_BLOCKS * 4 + cols - 1) / cols;  // >= 4 waves of blocks
  if (nch > n1own / 8) nch = n1own / 8;                              // chunks of >= 8 planes
  if (nch < 1) nch = 1;
  if (cols * nch > 8192) nch = 8192 / cols;                          // reduction scratch: 8192 blocks
  if (nch < 1) return false;
  m.pc = (int)((n1own + nch - 1) / nch);
  m.nch = (n1own + m.pc - 1) / m.pc;
  m.pitch = txmax + 4;
  m.slot = (tymax + 2 * m.hy) * m.pitch;
  blocks = (int)(cols * m.nch);
  smem = (size_t)kMarchRing * m.slot * sizeof(cplx) * (jac ? 2 : 1);
  return smem <= 200 * 1024;
}

static bool march_cfg(const StencilDev& A, bool jac, MarchCfg& m, int& blocks, size_t& smem) {
  const bool d3 = (A.pcode && A.nofs == 13 && A.n3 >= 2) || is_plus1_3d(A), d2 = A.pcode && A.nofs == 9 && A.n3 == 1;
  if (!d3 && !d2) return false;
  return march_dims(d3, A.n1own, d3 ? A.n2 : 1, d3 ? A.n3 : A.n2, jac, m, blocks, smem);
}

bool march_plan(int n1own, int n2, int n3, int jac, int* out) {
  MarchCfg m{};
  int blocks = 0;
  size_t smem = 0;
  const bool d3 = n3 > 1;
  if (!march_dims(d3, n1own, d3 ? n2 : 1, d3 ? n3 : n2, jac != 0, m, blocks, smem)) return false;
  const int v[10] = {m.nty, m.ntx, m.nch, m.pc, m.pitch, m.slot, m.hy, blocks, (int)smem, kMarchThreads * kMarchPpt};
  for (int i = 0; i < 10; ++i) out[i] = v[i];
  return true;
}

template <int NO, int INM, int OUTM, int RED, bool C32>
static void launch_march_t(const LaunchCfg& lc, const StencilArgs& a, const MarchCfg& m, int blocks, size_t smem) {
  static size_t enabled = 0;
  if (smem > enabled) {
    cudaFuncSetAttribute(k_stencil_march<NO, INM, OUTM, RED, C32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    enabled = smem;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(kMarchBlock);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = lc.stream;
  cudaLaunchAttribute at[1];
  cfg.numAttrs = pdl_attr(at);
  cfg.attrs = at;
  cudaLaunchKernelEx(&cfg, k_stencil_march<NO, INM, OUTM, RED, C32>, a, m);
  constexpr int NV = ((RED & RED_NORM) ? 1 : 0) + ((RED & (RED_DOT | RED_DOT_CENTER)) ? 2 : 0);
  if constexpr (NV > 0) launch_finalize<NV>(lc, Geo{blocks, 0}, a.gate, a.rs, a.epi);
}

// true when the marching kernel took the launch
static bool launch_march(const LaunchCfg& lc, int inm, int outm, int red, const StencilArgs& a) {
  MarchCfg m{};
  int blocks = 0;
  size_t smem = 0;
  if (!march_cfg(a.A, (inm & IN_JAC) != 0, m, blocks, smem)) return false;
  const bool c32 = a.A.nofs == 7 ? a.A.coef32 != nullptr : a.A.pcoef32 != nullptr;
  constexpr int J = IN_SCALE | IN_JAC | IN_WRITEV;
#define HADR_MCASE(I, O, R)                                      \
  if (inm == (I) && outm == (O) && red == (R)) {                 \
    if (a.A.nofs == 13) {                                        \
      if (c32)                                                   \
        launch_march_t<13, I, O, R, true>(lc, a, m, blocks, smem);  \
      else                                                       \
        launch_march_t<13, I, O, R, false>(lc, a, m, blocks, smem); \
    } else if (a.A.nofs == 7) {                                  \
      if (c32)                                                   \
        launch_march_t<7, I, O, R, true>(lc, a, m, blocks, smem);   \
      else                                                       \
        launch_march_t<7, I, O, R, false>(lc, a, m, blocks, smem);  \
    } else {                                                     \
      if (c32)                                                   \
        launch_march_t<9, I, O, R, true>(lc, a, m, blocks, smem);   \
      else                                                       \
        launch_march_t<9, I, O, R, false>(lc, a, m, blocks, smem);  \
    }                                                            \
    return true;                                                 \
  }
  HADR_MCASE(IN_PLAIN, OUT_APPLY, RED_NONE)
  HADR_MCASE(IN_PLAIN, OUT_APPLY, RED_NORM | RED_DOT)
  HADR_MCASE(IN_PLAIN, OUT_APPLY, RED_DOT)
  HADR_MCASE(IN_PLAIN, OUT_RESID, RED_NONE)
  HADR_MCASE(IN_PLAIN, OUT_RESID, RED_NORM)
  HADR_MCASE(J, OUT_APPLY, RED_DOT_CENTER)
  HADR_MCASE(J, OUT_APPLY, RED_DOT)
#undef HADR_MCASE
  return false;
}

int g_stencil_tile = 1;  // option "stencil_tile": 0 off, 1 policy (2D wide stencils), 2 always

template <int INM, int OUTM, int RED, int NO>
static void launch_tile_no(const LaunchCfg& lc, const StencilArgs& a, const TileCfg& t, int blocks) {
  const size_t smem = (size_t)(t.tp + 4) * (t.ty + 2 * t.hy) * (t.tx + 4) * sizeof(cplx);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = lc.stream;
  cudaLaunchAttribute at[1];
  cfg.numAttrs = pdl_attr(at);
  cfg.attrs = at;
  cudaLaunchKernelEx(&cfg, k_stencil_tile<INM, OUTM, RED, NO>, a, t);
}

template <int INM, int OUTM, int RED>
static void dispatch_tile(const LaunchCfg& lc, const StencilArgs& a, const TileCfg& t, int blocks) {
  const int n = a.A.nofs;
  if (n == 5)
    launch_tile_no<INM, OUTM, RED, 5>(lc, a, t, blocks);
  else if (n == 9)
    launch_tile_no<INM, OUTM, RED, 9>(lc, a, t, blocks);
  else if (n == 21)
    launch_tile_no<INM, OUTM, RED, 21>(lc, a, t, blocks);
  else if (n <= 7)
    launch_tile_no<INM, OUTM, RED, 7>(lc, a, t, blocks);
  else if (n <= 13)
    launch_tile_no<INM, OUTM, RED, 13>(lc, a, t, blocks);
  else if (n <= 25)
    launch_tile_no<INM, OUTM, RED, 25>(lc, a, t, blocks);
  else
    launch_tile_no<INM, OUTM, RED, 0>(lc, a, t, blocks);
  constexpr int NV = ((RED & RED_NORM) ? 1 : 0) + ((RED & (RED_DOT | RED_DOT_CENTER)) ? 2 : 0);
  if constexpr (NV > 0) launch_finalize<NV>(lc, Geo{blocks, 0}, a.gate, a.rs, a.epi);
}

template <int INM, int OUTM, int RED, int NO>
static void launch_stencil_no(const LaunchCfg& lc, const StencilArgs& a, const Geo& geo) {
  if (geo.cluster)
    launch_geo(k_stencil<INM, OUTM, RED, NO, 1>, geo, lc.stream, a);
  else
    launch_geo(k_stencil<INM, OUTM, RED, NO, 0>, geo, lc.stream, a);
}

template <int INM, int OUTM, int RED>
static void dispatch_no(const LaunchCfg& lc, const StencilArgs& a, const Geo& geo) {
  const int n = a.A.nofs;
  if (a.A.pcode && !geo.cluster && (n == 9 || n == 13)) {  // pair-compressed fine operator
    if (n == 9)
      launch_geo(k_stencil<INM, OUTM, RED, 9, 0, true>, geo, lc.stream, a);
    else
      launch_geo(k_stencil<INM, OUTM, RED, 13, 0, true>, geo, lc.stream, a);
  } else if (a.A.ccode && !geo.cluster) {  // class-compressed coarse operator
    launch_geo(k_stencil<INM, OUTM, RED, 0, 0, false, true>, geo, lc.stream, a);
  } else if (n == 5)
    launch_stencil_no<INM, OUTM, RED, 5>(lc, a, geo);
  else if (n == 9)
    launch_stencil_no<INM, OUTM, RED, 9>(lc, a, geo);
  else if (n == 21)
    launch_stencil_no<INM, OUTM, RED, 21>(lc, a, geo);
  else if (n <= 7)
    launch_stencil_no<INM, OUTM, RED, 7>(lc, a, geo);
  else if (n <= 13)
    launch_stencil_no<INM, OUTM, RED, 13>(lc, a, geo);
  else if (n <= 25)
    launch_stencil_no<INM, OUTM, RED, 25>(lc, a, geo);
  else
    launch_stencil_no<INM, OUTM, RED, 0>(lc, a, geo);
  constexpr int NV = ((RED & RED_NORM) ? 1 : 0) + ((RED & (RED_DOT | RED_DOT_CENTER)) ? 2 : 0);
  if constexpr (NV > 0) launch_finalize<NV>(lc, geo, a.gate, a.rs, a.epi);
}

void launch_stencil(const LaunchCfg& lc, int inm, int outm, int red, const StencilArgs& a) {
  ++g_launch_count;
  const long N = (long)a.A.n1own * a.A.n2 * a.A.n3;  // points computed (owned slab)
  const Geo geo = red ? geo_for(lc, N) : Geo{blocks_for(lc, N), 0};
  constexpr int J = IN_SCALE | IN_JAC | IN_WRITEV;
  // 3D pair-compressed fine level, plain input: the plane-marching bulk-copy kernel
  if (march_takes(a.A) && !geo.cluster && launch_march(lc, inm, outm, red, a)) return;
  // tiled kernel where it measured faster (B200): 2D operators with wide (Galerkin)
  // stencils; the 3D and 9-point fine-level sweeps keep the flat kernel, whose
  // neighbour re-reads L1 already absorbs (tools/prof_solve.py A/B)
  if (g_stencil_tile && !geo.cluster && a.A.n1own >= 2 && !a.A.pcode && !a.A.ccode &&
      (g_stencil_tile > 1 || (a.A.n3 == 1 && a.A.nofs > 9))) {
    const bool d3 = a.A.n3 > 1;
    TileCfg t{};
    t.tp = d3 ? 2 : 8;
    t.ty = d3 ? 4 : 1;
    t.tx = d3 ? 32 : 32;
    t.hy = d3 ? 2 : 0;
    const int nY = d3 ? a.A.n2 : 1, nX = d3 ? a.A.n3 : a.A.n2;
    t.ntp = (a.A.n1own + t.tp - 1) / t.tp;
    t.nty = (nY + t.ty - 1) / t.ty;
    t.ntx = (nX + t.tx - 1) / t.tx;
    const long ntiles = (long)t.ntp * t.nty * t.ntx;
    const int blocks = (int)(ntiles < lc.max_blocks ? ntiles : lc.max_blocks);
#define HADR_TCASE(I, O, R)                          \
  if (inm == (I) && outm == (O) && red == (R)) {     \
    dispatch_tile<I, O, R>(lc, a, t, blocks);        \
    return;                                          \
  }
    HADR_TCASE(IN_PLAIN, OUT_APPLY, RED_NONE)
    HADR_TCASE(IN_PLAIN, OUT_APPLY, RED_NORM | RED_DOT)
  HADR_TCASE(IN_PLAIN, OUT_APPLY, RED_DOT)
    HADR_TCASE(IN_PLAIN, OUT_RESID, RED_NONE)
    HADR_TCASE(IN_PLAIN, OUT_RESID, RED_NORM)
    HADR_TCASE(J, OUT_APPLY, RED_DOT_CENTER)
    HADR_TCASE(J, OUT_APPLY, RED_DOT)
    HADR_TCASE(IN_JAC, OUT_APPLY, RED_NONE)
#undef HADR_TCASE
  }
#define HADR_CASE(I, O, R)                       \
  if (inm == (I) && outm == (O) && red == (R)) { \
    dispatch_no<I, O, R>(lc, a, geo);            \
    return;                                      \
  }
  HADR_CASE(IN_PLAIN, OUT_APPLY, RED_NONE)
  HADR_CASE(IN_PLAIN, OUT_APPLY, RED_NORM | RED_DOT)
  HADR_CASE(IN_PLAIN, OUT_APPLY, RED_DOT)
  HADR_CASE(IN_PLAIN, OUT_RESID, RED_NONE)
  HADR_CASE(IN_PLAIN, OUT_RESID, RED_NORM)
  HADR_CASE(J, OUT_APPLY, RED_DOT_CENTER)
  HADR_CASE(J, OUT_APPLY, RED_DOT)
  HADR_CASE(IN_JAC, OUT_APPLY, RED_NONE)
#undef HADR_CASE
  throw std::runtime_error("launch_stencil: unsupported variant");
}

// ---------------------------------------------------------------------------
// K2/K3: MGS building blocks.  w -= h v (numpy: tmp = h*v; w = w - tmp) fused
// with the next inner product / norm of the updated w.
// ---------------------------------------------------------------------------
template <int RED, int CL>
__global__ void __launch_bounds__(kThreads) k_axpy_red(long n, cplx* __restrict__ w, const cplx* h,
                                                         const cplx* __restrict__ v, const cplx* __restrict__ u,
                                                         Gate g, RedScratch rs, Epi e, Pend in) {
  pdl_enter();
  if (!gate_open(g)) return;
  cplx hh;
  if (in.partials) {  // the deferred finalize of the producer (k_finalize<2>'s exact summation)
    __shared__ double smf[2 * 32];
    __shared__ double tot[2];
    double acc[2] = {0.0, 0.0};
    for (int b = threadIdx.x; b < in.nblocks; b += blockDim.x) {
      acc[0] += in.partials[b * 2];
      acc[1] += in.partials[b * 2 + 1];
    }
    block_sum<2>(acc, smf);
    if (threadIdx.x == 0) {
      tot[0] = acc[0];
      tot[1] = acc[1];
      if (blockIdx.x == 0) run_epi(in.e, acc, 2);
    }
    __syncthreads();
    hh = mk(tot[0], tot[1]);
  } else {
    hh = *h;
  }
  constexpr int NV = (RED == RED_NORM) ? 1 : 2;
  double red[NV];
#pragma unroll
  for (int q = 0; q < NV; ++q) red[q] = 0.0;
  const long stride = (long)gridDim.x * blockDim.x;
  for (long k = (long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride) {
    cplx y = csub(w[k], cmul_np(hh, ldc(v, k)));
    w[k] = y;
    if (RED == RED_NORM) {
      red[0] += y.x * y.x + y.y * y.y;
    } else {
      const cplx uu = ldc(u, k);
      red[0] += uu.x * y.x + uu.y * y.y;
      red[NV - 1] += uu.x * y.y - uu.y * y.x;
    }
  }
  finish<NV, CL>(red, rs, e);
}

void launch_axpy_red(const LaunchCfg& lc, long n, cplx* w, const cplx* h, const cplx* v, int red, const cplx* u,
                     Gate g, RedScratch rs, Epi e, Pend in) {
  ++g_launch_count;
  const Geo geo = geo_for(lc, n);
  if (in.partials && (geo.cluster || lc.dist)) throw std::logic_error("a deferred reduction needs a plain grid");
  if (red == RED_NORM) {
    if (geo.cluster)
      launch_geo(k_axpy_red<RED_NORM, 1>, geo, lc.stream, n, w, h, v, u, g, rs, e, in);
    else
      launch_geo(k_axpy_red<RED_NORM, 0>, geo, lc.stream, n, w, h, v, u, g, rs, e, in);
    launch_finalize<1>(lc, geo, g, rs, e);
  } else {
    if (geo.cluster)
      launch_geo(k_axpy_red<RED_DOT, 1>, geo, lc.stream, n, w, h, v, u, g, rs, e, in);
    else
      launch_geo(k_axpy_red<RED_DOT, 0>, geo, lc.stream, n, w, h, v, u, g, rs, e, in);
    launch_finalize<2>(lc, geo, g, rs, e);
  }
}

template <int CL>
__global__ void __launch_bounds__(kThreads) k_dot(long n, const cplx* __restrict__ u, const cplx* __restrict__ w,
                                                    Gate g, RedScratch rs, Epi e) {
  pdl_enter();
  if (!gate_open(g)) return;
  double red[2] = {0.0, 0.0};
  const long stride = (long)gridDim.x * blockDim.x;
  for (long k = (long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride) {
    const cplx uu = ldc(u, k), y = ldc(w, k);
    red[0] += uu.x * y.x + uu.y * y.y;
    red[1] += uu.x * y.y - uu.y * y.x;
  }
  finish<2, CL>(red, rs, e);
}

void launch_dot(const LaunchCfg& lc, long n, const cplx* u, const cplx* w, Gate g, RedScratch rs, Epi e) {
  ++g_launch_count;
  const Geo geo = geo_for(lc, n);
  if (geo.cluster)
    launch_geo(k_dot<1>, geo, lc.stream, n, u, w, g, rs, e);
  else
    launch_geo(k_dot<0>, geo, lc.stream, n, u, w, g, rs, e);
  launch_finalize<2>(lc, geo, g, rs, e);
}

template <int RED, int CL>
__global__ void __launch_bounds__(kThreads) k_scale(long n, const cplx* __restrict__ in, const double* s,
                                                      cplx* __restrict__ out, Gate g, RedScratch rs, Epi e) {
  pdl_enter();
  if (!gate_open(g)) return;
  const double sc = s ? *s : 1.0;
  double red[1] = {0.0};
  const long stride = (long)gridDim.x * blockDim.x;
  for (long k = (long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride) {
    cplx y = ldc(in, k);
    if (s) y = cscale(y, sc);
    if (out) out[k] = y;
    if (RED) red[0] += y.x * y.x + y.y * y.y;
  }
  if constexpr (RED != 0) finish<1, CL>(red, rs, e);
}

void launch_scale(const LaunchCfg& lc, long n, const cplx* in, const double* s, cplx* out, int red, Gate g,
                  RedScratch rs, Epi e) {
  ++g_launch_count;
  if (red) {
    const Geo geo = geo_for(lc, n);
    if (geo.cluster)
      launch_geo(k_scale<1, 1>, geo, lc.stream, n, in, s, out, g, rs, e);
    else
      launch_geo(k_scale<1, 0>, geo, lc.stream, n, in, s, out, g, rs, e);
    launch_finalize<1>(lc, geo, g, rs, e);
  } else {
    launch_k(k_scale<0, 0>, blocks_for(lc, n), kThreads, lc.stream, n, in, s, out, g, rs, e);
  }
}

__global__ void k_zero(long n, cplx* out, Gate g) {
  pdl_enter();
  if (!gate_open(g)) return;
  const long stride = (long)gridDim.x * blockDim.x;
  for (long k = (long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride) out[k] = mk(0.0, 0.0);
}
// Relaxation step input, split out of the stencil on large 3D levels (Hier::emit_relax):
// v = s x (the new basis vector) and z = D^-1 (.) v — the values the fused stencil would
// form per neighbour, formed once per point.
__global__ void __launch_bounds__(kThreads) k_scale_jac(long n, const cplx* __restrict__ in, const double* s,
                                                        const cplx* __restrict__ dinv, cplx* __restrict__ v,
                                                        cplx* __restrict__ z, Gate g) {
  pdl_enter();
  if (!gate_open(g)) return;
  const double sc = *s;
  for (long k = (long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (long)gridDim.x * blockDim.x) {
    const cplx a = cscale(ldc(in, k), sc);
    v[k] = a;
    z[k] = cmul_np(ldc(dinv, k), a);
  }
}

void launch_scale_jac(const LaunchCfg& lc, long n, const cplx* in, const double* s, const cplx* dinv, cplx* v,
                      cplx* z, Gate g) {
  ++g_launch_count;
  launch_k(k_scale_jac, blocks_for(lc, n), kThreads, lc.stream, n, in, s, dinv, v, z, g);
}

void launch_zero(const LaunchCfg& lc, long n, cplx* out, Gate g) {
  ++g_launch_count;
  launch_k(k_zero, blocks_for(lc, n), kThreads, lc.stream, n, out, g);
}

// K5: out = base + [dinv (.)] sum_i v_i y_i
__global__ void __launch_bounds__(kThreads) k_lincomb(long n, LinComb c, Gate g) {
  pdl_enter();
  if (!gate_open(g)) return;
  const int k = c.kptr ? *c.kptr : c.kfix;
  cplx y[MMAX];
#pragma unroll
  for (int i = 0; i < MMAX; ++i) y[i] = (i < k) ? (c.y ? c.y[i] : c.yv[i]) : mk(0.0, 0.0);
  const long stride = (long)gridDim.x * blockDim.x;
  for (long p = (long)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += stride) {
    cplx t = mk(0.0, 0.0);
    for (int i = 0; i < k; ++i) t = cadd(t, cmul_np(ldc(c.v[i], p), y[i]));
    if (c.dinv) t = cmul_np(ldc(c.dinv, p), t);
    c.out[p] = c.base ? cadd(ldc(c.base, p), t) : cadd(mk(0.0, 0.0), t);
  }
}
void launch_lincomb(const LaunchCfg& lc, long n, const LinComb& c, Gate g) {
  ++g_launch_count;
  launch_k(k_lincomb, blocks_for(lc, n), kThreads, lc.stream, n, c, g);
}

// brk_stage 1: first-cycle early exit, x = 0 + Z0*y0 (k<=1)
// brk_stage 0: final: ZERO -> 0 ; FIN/cycle0 -> x = Z0 y0 + Z1 y1 ; FIN/cycle1 -> x += Z1 y0
__global__ void __launch_bounds__(kThreads) k_fg_finalize(long n, FgCtl* f, const cplx* __restrict__ Z0,
                                                            const cplx* __restrict__ Z1, cplx* x, Gate g,
                                                            int brk_stage) {
  pdl_enter();
  if (!gate_open(g)) return;
  const int path = f->path, k = f->k, cyc = f->cycle;
  const cplx y0 = f->y[0], y1 = f->y[1];
  const long stride = (long)gridDim.x * blockDim.x;
  for (long p = (long)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += stride) {
    cplx out;
    if (brk_stage) {
      out = (k >= 1) ? cadd(mk(0.0, 0.0), cmul_np(ldc(Z0, p), y0)) : mk(0.0, 0.0);
    } else if (path == FG_ZERO) {
      out = mk(0.0, 0.0);
    } else if (cyc == 0) {
      cplx t = mk(0.0, 0.0);
      if (k >= 1) t = cadd(t, cmul_np(ldc(Z0, p), y0));
      if (k >= 2) t = cadd(t, cmul_np(ldc(Z1, p), y1));
      out = cadd(mk(0.0, 0.0), t);
    } else {
      out = (k >= 1) ? cadd(x[p], cmul_np(ldc(Z1, p), y0)) : x[p];
    }
    x[p] = out;
  }
}
void launch_fg_finalize(const LaunchCfg& lc, long n, FgCtl* f, const cplx* Z0, const cplx* Z1, cplx* x, Gate g,
                        int brk_stage) {
  ++g_launch_count;
  launch_k(k_fg_finalize, blocks_for(lc, n), kThreads, lc.stream, n, f, Z0, Z1, x, g, brk_stage);
}

// ---------------------------------------------------------------------------
// K6/K7: transfer operators for the (tri)linear P = kron(P1(n1), P1(n2), P1(n3)).
// Restriction rc = P^T r follows scipy csc_matvec: contributions added in
// ascending fine index, i.e. lexicographic (a, b, c) over the 3x3(x3) fine
// patch.  Prolongation follows csr_matvec: parents in ascending coarse index.
// Weights are powers of two, so each product is exact and the sums match the
// reference bit for bit.  An axis of size 1 (2D: n3 = 1) is not coarsened.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int coarse_n(int n) { return (n - 1) / 2 + 1; }

__global__ void __launch_bounds__(kThreads) k_restrict(int n1f, int n2f, int n3f, int p0f, int q0, int nq,
                                                         const cplx* __restrict__ r, cplx* __restrict__ rc, Gate g) {
  pdl_enter();
  // coarse planes [q0, q0 + nq) (rc points at plane q0); r points at fine plane p0f (halo at < 0)
  if (!gate_open(g)) return;
  const int n2c = coarse_n(n2f), n3c = coarse_n(n3f);
  const long Nc = (long)nq * n2c * n3c;
  const int c3lo = n3f > 1 ? -1 : 0, c3hi = n3f > 1 ? 1 : 0;
  const long stride = (long)gridDim.x * blockDim.x;
  for (long c = (long)blockIdx.x * blockDim.x + threadIdx.x; c < Nc; c += stride) {
    const int Il = (int)(c / ((long)n2c * n3c));
    const int I1 = Il + q0;
    const int rem = (int)(c - (long)Il * n2c * n3c);
    const int I2 = rem / n3c, I3 = rem - (rem / n3c) * n3c;
    cplx acc = mk(0.0, 0.0);
#pragma unroll
    for (int a = -1; a <= 1; ++a) {
      const int f1 = 2 * I1 + a;
      if (f1 < 0 || f1 >= n1f) continue;
      const double w1 = a == 0 ? 1.0 : 0.5;
#pragma unroll
      for (int b = -1; b <= 1; ++b) {
        const int f2 = 2 * I2 + b;
        if (f2 < 0 || f2 >= n2f) continue;
        const double w12 = w1 * (b == 0 ? 1.0 : 0.5);
        for (int cc = c3lo; cc <= c3hi; ++cc) {
          const int f3 = 2 * I3 + cc;
          if (f3 < 0 || f3 >= n3f) continue;
          const double w = w12 * (cc == 0 ? 1.0 : 0.5);
          acc = cadd(acc, cmul_sp(mk(w, 0.0), ldc(r, ((long)(f1 - p0f) * n2f + f2) * n3f + f3)));
        }
      }
    }
    rc[c] = acc;
  }
}
void launch_restrict(const LaunchCfg& lc, int n1f, int n2f, int n3f, const cplx* r, cplx* rc, Gate g, int p0f,
                     int q0, int nq) {
  ++g_launch_count;
  if (nq < 0) nq = (n1f - 1) / 2 + 1;
  const long Nc = (long)nq * ((n2f - 1) / 2 + 1) * ((n3f - 1) / 2 + 1);
  launch_k(k_restrict, blocks_for(lc, Nc), kThreads, lc.stream, n1f, n2f, n3f, p0f, q0, nq, r, rc, g);
}

__device__ __forceinline__ int parents(int f, int* p, double& w) {
  if (f & 1) {
    p[0] = f >> 1;
    p[1] = (f >> 1) + 1;
    w = 0.5;
    return 2;
  }
  p[0] = f >> 1;
  p[1] = p[0];
  w = 1.0;
  return 1;
}

__global__ void __launch_bounds__(kThreads) k_prolong_add(int n1f, int n2f, int n3f, int p0f, int nf, int q0c,
                                                            const cplx* __restrict__ ec, cplx* __restrict__ x, Gate g) {
  pdl_enter();
  // fine planes [p0f, p0f + nf) (x points at plane p0f); ec points at coarse plane q0c
  if (!gate_open(g)) return;
  const int n2c = coarse_n(n2f), n3c = coarse_n(n3f);
  const int n23 = n2f * n3f;
  const long Nf = (long)nf * n23;
  const long stride = (long)gridDim.x * blockDim.x;
  for (long f = (long)blockIdx.x * blockDim.x + threadIdx.x; f < Nf; f += stride) {
    const int fl = (int)(f / n23);
    const int f1 = fl + p0f;
    const int rem = (int)(f - (long)fl * n23);
    const int f2 = rem / n3f, f3 = rem - (rem / n3f) * n3f;
    int c1[2], c2[2], c3[2];
    double w1, w2, w3;
    const int m1 = parents(f1, c1, w1), m2 = parents(f2, c2, w2), m3 = parents(f3, c3, w3);
    cplx p = mk(0.0, 0.0);
    for (int a = 0; a < m1; ++a)
      for (int b = 0; b < m2; ++b)
        for (int cc = 0; cc < m3; ++cc)
          p = cadd(p, cmul_sp(mk(w1 * w2 * w3, 0.0), ldc(ec, ((long)(c1[a] - q0c) * n2c + c2[b]) * n3c + c3[cc])));
    x[f] = cadd(x[f], p);
  }
}
void launch_prolong_add(const LaunchCfg& lc, int n1f, int n2f, int n3f, const cplx* ec, cplx* x, Gate g, int p0f,
                        int nf, int q0c) {
  ++g_launch_count;
  if (nf < 0) nf = n1f;
  launch_k(k_prolong_add, blocks_for(lc, (long)nf * n2f * n3f), kThreads, lc.stream, n1f, n2f, n3f, p0f, nf, q0c,
           ec, x, g);
}

// ---------------------------------------------------------------------------
// gates and control initialisation (single thread)
// ---------------------------------------------------------------------------
__global__ void k_set_gate(int* dst, Gate g) {
  pdl_enter();
  *dst = gate_open(g) ? 1 : 0;
}
void launch_set_gate(cudaStream_t s, int* dst, Gate g) {
  ++g_launch_count; launch_k(k_set_gate, 1, 1, s, dst, g); }

__global__ void k_relax_init(RelaxCtl* c, int steps, Gate g) {
  pdl_enter();
  if (!gate_open(g)) return;
  c->steps = steps;
  c->k = 0;
  c->cur = kStopped;
}
void launch_relax_init(cudaStream_t s, RelaxCtl* c, int steps, Gate g) {
  ++g_launch_count; launch_k(k_relax_init, 1, 1, s, c, steps, g); }

__global__ void k_fg_setup(FgCtl* f, double tol, Gate g) {
  pdl_enter();
  if (!gate_open(g)) return;
  f->tol = tol;
  f->reo = 0;
}
void launch_fg_setup(cudaStream_t s, FgCtl* f, double tol, Gate g) {
  ++g_launch_count; launch_k(k_fg_setup, 1, 1, s, f, tol, g); }

// ---------------------------------------------------------------------------
// operator construction (setup; not on the solve's inner loop)
// ---------------------------------------------------------------------------
__device__ __forceinline__ void decomp3(long k, int n2, int n3, int& i1, int& i2, int& i3) {
  const long n23 = (long)n2 * n3;
  i1 = (int)(k / n23);
  const int rem = (int)(k - (long)i1 * n23);
  i2 = rem / n3;
  i3 = rem - i2 * n3;
}

__global__ void k_csr_mask(int n1, int n2, int n3, const int64_t* indptr, const int32_t* indices,
                           unsigned long long* mask) {
  const long N = (long)n1 * n2 * n3;
  unsigned long long m0 = 0ull, m1 = 0ull, bad = 0ull;
  for (long row = (long)blockIdx.x * blockDim.x + threadIdx.x; row < N; row += (long)gridDim.x * blockDim.x) {
    int i1, i2, i3;
    decomp3(row, n2, n3, i1, i2, i3);
    for (int64_t p = indptr[row]; p < indptr[row + 1]; ++p) {
      int j1, j2, j3;
      decomp3(indices[p], n2, n3, j1, j2, j3);
      const int d1 = j1 - i1, d2 = j2 - i2, d3 = j3 - i3;
      if (d1 < -2 || d1 > 2 || d2 < -2 || d2 > 2 || d3 < -2 || d3 > 2) {
        bad = 1ull;
      } else {
        const int q = slot125(d1, d2, d3);
        if (q < 64) m0 |= 1ull << q; else m1 |= 1ull << (q - 64);
      }
    }
  }
  if (m0) atomicOr(mask, m0);
  if (m1) atomicOr(mask + 1, m1);
  if (bad) atomicOr(mask + 2, 1ull);
}
void launch_csr_mask(cudaStream_t s, int n1, int n2, int n3, const int64_t* indptr, const int32_t* indices,
                     unsigned long long* mask) {
  ++g_launch_count;
  long N = (long)n1 * n2 * n3;
  int blocks = (int)((N + 255) / 256);
  if (blocks > 4096) blocks = 4096;
  k_csr_mask<<<blocks, 256, 0, s>>>(n1, n2, n3, indptr, indices, mask);
}

__global__ void k_csr_scatter(int n1, int n2, int n3, const int64_t* indptr, const int32_t* indices,
                              const cplx* data, const int* slot_of, cplx* coef) {
  const long N = (long)n1 * n2 * n3;
  for (long row = (long)blockIdx.x * blockDim.x + threadIdx.x; row < N; row += (long)gridDim.x * blockDim.x) {
    int i1, i2, i3;
    decomp3(row, n2, n3, i1, i2, i3);
    for (int64_t p = indptr[row]; p < indptr[row + 1]; ++p) {
      int j1, j2, j3;
      decomp3(indices[p], n2, n3, j1, j2, j3);
      const int sl = slot_of[slot125(j1 - i1, j2 - i2, j3 - i3)];
      cplx* dst = coef + (long)sl * N + row;
      *dst = cadd(*dst, data[p]);
    }
  }
}
void launch_csr_scatter(cudaStream_t s, int n1, int n2, int n3, const int64_t* indptr, const int32_t* indices,
                        const cplx* data, const int* slot_of, cplx* coef) {
  ++g_launch_count;
  long N = (long)n1 * n2 * n3;
  int blocks = (int)((N + 255) / 256);
  if (blocks > 4096) blocks = 4096;
  k_csr_scatter<<<blocks, 256, 0, s>>>(n1, n2, n3, indptr, indices, data, slot_of, coef);
}

// z = r / d elementwise (numpy complex division), helmadr/krylov.py:68-73
__global__ void k_cdiv(long n, const cplx* r, const cplx* d, cplx* z) {
  for (long k = (long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (long)gridDim.x * blockDim.x)
    z[k] = cdiv_np(r[k], d[k]);
}
void launch_cdiv(cudaStream_t s, long n, const cplx* r, const cplx* d, cplx* z) {
  ++g_launch_count;
  int blocks = (int)((n + 255) / 256);
  if (blocks > 4096) blocks = 4096;
  k_cdiv<<<blocks, 256, 0, s>>>(n, r, d, z);
}

// dinv = 1.0 / diag (numpy complex division), helmadr/multigrid.py:74-81
__global__ void k_inv_diag(long n, const cplx* diag, cplx* dinv, int* zero_flag) {
  for (long k = (long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (long)gridDim.x * blockDim.x) {
    const cplx d = diag ? diag[k] : mk(0.0, 0.0);
    if (d.x == 0.0 && d.y == 0.0) atomicOr(zero_flag, 1);
    dinv[k] = cdiv_np(mk(1.0, 0.0), d);
  }
}
void launch_inv_diag(cudaStream_t s, long n, const cplx* diag, cplx* dinv, int* zero_flag) {
  ++g_launch_count;
  int blocks = (int)((n + 255) / 256);
  if (blocks > 4096) blocks = 4096;
  k_inv_diag<<<blocks, 256, 0, s>>>(n, diag, dinv, zero_flag);
}

// dst[dst_slot[o]] (+)= alpha * src[o]   (scalar * CSR data, then CSR + CSR)
__global__ void k_remap_planes(long n, const cplx* src, int nsrc, const int* dst_slot, cplx* dst, cplx alpha,
                               int accumulate, int scaled) {
  for (long k = (long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (long)gridDim.x * blockDim.x) {
    for (int o = 0; o < nsrc; ++o) {
      cplx v = src[(long)o * n + k];
      if (scaled) v = cmul_np(v, alpha);
      cplx* d = dst + (long)dst_slot[o] * n + k;
      *d = accumulate ? cadd(*d, v) : v;
    }
  }
}
void launch_remap_planes(cudaStream_t s, long n, const cplx* src, int nsrc, const int* dst_slot, cplx* dst,
                         cplx alpha, int accumulate) {
  ++g_launch_count;
  int blocks = (int)((n + 255) / 256);
  if (blocks > 4096) blocks = 4096;
  const int scaled = !(alpha.x == 1.0 && alpha.y == 0.0);
  k_remap_planes<<<blocks, 256, 0, s>>>(n, src, nsrc, dst_slot, dst, alpha, accumulate, scaled);
}

// center += sc * field  (complex scalar times real field, numpy product; then CSR add)
__global__ void k_add_diag_real(long n, cplx* center, cplx sc, const double* field) {
  for (long k = (long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (long)gridDim.x * blockDim.x)
    center[k] = cadd(center[k], cmul_np(sc, mk(field[k], 0.0)));
}
void launch_add_diag_real(cudaStream_t s, long n, cplx* center, cplx sc, const double* field) {
  ++g_launch_count;
  int blocks = (int)((n + 255) / 256);
  if (blocks > 4096) blocks = 4096;
  k_add_diag_real<<<blocks, 256, 0, s>>>(n, center, sc, field);
}

// diag(left) @ A @ diag(right): scipy csr_matmat products, left first (helmadr/operators.py:264)
__global__ void k_similarity(StencilDev A, cplx* out, const cplx* left, const cplx* right) {
  const int n1 = A.n1, n2 = A.n2, n3 = A.n3;
  const long N = (long)n1 * n2 * n3;
  for (long k = (long)blockIdx.x * blockDim.x + threadIdx.x; k < N; k += (long)gridDim.x * blockDim.x) {
    int i1, i2, i3;
    decomp3(k, n2, n3, i1, i2, i3);
    for (int o = 0; o < A.nofs; ++o) {
      const int j1 = i1 + A.d1[o], j2 = i2 + A.d2[o], j3 = i3 + A.d3[o];
      cplx v = mk(0.0, 0.0);
      if (j1 >= 0 && j1 < n1 && j2 >= 0 && j2 < n2 && j3 >= 0 && j3 < n3) {
        const cplx c = A.coef[(long)o * N + k];
        v = cmul_sp(cmul_sp(left[k], c), right[((long)j1 * n2 + j2) * n3 + j3]);
      }
      out[(long)o * N + k] = v;
    }
  }
}
void launch_similarity(cudaStream_t s, const StencilDev& A, cplx* out, const cplx* left, const cplx* right) {
  ++g_launch_count;
  long N = (long)A.n1 * A.n2 * A.n3;
  int blocks = (int)((N + 255) / 256);
  if (blocks > 4096) blocks = 4096;
  k_similarity<<<blocks, 256, 0, s>>>(A, out, left, right);
}

// K8: Galerkin coarse operator A_c = P^T A P on the stencil representation.
// Pass 1 (coef_c == null): OR the mask of non-zero coarse offsets (5x5x5 box).
// Pass 2: write the compacted planes (slot_of maps box slot -> plane).
// Slabs: coarse planes [q0, q0 + nq) are produced (coef_c points at plane q0, planes cstride apart); the fine
// coefficients are read relative to Af.p0 with plane stride Af.pstride (one halo plane below is read).
__global__ void k_galerkin(StencilDev Af, int n1c, int n2c, int n3c, int q0, int nq, long cstride,
                           unsigned long long* mask, const int* slot_of, cplx* coef_c) {
  const int n1f = Af.n1, n2f = Af.n2, n3f = Af.n3;
  const long Nf = Af.pstride, Nc = (long)nq * n2c * n3c;
  const long fbase = (long)Af.p0 * n2f * n3f;
  const int c3lo = n3f > 1 ? -1 : 0, c3hi = n3f > 1 ? 1 : 0;
  unsigned long long m0 = 0ull, m1 = 0ull;
  for (long c = (long)blockIdx.x * blockDim.x + threadIdx.x; c < Nc; c += (long)gridDim.x * blockDim.x) {
    int I1, I2, I3;
    decomp3(c, n2c, n3c, I1, I2, I3);
    I1 += q0;
    cplx acc[125];
    for (int q = 0; q < 125; ++q) acc[q] = mk(0.0, 0.0);
    for (int a = -1; a <= 1; ++a) {
      const int f1 = 2 * I1 + a;
      if (f1 < 0 || f1 >= n1f) continue;
      for (int b = -1; b <= 1; ++b) {
        const int f2 = 2 * I2 + b;
        if (f2 < 0 || f2 >= n2f) continue;
        for (int cc = c3lo; cc <= c3hi; ++cc) {
          const int f3 = 2 * I3 + cc;
          if (f3 < 0 || f3 >= n3f) continue;
          const double wf = (a == 0 ? 1.0 : 0.5) * (b == 0 ? 1.0 : 0.5) * (cc == 0 ? 1.0 : 0.5);
          const long f = ((long)f1 * n2f + f2) * n3f + f3 - fbase;
          for (int o = 0; o < Af.nofs; ++o) {
            const int g1 = f1 + Af.d1[o], g2 = f2 + Af.d2[o], g3 = f3 + Af.d3[o];
            if (g1 < 0 || g1 >= n1f || g2 < 0 || g2 >= n2f || g3 < 0 || g3 >= n3f) continue;
            const cplx cf = Af.coef[(long)o * Nf + f];
            if (cf.x == 0.0 && cf.y == 0.0) continue;
            const cplx wc = mk(wf * cf.x, wf * cf.y);
            int p1[2], p2[2], p3[2];
            double v1, v2, v3;
            const int m1n = parents(g1, p1, v1), m2n = parents(g2, p2, v2), m3n = parents(g3, p3, v3);
            for (int x = 0; x < m1n; ++x)
              for (int y = 0; y < m2n; ++y)
                for (int z = 0; z < m3n; ++z) {
                  const int sl = slot125(p1[x] - I1, p2[y] - I2, p3[z] - I3);
                  const double pw = v1 * v2 * v3;
                  acc[sl] = cadd(acc[sl], mk(pw * wc.x, pw * wc.y));
                }
          }
        }
      }
    }
    for (int q = 0; q < 125; ++q) {
      if (acc[q].x != 0.0 || acc[q].y != 0.0) {
        if (q < 64) m0 |= 1ull << q; else m1 |= 1ull << (q - 64);
      }
      if (coef_c && slot_of[q] >= 0) coef_c[(long)slot_of[q] * cstride + c] = acc[q];
    }
  }
  if (mask) {
    if (m0) atomicOr(mask, m0);
    if (m1) atomicOr(mask + 1, m1);
  }
}
void launch_galerkin(cudaStream_t s, const StencilDev& Af, int n1c, int n2c, int n3c, unsigned long long* mask,
                     const int* slot_of, cplx* coef_c, int q0, int nq, long cstride) {
  ++g_launch_count;
  if (nq < 0) nq = n1c;
  if (cstride < 0) cstride = (long)n1c * n2c * n3c;
  long Nc = (long)nq * n2c * n3c;
  int blocks = (int)((Nc + 127) / 128);
  if (blocks > 4096) blocks = 4096;
  if (blocks < 1) return;
  k_galerkin<<<blocks, 128, 0, s>>>(Af, n1c, n2c, n3c, q0, nq, cstride, mask, slot_of, coef_c);
}

}  // namespace hadr

namespace hadr {

// ---------------------------------------------------------------------------
// On-device assembly of the ADR / Helmholtz operators (helmadr/operators.py:85-234),
// per axis, into the plus-radius-2 planes of `dim` axes, ordered (d1, d2, d3):
//   2D (9):  (-2,0) (-1,0) (0,-2) (0,-1) (0,0) (0,1) (0,2) (1,0) (2,0)
//   3D (13): the same with a third axis.
// Each term is formed with the reference's numpy expression semantics; the
// duplicates of a row are summed in the order the reference appends them.
// 3D restatement decisions: faces (left,right) / (front,back) / (top,bottom) for
// axes 0 / 1 / last; mass weight -i/(2 dim) (2D: the reference's -0.25j).
// ---------------------------------------------------------------------------
__device__ __forceinline__ int pl(int dim, int ax, int d) {  // plane of offset d along axis ax
  if (dim == 2) {
    if (d == 0) return 4;
    if (ax == 0) return d == -2 ? 0 : d == -1 ? 1 : d == 1 ? 7 : 8;
    return d == -2 ? 2 : d == -1 ? 3 : d == 1 ? 5 : 6;
  }
  // 3D order: (-2,0,0) (-1,0,0) (0,-2,0) (0,-1,0) (0,0,-2) (0,0,-1) (0,0,0) (0,0,1) (0,0,2) (0,1,0) (0,2,0) (1,0,0) (2,0,0)
  if (d == 0) return 6;
  if (ax == 0) return d == -2 ? 0 : d == -1 ? 1 : d == 1 ? 11 : 12;
  if (ax == 1) return d == -2 ? 2 : d == -1 ? 3 : d == 1 ? 9 : 10;
  return d == -2 ? 4 : d == -1 ? 5 : d == 1 ? 7 : 8;
}

// complex scalar (python complex) times real array element, numpy complex multiply
__device__ __forceinline__ cplx cs_times_real(cplx s, double v) { return cmul_np(s, mk(v, 0.0)); }
// complex / real, numpy Smith division by (d, 0)
__device__ __forceinline__ cplx cdiv_real(cplx a, double d) { return cdiv_np(a, mk(d, 0.0)); }

struct AsmArgs {
  int dim;
  int n[3];
  double h[3];
  double omega;
  int scheme;       // 0 central, 1 upwind1, 2 upwind2, 3 helmholtz
  int face[3][2];   // per axis (low, high): 0 neumann, 1 sommerfeld
  int src[3];       // source node (near-source set), src[0] = -1: none
  const double *ksq, *gam, *g[3], *lap;
  cplx* coef;       // 9 (2D) / 13 (3D) planes, `pstride` apart
  unsigned* mask;   // OR of non-zero planes
  int r0, nr;       // rows (axis-0 planes) [r0, r0 + nr); fields and coef point at plane r0
  long pstride;
};

__global__ void k_assemble(AsmArgs a) {
  const int dim = a.dim;
  const int n1 = a.n[0], n2 = a.n[1], n3 = dim == 3 ? a.n[2] : 1;
  const long N = (long)a.nr * n2 * n3;
  const int NP = dim == 2 ? 9 : 13;
  unsigned m = 0u;
  const double om = a.omega;
  for (long k = (long)blockIdx.x * blockDim.x + threadIdx.x; k < N; k += (long)gridDim.x * blockDim.x) {
    int ii[3];
    decomp3(k, n2, n3, ii[0], ii[1], ii[2]);
    ii[0] += a.r0;
    cplx acc[13];
    bool has[13];
#pragma unroll
    for (int q = 0; q < 13; ++q) {
      acc[q] = mk(0.0, 0.0);
      has[q] = false;
    }
    auto put = [&](int q, cplx v) {
      acc[q] = has[q] ? cadd(acc[q], v) : v;
      has[q] = true;
    };
    const bool helm = a.scheme == 3;
    double gr[3] = {0.0, 0.0, 0.0};
    if (!helm)
      for (int ax = 0; ax < dim; ++ax) gr[ax] = a.g[ax][k];
    const double kap = sqrt(a.ksq[k]);
    const int cen = pl(dim, 0, 0);
    // ---- Laplacian + ghost-eliminated BC (helmadr/operators.py:85-120) ----
    for (int ax = 0; ax < dim; ++ax) {
      const double h = a.h[ax];
      const int idx = ii[ax], size = a.n[ax];
      const double ih2 = 1.0 / (h * h);
      if (idx >= 1) put(pl(dim, ax, -1), mk(ih2, 0.0));
      if (idx <= size - 2) put(pl(dim, ax, 1), mk(ih2, 0.0));
      put(cen, mk(-2.0 * ih2, 0.0));
      for (int lo = 1; lo >= 0; --lo) {
        if (lo ? idx != 0 : idx != size - 1) continue;
        const double nd = lo ? -gr[ax] : gr[ax];
        const int kind = a.face[ax][lo ? 0 : 1];
        if (kind == 0) {
          put(pl(dim, ax, lo ? 1 : -1), mk(ih2, 0.0));
          const cplx c2 = mk(0.0 * om, 2.0 * om);  // 2j * omega * nd / h
          put(cen, cdiv_real(cs_times_real(c2, nd), h));
        } else {
          const cplx c1 = mk(0.0 * om * h, 1.0 * om * h);  // (1.0 + 1j*omega*h*(nd - kappa)) * ih2
          const cplx t = cs_times_real(c1, nd - kap);
          const cplx u = mk(1.0 + t.x, t.y);
          put(cen, cmul_np(u, mk(ih2, 0.0)));
        }
      }
    }
    if (!helm) {
      // ---- advection (helmadr/operators.py:123-170) ----
      bool near = a.src[0] >= 0;
      for (int ax = 0; ax < dim; ++ax) near = near && abs(ii[ax] - a.src[ax]) <= 1;
      for (int ax = 0; ax < dim; ++ax) {
        const double h = a.h[ax];
        const int idx = ii[ax], size = a.n[ax];
        const double c = gr[ax];
        const cplx F = cs_times_real(mk(-0.0 * om, -2.0 * om), c);  // -2j * omega * c
        const bool inner = idx >= 1 && idx <= size - 2;
        const bool ctr = a.scheme == 0 ? inner : (inner && near);
        if (ctr) {
          put(pl(dim, ax, 1), cdiv_real(F, 2.0 * h));
          put(pl(dim, ax, -1), cdiv_real(cneg(F), 2.0 * h));
        } else if (c != 0.0) {
          const int sg = c > 0 ? 1 : -1;
          const bool ok2 = sg == 1 ? idx >= 2 : idx <= size - 3;
          const bool ok1 = sg == 1 ? idx >= 1 : idx <= size - 2;
          if (a.scheme != 1 && ok2) {
            put(cen, cdiv_real(cs_times_real(F, sg * 3.0), 2.0 * h));
            put(pl(dim, ax, -sg), cdiv_real(cs_times_real(F, -sg * 4.0), 2.0 * h));
            put(pl(dim, ax, -2 * sg), cdiv_real(cs_times_real(F, (double)sg), 2.0 * h));
          } else if (ok1) {
            put(cen, cdiv_real(cs_times_real(F, (double)sg), h));
            put(pl(dim, ax, -sg), cdiv_real(cs_times_real(F, (double)-sg), h));
          } else {
            put(cen, cdiv_real(cs_times_real(F, (double)-sg), h));
            put(pl(dim, ax, sg), cdiv_real(cs_times_real(F, (double)sg), h));
          }
        }
      }
      // ---- neighbour-averaged mass term (helmadr/operators.py:173-187) ----
      const cplx mw = dim == 2 ? mk(-0.0, -0.25) : mk(-0.0, -1.0 / 6.0);
      const cplx G = cs_times_real(mk(mw.x * om, mw.y * om), a.lap[k]);
      for (int ax = 0; ax < dim; ++ax) {
        const int idx = ii[ax], size = a.n[ax];
        for (int sg = 1; sg >= -1; sg -= 2) {
          const bool ins = sg == 1 ? idx <= size - 2 : idx >= 1;
          put(ins ? pl(dim, ax, sg) : cen, G);
        }
      }
      // ---- reaction + attenuation (helmadr/operators.py:230-233) ----
      double gsq = gr[0] * gr[0] + gr[1] * gr[1];
      if (dim == 3) gsq = gsq + gr[2] * gr[2];
      const double react = -(om * om) * (gsq - a.ksq[k]);
      const cplx att = cs_times_real(cs_times_real(mk(-0.0 * om, -1.0 * om), a.gam[k]), a.ksq[k]);
      put(cen, mk(react + att.x, att.y));
    } else {
      // omega**2 * kappa_sq - 1j * omega * gamma * kappa_sq (helmadr/operators.py:198)
      const double w2k = (om * om) * a.ksq[k];
      const cplx t = cs_times_real(cs_times_real(mk(0.0 * om, 1.0 * om), a.gam[k]), a.ksq[k]);
      put(cen, mk(w2k - t.x, 0.0 - t.y));
    }
    for (int q = 0; q < NP; ++q) {
      a.coef[(long)q * a.pstride + k] = acc[q];
      if (acc[q].x != 0.0 || acc[q].y != 0.0) m |= 1u << q;
    }
  }
  if (m) atomicOr(a.mask, m);
}

void launch_assemble(cudaStream_t s, int dim, int n1, int n2, int n3, double h1, double h2, double h3, double omega,
                     int scheme, const int* bc, int src1, int src2, int src3, const double* ksq, const double* gam,
                     const double* g1, const double* g2, const double* g3, const double* lap, cplx* coefp,
                     unsigned* mask, int r0, int nr, long pstride) {
  ++g_launch_count;
  AsmArgs a{};
  if (nr < 0) nr = n1;
  if (pstride < 0) pstride = (long)n1 * n2 * (dim == 3 ? n3 : 1);
  a.r0 = r0;
  a.nr = nr;
  a.pstride = pstride;
  a.dim = dim;
  a.n[0] = n1;
  a.n[1] = n2;
  a.n[2] = n3;
  a.h[0] = h1;
  a.h[1] = h2;
  a.h[2] = h3;
  a.omega = omega;
  a.scheme = scheme;
  // bc = (top, bottom, left, right, front, back)
  a.face[0][0] = bc[2];
  a.face[0][1] = bc[3];
  if (dim == 2) {
    a.face[1][0] = bc[0];
    a.face[1][1] = bc[1];
  } else {
    a.face[1][0] = bc[4];
    a.face[1][1] = bc[5];
    a.face[2][0] = bc[0];
    a.face[2][1] = bc[1];
  }
  a.src[0] = src1;
  a.src[1] = src2;
  a.src[2] = src3;
  a.ksq = ksq;
  a.gam = gam;
  a.g[0] = g1;
  a.g[1] = g2;
  a.g[2] = g3;
  a.lap = lap;
  a.coef = coefp;
  a.mask = mask;
  long N = (long)nr * n2 * (dim == 3 ? n3 : 1);
  int blocks = (int)((N + 127) / 128);
  if (blocks > 4096) blocks = 4096;
  if (blocks < 1) return;
  k_assemble<<<blocks, 128, 0, s>>>(a);
}

}  // namespace hadr

namespace hadr {

// complex128 -> complex64 (round to nearest) for the mixed-precision K-cycle operators
// out = q (.) exp(sign * i * omega * tau)  (helmadr/operators.py:269-278 rhs_transform; numpy's
// complex product formula; cos/sin are CUDA's, within an ulp of the host libm's)
__global__ void k_phase(long n, const cplx* __restrict__ q, const double* __restrict__ tau, double omega, int sign,
                        cplx* __restrict__ out) {
  for (long k = (long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (long)gridDim.x * blockDim.x) {
    double sn, cs;
    sincos(omega * tau[k], &sn, &cs);
    out[k] = cmul_np(q[k], mk(cs, sign > 0 ? sn : -sn));
  }
}
void launch_phase(cudaStream_t s, long n, const cplx* q, const double* tau, double omega, int sign, cplx* out) {
  ++g_launch_count;
  int blocks = (int)((n + 255) / 256);
  if (blocks > 4096) blocks = 4096;
  if (blocks < 1) return;
  k_phase<<<blocks, 256, 0, s>>>(n, q, tau, omega, sign, out);
}

// ---------------------------------------------------------------------------
// tau_derivatives (helmadr/eikonal.py:180-226) with the distance factor of
// AnalyticBase (helmadr/eikonal.py:15-36): tau = tau0*tau1, grad(tau), lap(tau) from
// tau1 by the chain rule, every expression in the reference's (numpy) order, so the
// fields are bit-identical to the reference's on the same tau1 (tests).
// ---------------------------------------------------------------------------
// np.hypot on this image = glibc 2.39 __hypot (sysdeps/ieee754/dbl-64/e_hypot.c, the
// non-FMA kernel of Borges' correction); grid offsets never reach its huge/tiny
// scaling branches (|e| is 0 or >= one grid step).
__device__ __forceinline__ double glibc_hypot(double x, double y) {
  x = fabs(x);
  y = fabs(y);
  const double ax = x < y ? y : x, ay = x < y ? x : y;
  if (ay <= ax * 0x1p-54) return ax + ay;
  double h = sqrt(ax * ax + ay * ay), t1, t2;
  if (h <= 2.0 * ay) {
    const double d = h - ay;
    t1 = ax * (2.0 * d - ax);
    t2 = (d - 2.0 * (ax - ay)) * d;
  } else {
    const double d = h - ax;
    t1 = 2.0 * d * (ax - 2.0 * ay);
    t2 = (4.0 * d - ay) * ay + d * d;
  }
  return h - (t1 + t2) / (2.0 * h);
}

struct TauGeom {
  int dim;
  int n[3];
  double h[3], L[3];
  int src[3];
};

// first difference along one axis: central inside, one-sided first order at the ends
// (helmadr/eikonal.py:180-188); t(d) = tau1 at offset d along the axis
__device__ __forceinline__ double tau_d1(const double* t, long k, long st, int i, int n, double h) {
  if (i == 0) return (t[k + st] - t[k]) / h;
  if (i == n - 1) return (t[k] - t[k - st]) / h;
  return (t[k + st] - t[k - st]) / (2.0 * h);
}
// second difference: 3-point inside, one-sided 4-point at the ends (helmadr/eikonal.py:191-201)
__device__ __forceinline__ double tau_d2(const double* t, long k, long st, int i, int n, double h) {
  const double hh = h * h;
  if (i == 0) return (2.0 * t[k] - 5.0 * t[k + st] + 4.0 * t[k + 2 * st] - t[k + 3 * st]) / hh;
  if (i == n - 1) return (2.0 * t[k] - 5.0 * t[k - st] + 4.0 * t[k - 2 * st] - t[k - 3 * st]) / hh;
  return (t[k + st] - 2.0 * t[k] + t[k - st]) / hh;
}

__global__ void __launch_bounds__(256) k_tau_derivs(TauGeom g, const double* __restrict__ tau1,
                                                      double* __restrict__ tau, double* __restrict__ gr0,
                                                      double* __restrict__ gr1, double* __restrict__ gr2,
                                                      double* __restrict__ lap) {
  const int n1 = g.n[0], n2 = g.n[1], n3 = g.dim == 3 ? g.n[2] : 1;
  const long n = (long)n1 * n2 * n3;
  const long st[3] = {(long)n2 * n3, (long)n3, 1};
  for (long k = (long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (long)gridDim.x * blockDim.x) {
    const int i[3] = {(int)(k / st[0]), (int)((k / n3) % n2), (int)(k % n3)};
    double e[3], a[3];
    // x = np.linspace(0, L, n): i * step, the last node exactly L; source position i_s * h
    for (int ax = 0; ax < g.dim; ++ax) {
      const double x = i[ax] == g.n[ax] - 1 ? g.L[ax] : (double)i[ax] * g.h[ax];
      e[ax] = x - (double)g.src[ax] * g.h[ax];
      a[ax] = tau_d1(tau1, k, st[ax], i[ax], g.n[ax], g.h[ax]);
    }
    const double t1 = tau1[k];
    const bool at_src = i[0] == g.src[0] && i[1] == g.src[1] && (g.dim == 2 || i[2] == g.src[2]);
    double r, l0;
    if (g.dim == 2) {
      r = glibc_hypot(e[0], e[1]);  // AnalyticBase: tau0 = hypot, lap(tau0) = 1/r
      l0 = r > 0 ? 1.0 / r : 0.0;
    } else {  // per-axis generalisation: lap(tau0) = (d - 1)/r = 2/r
      r = sqrt(e[0] * e[0] + e[1] * e[1] + e[2] * e[2]);
      l0 = r > 0 ? 2.0 / r : 0.0;
    }
    double lap1 = tau_d2(tau1, k, st[0], i[0], n1, g.h[0]) + tau_d2(tau1, k, st[1], i[1], n2, g.h[1]);
    if (g.dim == 3) lap1 = lap1 + tau_d2(tau1, k, st[2], i[2], n3, g.h[2]);
    double s = (r > 0 ? e[0] / r : 0.0) * a[0] + (r > 0 ? e[1] / r : 0.0) * a[1];
    if (g.dim == 3) s = s + (r > 0 ? e[2] / r : 0.0) * a[2];
    double* gr[3] = {gr0, gr1, gr2};
    for (int ax = 0; ax < g.dim; ++ax) {
      const double gax = r > 0 ? e[ax] / r : 0.0;
      gr[ax][k] = at_src ? 0.0 : r * a[ax] + t1 * gax;
    }
    lap[k] = at_src ? 2.0 * t1 : t1 * l0 + 2.0 * s + r * lap1;
    if (tau) tau[k] = r * t1;
  }
}

void launch_tau_derivs(cudaStream_t s, int dim, const int* n, const double* h, const double* L, const int* src,
                       const double* tau1, double* tau, double* const* grads, double* lap) {
  TauGeom g{};
  g.dim = dim;
  for (int a = 0; a < 3; ++a) {
    g.n[a] = a < dim ? n[a] : 1;
    g.h[a] = a < dim ? h[a] : 1.0;
    g.L[a] = a < dim ? L[a] : 0.0;
    g.src[a] = a < dim ? src[a] : 0;
  }
  const long N = (long)g.n[0] * g.n[1] * g.n[2];
  ++g_launch_count;
  int blocks = (int)((N + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) return;
  k_tau_derivs<<<blocks, 256, 0, s>>>(g, tau1, tau, grads[0], grads[1], dim == 3 ? grads[2] : nullptr, lap);
}

struct PairTab {
  int pos_a[HADR_MAX_OFS], pos_b[HADR_MAX_OFS], bit[HADR_MAX_OFS];
  int nslot;
};
// Pair compression (setup): one pass over the owned rows of the union planes.
// Slot q holds union plane pos_a[q], or for a pair (pos_b[q] >= 0) whichever of
// pos_a / pos_b is non-zero in the row, with code bit bit[q] set for pos_b.
__global__ void k_pair_compress(StencilDev A, PairTab t, cplx* __restrict__ pcoef, long pstr,
                                uint8_t* __restrict__ pcode, int* conflict) {
  const long n = (long)A.n1own * A.n2 * A.n3;
  for (long k = (long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (long)gridDim.x * blockDim.x) {
    unsigned code = 0;
    int bad = 0;
    for (int q = 0; q < t.nslot; ++q) {
      const cplx ca = A.coef[(long)t.pos_a[q] * A.pstride + k];
      cplx v = ca;
      if (t.pos_b[q] >= 0) {
        const cplx cb = A.coef[(long)t.pos_b[q] * A.pstride + k];
        const bool nza = ca.x != 0.0 || ca.y != 0.0, nzb = cb.x != 0.0 || cb.y != 0.0;
        bad |= nza && nzb;
        if (nzb) {
          code |= 1u << t.bit[q];
          v = cb;
        }
      }
      pcoef[(long)q * pstr + k] = v;
    }
    pcode[k] = (uint8_t)code;
    if (bad) atomicOr(conflict, 1);
  }
}

void launch_pair_compress(cudaStream_t s, const StencilDev& A, int nslot, const int* pos_a, const int* pos_b,
                          const int* bit, cplx* pcoef, long pstr, uint8_t* pcode, int* conflict) {
  PairTab t{};
  for (int q = 0; q < nslot; ++q) {
    t.pos_a[q] = pos_a[q];
    t.pos_b[q] = pos_b[q];
    t.bit[q] = bit[q];
  }
  t.nslot = nslot;
  const long n = (long)A.n1own * A.n2 * A.n3;
  long b = (n + 255) / 256;
  if (b > 148 * 16) b = 148 * 16;
  k_pair_compress<<<(int)b, 256, 0, s>>>(A, t, pcoef, pstr, pcode, conflict);
}

__global__ void k_class_classify(StencilDev A, int ncls, const unsigned long long* __restrict__ live,
                                 const int* __restrict__ cnsl, const int* __restrict__ mixed,
                                 uint16_t* __restrict__ ccode, unsigned long long* stats) {
  const long n = (long)A.n1own * A.n2 * A.n3;
  unsigned long long slots = 0, nmix = 0;
  int mx = 0;
  for (long k = (long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (long)gridDim.x * blockDim.x) {
    unsigned long long m0 = 0, m1 = 0;
    for (int o = 0; o < A.nofs; ++o) {
      const cplx c = A.coef[(long)o * A.pstride + k];
      if (c.x != 0.0 || c.y != 0.0) {
        if (o < 64)
          m0 |= 1ull << o;
        else
          m1 |= 1ull << (o - 64);
      }
    }
    int cls = ncls - 1;  // the last class (every axis 'both') is the whole union
    for (int c = 0; c < ncls; ++c)
      if ((m0 & ~live[2 * c]) == 0 && (m1 & ~live[2 * c + 1]) == 0) {
        cls = c;
        break;
      }
    ccode[k] = (uint16_t)(cls | (cnsl[cls] << 8));
    slots += cnsl[cls];
    nmix += mixed[cls];
    mx = max(mx, cnsl[cls]);
  }
  for (int o = 16; o > 0; o >>= 1) {
    slots += __shfl_xor_sync(0xffffffffu, slots, o);
    nmix += __shfl_xor_sync(0xffffffffu, nmix, o);
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(stats, slots);
    atomicMax(stats + 1, (unsigned long long)mx);
    atomicAdd(stats + 2, nmix);
  }
}

__global__ void k_class_fill(StencilDev A, const uint16_t* __restrict__ ccode, const int* __restrict__ cnsl,
                             const int* __restrict__ otab, int nsl, cplx* __restrict__ ccoef, long cstr) {
  const long n = (long)A.n1own * A.n2 * A.n3;
  for (long k = (long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (long)gridDim.x * blockDim.x) {
    const int c = ccode[k] & 0xFF;
    const int m = cnsl[c];
    for (int q = 0; q < m; ++q) ccoef[(long)q * cstr + k] = A.coef[(long)otab[c * nsl + q] * A.pstride + k];
  }
}

static int setup_blocks(long n) {
  long b = (n + 255) / 256;
  if (b > 148 * 16) b = 148 * 16;
  return (int)(b < 1 ? 1 : b);
}

void launch_class_classify(cudaStream_t s, const StencilDev& A, int ncls, const unsigned long long* live_dev,
                           const int* cnsl_dev, const int* mixed_dev, uint16_t* ccode, unsigned long long* stats) {
  const long n = (long)A.n1own * A.n2 * A.n3;
  k_class_classify<<<setup_blocks(n), 256, 0, s>>>(A, ncls, live_dev, cnsl_dev, mixed_dev, ccode, stats);
}

void launch_class_fill(cudaStream_t s, const StencilDev& A, const uint16_t* ccode, const int* cnsl_dev,
                       const int* otab_dev, int nsl, cplx* ccoef, long cstr) {
  const long n = (long)A.n1own * A.n2 * A.n3;
  k_class_fill<<<setup_blocks(n), 256, 0, s>>>(A, ccode, cnsl_dev, otab_dev, nsl, ccoef, cstr);
}

// slot layout of the pair-compressed plus-radius-2 union (nofs 9 or 13), see PcLayout
int pair_layout(int nofs, int* pos_a, int* pos_b, int* bit) {
  if (nofs == 9) {
    using L = PcLayout<9>;
    for (int q = 0; q < L::NS; ++q) {
      pos_a[q] = L::first_pos(q);
      pos_b[q] = L::plus_pos(q);
      bit[q] = L::pair(L::first_pos(q));
    }
    return L::NS;
  }
  if (nofs == 13) {
    using L = PcLayout<13>;
    for (int q = 0; q < L::NS; ++q) {
      pos_a[q] = L::first_pos(q);
      pos_b[q] = L::plus_pos(q);
      bit[q] = L::pair(L::first_pos(q));
    }
    return L::NS;
  }
  return 0;
}

__global__ void k_to_c64(long n, const cplx* __restrict__ in, float2* __restrict__ out) {
  for (long k = (long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (long)gridDim.x * blockDim.x) {
    const cplx v = in[k];
    out[k] = make_float2(__double2float_rn(v.x), __double2float_rn(v.y));
  }
}
void launch_to_c64(cudaStream_t s, long n, const cplx* in, float2* out) {
  ++g_launch_count;
  int blocks = (int)((n + 255) / 256);
  if (blocks > 8192) blocks = 8192;
  k_to_c64<<<blocks, 256, 0, s>>>(n, in, out);
}

}  // namespace hadr
