// Cluster engine: the coarse part of the K-cycle as ONE persistent kernel on
// one thread-block cluster (16 CTAs x 384 threads, non-portable cluster size).
//
// Why: on the coarse grids (<= ~32k points) every Krylov/multigrid operation
// is latency-bound.  As separate kernels each op costs ~5 us (launch + a chain
// of dependent global-memory round trips for gates, scalars and the reduction
// epilogue).  Inside one cluster an op costs one DSMEM all-reduce (~0.55 us
// measured) or one cluster barrier (~0.34 us): the Krylov control state (the
// Hessenberg matrices, Givens rotations, branch decisions of
// helmadr/krylov.py:91-242 and helmadr/multigrid.py:132-171) lives in shared
// memory, computed redundantly and identically by every CTA from the same
// deterministic all-reduced values, so control flow is uniform with no
// global-memory round trip.
//
// Arithmetic is exactly the graph path's (same element formulas, same
// reduction algebra), so the two paths agree to rounding in the reductions'
// association only.
#include "cluster_engine.h"
#include "krylov_ctl.cuh"

#include <set>

namespace hadr {

struct CEShared {
  double pslot[2][CE_CTAS][4];  // all-reduce: CTA r's total, pushed here by CTA r (double-buffered)
  double bsum[4 * 32];
  int ph[CE_THREADS / 32];      // per-warp parity of the all-reduce slot buffers
  int prof_on;
  int cgs2;                     // relaxations orthogonalise by CGS2 (two batched reductions per step)
  alignas(16) double rout[32];  // batched all-reduce: cluster totals (read as complex pairs)
  double vslot[2][32];          // batched all-reduce: this CTA's partials (read by every CTA)
  double rin[32];                    // batched all-reduce: this CTA's partials (warp 0)
  double wpart[CE_THREADS / 32][2];  // per-warp partial sums of the batched dots
  RelaxCtl rc;            // the (single) live relaxation
  FgCtl2 fg[CE_MAXLEV];   // one inner FGMRES(2) per level (nested)
  CELevel lv[CE_MAXLEV];
  int nlev, coarse_steps;
  double coarse_tol;
};

// The engine's state lives in shared memory (ce_S) and special registers only: nothing
// per thread in local memory.  (A per-thread context struct passed by reference into the
// __noinline__ phases lived in the stack frame — every access an LDL / generic load, and
// every cluster barrier invalidates L1 (CCTL.IVALL), so those reloads went to L2.)
__shared__ CEShared ce_S;
constexpr int CE_CGS_MAX = 10;  // relaxations up to this length orthogonalise by CGS2 (when on)
constexpr int CE_CGS_FROM = 4;  // ... from this step on

struct CEC {};  // phase functions keep a context parameter; all state is in ce_S / special registers

__device__ __forceinline__ unsigned ce_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned ce_nctas() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ long ce_gtid() { return (long)blockIdx.x * blockDim.x + threadIdx.x; }
__device__ __forceinline__ long ce_gstride() { return (long)gridDim.x * blockDim.x; }

// Phase profile of the engine (hadr_ce_profile): cycles seen by CTA 0 — thread 0, except
// slot 3 (relaxation control), owned by the control thread (blockDim.x - 1).  Every slot
// pair (cycles, count) has a single writer thread.  Slots: 0 total, 1 all-reduce, 3 relaxation
// control, 5 stencil, 7 launches, 8 vector ops, 10 barriers, 12 transfers, 14 lincomb,
// 16 stencil on levels > 8192 points, 18 / 20 shared-memory relaxation staging / stencil
// rows on levels > 8192 points, 22 / 24 the same on smaller levels, 26 all-reduce cluster-
// barrier wait, 28 inner-FGMRES control (thread 0), 30 CGS2 orthogonalisation of the relaxations.
constexpr int CE_NPROF = 48;
__device__ unsigned long long g_ce_prof[CE_NPROF];
// CTA 0's thread 0 (and, for slot 3, its control thread) count when profiling is on
__device__ __forceinline__ unsigned long long* ce_prof() {
  return (ce_S.prof_on && blockIdx.x == 0 && threadIdx.x == 0) ? g_ce_prof : nullptr;
}
__device__ __forceinline__ unsigned long long* ce_prof_ctl() {
  return (ce_S.prof_on && blockIdx.x == 0 && threadIdx.x == blockDim.x - 1) ? g_ce_prof : nullptr;
}
struct CEProfScope {
  unsigned long long* p;
  int slot;
  long long t0;
  __device__ CEProfScope(const CEC&, int s) : p(ce_prof()), slot(s), t0(0) {
    if (p) t0 = clock64();
  }
  __device__ CEProfScope(unsigned long long* q, int s) : p(q), slot(s), t0(0) {
    if (p) t0 = clock64();
  }
  __device__ void stop() {
    if (p) {
      p[slot] += clock64() - t0;
      p[slot + 1] += 1;
      p = nullptr;
    }
  }
  __device__ ~CEProfScope() { stop(); }
};

__device__ __forceinline__ void ce_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// standalone barrier between vector ops (profiled as slot 10)
#define CE_SYNC(c)                 \
  do {                             \
    CEProfScope prof_sync_(c, 10); \
    ce_sync();                     \
  } while (0)
// mutable vectors are read through L2 (written by other CTAs of the cluster)
__device__ __forceinline__ cplx ldm(const cplx* p, long i) { return __ldcg(p + i); }
__device__ __forceinline__ cplx ldk(const cplx* p, long i) { return __ldg(p + i); }

__device__ __forceinline__ void ce_store_remote(double* p, unsigned rank, double v) {
  unsigned long long in = reinterpret_cast<unsigned long long>(p), out;
  asm volatile("mapa.u64 %0, %1, %2;" : "=l"(out) : "l"(in), "r"(rank));
  *reinterpret_cast<volatile double*>(out) = v;
}

// Cluster all-reduce of NV doubles: every thread of every CTA ends with bit-identical
// totals.  Per CTA: warp partials (shuffle tree) -> warp 0 sums them in warp order and
// PUSHES the CTA total into slot [rank] of every CTA (DSMEM stores, issued before the
// barrier's release) -> cluster barrier -> every warp sums the 16 local slots in rank
// order (the same shuffle tree in every warp and CTA).  No DSMEM load sits behind the
// barrier and no block barrier follows it (the pull version read the 16 remote slots
// from warp 0 after the barrier and broadcast through shared memory + __syncthreads).
// Slots are double-buffered: a CTA pushes into a parity again only two all-reduces
// later, after a barrier every thread reaches only once its reads of that parity are done.
template <int NV>
__device__ void ce_allreduce(CEC& c, double (&v)[NV]) {
  CEProfScope prof_(c, 1);
  CEShared* S = &ce_S;
#pragma unroll
  for (int q = 0; q < NV; ++q) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[q] += __shfl_xor_sync(0xffffffffu, v[q], o);
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int ph = S->ph[wid];
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q) S->bsum[q * 32 + wid] = v[q];
  }
  __syncthreads();
  if (wid == 0) {
    const int nw = blockDim.x >> 5;
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      double t = lane < nw ? S->bsum[q * 32 + lane] : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      if (lane < (int)ce_nctas()) ce_store_remote(&S->pslot[ph][ce_rank()][q], lane, t);
    }
  }
  {
    CEProfScope prof_w_(c, 26);
    ce_sync();
  }
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    double t = lane < (int)ce_nctas() ? S->pslot[ph][lane][q] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    v[q] = t;
  }
  __syncwarp();
  if (lane == 0) S->ph[wid] = ph ^ 1;
  __syncwarp();
}

// Batched all-reduce of the nv (<= 32) CTA partials in ce_S.rin: every CTA ends with the
// cluster totals in ce_S.rout, lane q of warp 0 adding the 16 CTAs' value q in rank order
// (identical operations in every CTA: bit-identical totals).
__device__ __forceinline__ double ce_remote(const double* p, unsigned rank) {
  unsigned long long in = reinterpret_cast<unsigned long long>(p), out;
  asm volatile("mapa.u64 %0, %1, %2;" : "=l"(out) : "l"(in), "r"(rank));
  return *reinterpret_cast<const volatile double*>(out);
}
// Barrier of the worker warps only (all but the CTA's last warp, the relaxation control
// warp): named barrier 1, so the control thread's Givens update of the previous step is
// not waited for by the intra-step syncs of the shared-memory relaxation.
__device__ __forceinline__ void ce_worker_sync() {
  asm volatile("bar.sync 1, %0;" ::"r"(blockDim.x - 32) : "memory");
}

// CTA partials of nd complex dots <V_i, w> (i < nd; V_i = V + i * vs) over the CTA's np own
// points, plus (norm) the real ||w||^2: dot i -> rin[2i], rin[2i+1], the norm -> rin[2 nd].
// One dot per group of worker warps (the control warp takes none), each warp over a
// contiguous chunk of the points, lanes strided; the per-warp sums are combined in warp
// order by thread d < nd(+1) of warp 0: deterministic.  Worker warps only; rin is
// complete for warp 0 when this returns.
__device__ __forceinline__ void ce_dots_cta(const cplx* V, long vs, int nd, const cplx* w, long np, bool norm) {
  CEShared* S = &ce_S;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nww = (blockDim.x >> 5) - 1;  // worker warps
  const int ndt = nd + (norm ? 1 : 0);
  const int per = nww / ndt;              // warps per dot (>= 1: nd + 1 <= nww, checked by the caller)
  if (wid < ndt * per) {
    const int d = wid / per, part = wid - d * per;
    const long p0 = np * part / per, p1 = np * (part + 1) / per;
    double a = 0.0, b = 0.0;
    if (d < nd) {
      const cplx* u = V + (long)d * vs;
      for (long p = p0 + lane; p < p1; p += 32) {
        const cplx uu = u[p], y = w[p];
        a += uu.x * y.x + uu.y * y.y;
        b += uu.x * y.y - uu.y * y.x;
      }
    } else {
      for (long p = p0 + lane; p < p1; p += 32) {
        const cplx y = w[p];
        a += y.x * y.x + y.y * y.y;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      b += __shfl_xor_sync(0xffffffffu, b, o);
    }
    if (lane == 0) {
      S->wpart[wid][0] = a;
      S->wpart[wid][1] = b;
    }
  }
  ce_worker_sync();
  if ((int)threadIdx.x < ndt) {
    const int d = threadIdx.x;
    double a = S->wpart[d * per][0], b = S->wpart[d * per][1];
    for (int q = 1; q < per; ++q) {
      a += S->wpart[d * per + q][0];
      b += S->wpart[d * per + q][1];
    }
    if (d < nd) {
      S->rin[2 * d] = a;
      S->rin[2 * d + 1] = b;
    } else {
      S->rin[2 * nd] = a;
    }
  }
}

// Batched cluster all-reduce of the nv (<= 32) CTA partials warp 0 holds in ce_S.rin (from
// ce_dots_cta): every CTA ends with the totals in ce_S.rout, value q summed over the CTAs in
// rank order by lane q of warp 0 (identical in every CTA).  All threads take part.
__device__ void ce_allreduce_cta(CEC& c, int nv) {
  CEProfScope prof_(c, 1);
  CEShared* S = &ce_S;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int ph = S->ph[wid];
  __syncwarp();
  if (wid == 0 && lane < nv) S->vslot[ph][lane] = S->rin[lane];
  {
    CEProfScope prof_w_(c, 26);
    ce_sync();
  }
  if (wid == 0 && lane < nv) {
    double r[CE_CTAS];
#pragma unroll
    for (int q = 0; q < CE_CTAS; ++q) r[q] = ce_remote(&S->vslot[ph][lane], q);
    double t = r[0];
#pragma unroll
    for (int q = 1; q < CE_CTAS; ++q) t += r[q];
    S->rout[lane] = t;
  }
  __syncthreads();
  __syncwarp();
  if (lane == 0) S->ph[wid] = ph ^ 1;
  __syncwarp();
}

// ---------------------------------------------------------------------------
// vector operations (same element formulas as kernels.cu)
// ---------------------------------------------------------------------------
// Stencil on a point partition: CTA r owns points [r ppc, (r+1) ppc) of the level grid
// (ce_ppc).  The (transformed) input points within StencilDev::halo of them (the largest
// linear displacement of the offsets) are staged once in shared memory,
// so every neighbour is an LDS instead of an L2 round trip; D^-1 and the scale
// are applied once per point (same values as applying them per neighbour).
// Class-compressed row (StencilDev::ccode, kernels.cu stencil_cc; 3D engine levels): the
// row's class slots in ascending union order; neighbours from the staged tile (linear
// index k - tbase + displacement).
template <bool C32>
__device__ __forceinline__ cplx ce_cc_row(const StencilDev& A, const cplx* tile, long k, long tbase, int i1, int i2,
                                          int i3, int n1, int n2, int n3) {
  const unsigned cw = __ldg(A.ccode + k);
  const int nslc = (int)(cw >> 8);
  const int4* tab = A.ctab + (long)(cw & 0xFFu) * A.nsl;
  cplx acc = mk(0.0, 0.0);
  for (int q0 = 0; q0 < nslc; q0 += 9) {
    int4 t[9];
    cplx cv[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) {
      const bool live = q0 + q < nslc;
      t[q] = __ldg(tab + (live ? q0 + q : 0));
      const long ci = (long)(live ? q0 + q : 0) * A.cstr + k;
      if constexpr (C32) {
        const float2 f = __ldg(A.ccoef32 + ci);
        cv[q] = make_double2((double)f.x, (double)f.y);
      } else {
        cv[q] = __ldg(A.ccoef + ci);
      }
    }
#pragma unroll
    for (int q = 0; q < 9; ++q) {
      const int j1 = i1 + t[q].y, j2 = i2 + t[q].z, j3 = i3 + t[q].w;
      const bool ok = q0 + q < nslc && j1 >= 0 && j1 < n1 && j2 >= 0 && j2 < n2 && j3 >= 0 && j3 < n3;
      const cplx v = tile[ok ? k - tbase + t[q].x : 0];
      const cplx tt = cadd(acc, cmul_sp(cv[q], v));
      acc = ok ? tt : acc;
    }
  }
  return acc;
}

extern __shared__ cplx ce_tile[];

// Fast rows of a standard 2D offset set (Std2D, compile-time offsets): the coefficient
// pointer, sizes and offsets live in registers / immediates (the generic loop re-reads the
// level descriptor from shared memory every point: its smem stores may alias it), and all
// NO coefficient loads of a point are issued together.  Same accumulation order as
// csr_matvec (ascending offsets, no FMA): bit-identical to the generic loop.
// out(k, acc) consumes point k.
// cs != null: the coefficients come from the CTA's shared-memory copy of its own points
// (plane o at cs + o * css, point k at k - own0).
template <int NO, bool C32, bool SMC = false, class F>
__device__ __forceinline__ void ce_rows_std2d(const StencilDev& A, const cplx* tile, long tb, long own0, long own1,
                                              long tw, long nwk, F&& out, const cplx* cs = nullptr, long css = 0) {
  const int n1 = A.n1, n2 = A.n2;
  const long N = (long)n1 * n2;
  const cplx* __restrict__ coef = A.coef;
  const float2* __restrict__ coef32 = A.coef32;
  for (long k = own0 + tw; k < own1; k += nwk) {
    const int i1 = (int)(k / n2), i2 = (int)(k - (long)(k / n2) * n2);
    cplx cv[NO];
#pragma unroll
    for (int o = 0; o < NO; ++o) {
      if constexpr (SMC) {
        cv[o] = cs[(long)o * css + (k - own0)];
      } else if constexpr (C32) {
        const float2 f = __ldg(coef32 + (long)o * N + k);
        cv[o] = make_double2((double)f.x, (double)f.y);
      } else {
        cv[o] = __ldg(coef + (long)o * N + k);
      }
    }
    cplx acc = mk(0.0, 0.0);
#pragma unroll
    for (int o = 0; o < NO; ++o) {
      const int j1 = i1 + Std2D::d1<NO>(o), j2 = i2 + Std2D::d2<NO>(o);
      const bool ok = j1 >= 0 && j1 < n1 && j2 >= 0 && j2 < n2;
      const cplx v = tile[ok ? (long)j1 * n2 + j2 - tb : 0];
      const cplx t = cadd(acc, cmul_sp(cv[o], v));
      acc = ok ? t : acc;
    }
    out(k, acc);
  }
}


template <int NO, int INM, int OUTM, int RED, bool C32>
__device__ void ce_stencil_no(CEC& c, const StencilDev& A, const cplx* x, double s, const cplx* dinv, cplx* vout,
                              const cplx* b, cplx* y, const cplx* u, double (&red)[3]) {
  const int n1 = A.n1, n2 = A.n2, n3 = A.n3, nofs = A.nofs;
  const int n23 = n2 * n3;
  const long N = (long)n1 * n23;
  const long ppc = (N + ce_nctas() - 1) / ce_nctas();
  const long own0 = min(N, (long)ce_rank() * ppc), own1 = min(N, own0 + ppc);
  const long base = max(0L, own0 - A.halo), tn = own1 > own0 ? min(N, own1 + A.halo) - base : 0;
  for (long p = threadIdx.x; p < tn; p += blockDim.x) {
    cplx v = ldm(x, base + p);
    if (INM & IN_SCALE) v = cscale(v, s);
    if (INM & IN_JAC) v = cmul_np(ldk(dinv, base + p), v);
    ce_tile[p] = v;
  }
  __syncthreads();
  if constexpr (NO == 5 || NO == 9 || NO == 21) {
    if (A.std2d == NO) {
      ce_rows_std2d<NO, C32>(A, ce_tile, base, own0, own1, threadIdx.x, blockDim.x, [&](long k, cplx acc) {
        cplx vc = mk(0.0, 0.0);
        if ((INM & IN_WRITEV) || (RED & RED_DOT_CENTER)) {
          vc = ldm(x, k);
          if (INM & IN_SCALE) vc = cscale(vc, s);
          if (INM & IN_WRITEV) vout[k] = vc;
        }
        const cplx yy = (OUTM == OUT_RESID) ? csub(ldm(b, k), acc) : acc;
        y[k] = yy;
        if (RED & RED_NORM) red[0] += yy.x * yy.x + yy.y * yy.y;
        if (RED & (RED_DOT | RED_DOT_CENTER)) {
          const cplx uu = (RED & RED_DOT_CENTER) ? vc : ldm(u, k);
          constexpr int o = (RED & RED_NORM) ? 1 : 0;
          red[o] += uu.x * yy.x + uu.y * yy.y;
          red[o + 1] += uu.x * yy.y - uu.y * yy.x;
        }
      });
      __syncthreads();  // the tile is reused by the next stencil
      return;
    }
  }
  for (long k = own0 + threadIdx.x; k < own1; k += blockDim.x) {
    const int i1 = (int)(k / n23);
    const int rem = (int)(k - (long)i1 * n23);
    const int i2 = rem / n3, i3 = rem - (rem / n3) * n3;
    cplx acc = mk(0.0, 0.0);
    constexpr int CH = NO > 0 ? NO : 9;
    const int nch = (NO == 0 && A.ccode) ? 0 : NO > 0 ? 1 : (nofs + CH - 1) / CH;
    if (NO == 0 && A.ccode) acc = ce_cc_row<C32>(A, ce_tile, k, base, i1, i2, i3, n1, n2, n3);
    for (int ch = 0; ch < nch; ++ch) {
      const int o0 = ch * CH;
      cplx cv[CH];
#pragma unroll
      for (int q = 0; q < CH; ++q) {
        const int o = o0 + q;
        const long ci = o < nofs ? (long)o * N + k : k;
        if constexpr (C32)
          cv[q] = ld_c64(A, ci);
        else
          cv[q] = ldk(A.coef, ci);
      }
#pragma unroll
      for (int q = 0; q < CH; ++q) {
        const int o = o0 + q;
        const int oo = o < nofs ? o : 0;
        const int j1 = i1 + A.d1[oo], j2 = i2 + A.d2[oo], j3 = i3 + A.d3[oo];
        const bool ok = o < nofs && j1 >= 0 && j1 < n1 && j2 >= 0 && j2 < n2 && j3 >= 0 && j3 < n3;
        const cplx v = ce_tile[ok ? ((long)j1 * n2 + j2) * n3 + j3 - base : 0];
        const cplx t = cadd(acc, cmul_sp(cv[q], v));
        acc = ok ? t : acc;
      }
    }
    cplx vc = mk(0.0, 0.0);
    if ((INM & IN_WRITEV) || (RED & RED_DOT_CENTER)) {
      vc = ldm(x, k);
      if (INM & IN_SCALE) vc = cscale(vc, s);
      if (INM & IN_WRITEV) vout[k] = vc;
    }
    const cplx yy = (OUTM == OUT_RESID) ? csub(ldm(b, k), acc) : acc;
    y[k] = yy;
    if (RED & RED_NORM) red[0] += yy.x * yy.x + yy.y * yy.y;
    if (RED & (RED_DOT | RED_DOT_CENTER)) {
      const cplx uu = (RED & RED_DOT_CENTER) ? vc : ldm(u, k);
      constexpr int o = (RED & RED_NORM) ? 1 : 0;
      red[o] += uu.x * yy.x + uu.y * yy.y;
      red[o + 1] += uu.x * yy.y - uu.y * yy.x;
    }
  }
  __syncthreads();  // the tile is reused by the next stencil
}

template <int INM, int OUTM, int RED>
__device__ __noinline__ void ce_stencil(CEC& c, const StencilDev& A, const cplx* x, double s, const cplx* dinv,
                                        cplx* vout, const cplx* b, cplx* y, const cplx* u, double (&red)[3]) {
  CEProfScope prof_(c, 5);
  CEProfScope prof_big_(A.n1 * A.n2 * A.n3 > 8192 ? ce_prof() : nullptr, 16);
  red[0] = red[1] = red[2] = 0.0;
  if (A.coef32) {  // mixed precision: complex64-stored operator
    switch (A.nofs) {
      case 9: ce_stencil_no<9, INM, OUTM, RED, true>(c, A, x, s, dinv, vout, b, y, u, red); break;
      case 21: ce_stencil_no<21, INM, OUTM, RED, true>(c, A, x, s, dinv, vout, b, y, u, red); break;
      default: ce_stencil_no<0, INM, OUTM, RED, true>(c, A, x, s, dinv, vout, b, y, u, red); break;
    }
    return;
  }
  switch (A.nofs) {
    case 5: ce_stencil_no<5, INM, OUTM, RED, false>(c, A, x, s, dinv, vout, b, y, u, red); break;
    case 9: ce_stencil_no<9, INM, OUTM, RED, false>(c, A, x, s, dinv, vout, b, y, u, red); break;
    case 21: ce_stencil_no<21, INM, OUTM, RED, false>(c, A, x, s, dinv, vout, b, y, u, red); break;
    default: ce_stencil_no<0, INM, OUTM, RED, false>(c, A, x, s, dinv, vout, b, y, u, red); break;
  }
}

// w -= h*v ; RED_DOT: <u, w> ; RED_NORM: ||w||^2
template <int RED>
__device__ void ce_axpy(CEC& c, long n, cplx* w, cplx h, const cplx* v, const cplx* u, double (&red)[2]) {
  CEProfScope prof_(c, 8);
  red[0] = red[1] = 0.0;
  for (long k = ce_gtid(); k < n; k += ce_gstride()) {
    const cplx y = csub(ldm(w, k), cmul_np(h, ldm(v, k)));
    w[k] = y;
    if (RED == RED_NORM) {
      red[0] += y.x * y.x + y.y * y.y;
    } else {
      const cplx uu = ldm(u, k);
      red[0] += uu.x * y.x + uu.y * y.y;
      red[1] += uu.x * y.y - uu.y * y.x;
    }
  }
}

__device__ void ce_dot(CEC& c, long n, const cplx* u, const cplx* w, double (&red)[2]) {
  CEProfScope prof_(c, 8);
  red[0] = red[1] = 0.0;
  for (long k = ce_gtid(); k < n; k += ce_gstride()) {
    const cplx uu = ldm(u, k), y = ldm(w, k);
    red[0] += uu.x * y.x + uu.y * y.y;
    red[1] += uu.x * y.y - uu.y * y.x;
  }
}

// out = in * s (s < 0: copy) ; returns ||out||^2 partial
__device__ double ce_scale(CEC& c, long n, const cplx* in, double s, bool scaled, cplx* out) {
  CEProfScope prof_(c, 8);
  double r = 0.0;
  for (long k = ce_gtid(); k < n; k += ce_gstride()) {
    cplx y = ldm(in, k);
    if (scaled) y = cscale(y, s);
    if (out) out[k] = y;
    r += y.x * y.x + y.y * y.y;
  }
  return r;
}

// ---------------------------------------------------------------------------
// Jacobi-GMRES(s) relaxation (helmadr/krylov.py:91-119)
// ---------------------------------------------------------------------------
__device__ __noinline__ void ce_relax(CEC& c, const CELevel& L, const cplx* b, const cplx* x, cplx* xo, int s) {
  RelaxCtl* R = &ce_S.rc;
  const long n = L.N;
  // the control thread: the CTA's last, whose share of the vector work is the smallest
  // (none at all on the coarsest grids), so the Givens updates run beside the other
  // threads' work instead of ahead of it
  const bool ctl = threadIdx.x == blockDim.x - 1;
  if (ctl) {
    R->steps = s;
    R->k = 0;
    R->cur = kStopped;
  }
  // branch state and scales formed locally from the all-reduced values (see ce_relax_sm)
  double beta = 0.0, sc_next = 0.0;
  int cur = kStopped;
  cplx hcol = mk(0.0, 0.0);
  const cplx* r = b;
  {
    double v[1];
    if (x) {
      double red[3];
      ce_stencil<IN_PLAIN, OUT_RESID, RED_NORM>(c, L.A, x, 1.0, nullptr, nullptr, b, L.w[1], nullptr, red);
      v[0] = red[0];
      r = L.w[1];
    } else {
      v[0] = ce_scale(c, n, b, 1.0, false, nullptr);
    }
    ce_allreduce<1>(c, v);
    if (ctl) relax_beta(R, v[0]);
    beta = sqrt(v[0]);
    cur = (beta == 0.0 || s < 1) ? kStopped : 0;
    sc_next = 1.0 / beta;
  }
  for (int j = 0; j < s; ++j) {
    if (cur != j) break;
    cplx* w = L.w[j % 2];
    const cplx* src = (j == 0) ? r : L.w[(j - 1) % 2];
    const double sc = sc_next;
    {
      double red[3];
      if (j == 0)
        ce_stencil<IN_SCALE | IN_JAC | IN_WRITEV, OUT_APPLY, RED_DOT_CENTER>(c, L.A, src, sc, L.dinv, L.V[j], nullptr,
                                                                             w, nullptr, red);
      else
        ce_stencil<IN_SCALE | IN_JAC | IN_WRITEV, OUT_APPLY, RED_DOT>(c, L.A, src, sc, L.dinv, L.V[j], nullptr, w,
                                                                      L.V[0], red);
      double v[2] = {red[0], red[1]};
      ce_allreduce<2>(c, v);
      hcol = mk(v[0], v[1]);
      if (ctl) R->H[0 * RMAX + j] = hcol;
    }
    for (int i = 0; i < j; ++i) {
      double v[2];
      ce_axpy<RED_DOT>(c, n, w, hcol, L.V[i], L.V[i + 1], v);  // h = H[i][j]
      ce_allreduce<2>(c, v);
      hcol = mk(v[0], v[1]);
      if (ctl) R->H[(i + 1) * RMAX + j] = hcol;
    }
    {
      double v2[2];
      ce_axpy<RED_NORM>(c, n, w, hcol, L.V[j], nullptr, v2);  // h = H[j][j]
      double v[1] = {v2[0]};
      ce_allreduce<1>(c, v);
      if (ctl) {
        CEProfScope prof_(ce_prof_ctl(), 3);
        relax_step_sm(R, j, v[0]);
      }
      const double hn = sqrt(v[0]);
      const bool stop = (hn <= kBreakdownEps * beta) || (j + 1 >= s);  // helmadr/krylov.py:113-114
      cur = stop ? kStopped : j + 1;
      sc_next = 1.0 / hn;
    }
  }
  __syncthreads();  // the control thread's y / k
  // xo = x + dinv (.) (V[:k]^T y)
  const int k = R->k;
  CEProfScope prof_lc_(c, 14);
  for (long p = ce_gtid(); p < n; p += ce_gstride()) {
    cplx t = mk(0.0, 0.0);
    for (int i = 0; i < k; ++i) t = cadd(t, cmul_np(ldm(L.V[i], p), R->y[i]));
    t = cmul_np(ldk(L.dinv, p), t);
    xo[p] = x ? cadd(ldm(x, p), t) : cadd(mk(0.0, 0.0), t);
  }
  CE_SYNC(c);
}

// ---------------------------------------------------------------------------
// The same relaxation with every vector of it in shared memory: CTA r keeps its
// own points of the basis V[0..s] and of the Arnoldi vector w (double-buffered);
// the stencil input tile takes its halo points from the neighbouring CTAs' w over
// DSMEM.  Only the right-hand side, the starting guess and the result touch
// global memory.  Element formulas are those of ce_relax (the reductions sum in
// a different order: rounding-level differences only).
// ---------------------------------------------------------------------------
__device__ __forceinline__ cplx ce_remote_c(const cplx* p, unsigned rank) {
  unsigned long long in = reinterpret_cast<unsigned long long>(p), out;
  asm volatile("mapa.u64 %0, %1, %2;" : "=l"(out) : "l"(in), "r"(rank));
  return *reinterpret_cast<const cplx*>(out);
}

template <int NO, bool C32>
__device__ __forceinline__ void sm_stencil_rows(CEC& c, const StencilDev& A, const cplx* tile, long own0, long own1,
                                                long tb, cplx* w, const cplx* v0, double (&red)[2], long tw,
                                                long nwk, const cplx* cs = nullptr, long css = 0) {
  const int n1 = A.n1, n2 = A.n2, n3 = A.n3, nofs = A.nofs;
  const int n23 = n2 * n3;
  const long N = (long)n1 * n23;
  if constexpr (NO == 5 || NO == 9 || NO == 21) {
    if (A.std2d == NO) {
      auto epi = [&](long k, cplx acc) {
        const long p = k - own0;
        w[p] = acc;
        const cplx u = v0[p];
        red[0] += u.x * acc.x + u.y * acc.y;
        red[1] += u.x * acc.y - u.y * acc.x;
      };
      if (!C32 && cs)
        ce_rows_std2d<NO, C32, true>(A, tile, tb, own0, own1, tw, nwk, epi, cs, css);
      else
        ce_rows_std2d<NO, C32, false>(A, tile, tb, own0, own1, tw, nwk, epi);
      return;
    }
  }
  for (long k = own0 + tw; k < own1; k += nwk) {
    const int i1 = (int)(k / n23);
    const int rem = (int)(k - (long)i1 * n23);
    const int i2 = rem / n3, i3 = rem - (rem / n3) * n3;
    cplx acc = mk(0.0, 0.0);
    constexpr int CH = NO > 0 ? NO : 9;
    const int nch = (NO == 0 && A.ccode) ? 0 : NO > 0 ? 1 : (nofs + CH - 1) / CH;
    if (NO == 0 && A.ccode) acc = ce_cc_row<C32>(A, tile, k, tb, i1, i2, i3, n1, n2, n3);
    for (int ch = 0; ch < nch; ++ch) {
      const int o0 = ch * CH;
      cplx cv[CH];
#pragma unroll
      for (int q = 0; q < CH; ++q) {
        const int o = o0 + q;
        const long ci = o < nofs ? (long)o * N + k : k;
        cv[q] = C32 ? ld_c64(A, ci) : ldk(A.coef, ci);
      }
#pragma unroll
      for (int q = 0; q < CH; ++q) {
        const int o = o0 + q;
        const int oo = o < nofs ? o : 0;
        const int j1 = i1 + A.d1[oo], j2 = i2 + A.d2[oo], j3 = i3 + A.d3[oo];
        const bool ok = o < nofs && j1 >= 0 && j1 < n1 && j2 >= 0 && j2 < n2 && j3 >= 0 && j3 < n3;
        const cplx v = tile[ok ? ((long)j1 * n2 + j2) * n3 + j3 - tb : 0];
        const cplx t = cadd(acc, cmul_sp(cv[q], v));
        acc = ok ? t : acc;
      }
    }
    const long p = k - own0;
    w[p] = acc;
    const cplx u = v0[p];
    red[0] += u.x * acc.x + u.y * acc.y;
    red[1] += u.x * acc.y - u.y * acc.x;
  }
}

__device__ __noinline__ void ce_relax_sm(CEC& c, const CELevel& L, const cplx* b, const cplx* x, cplx* xo, int s) {
  RelaxCtl* R = &ce_S.rc;
  const long N = (long)L.A.n1 * L.A.n2 * L.A.n3;
  const long rs = (N + ce_nctas() - 1) / ce_nctas();  // points per CTA = per-buffer stride (ce_ppc)
  const long own0 = min(N, (long)ce_rank() * rs), own1 = min(N, own0 + rs), np = own1 - own0;
  const long tb = max(0L, own0 - L.A.halo), tn = np > 0 ? min(N, own1 + L.A.halo) - tb : 0;
  cplx* tile = ce_tile;                          // tn <= rs + 2 halo points
  cplx* Vb = ce_tile + rs + 2L * L.A.halo;       // V[i] = Vb + i * rs, i <= s
  cplx* wb = Vb + (long)(s + 1) * rs;            // w[0], w[1]
  cplx* cs = L.smc ? wb + 2 * rs : nullptr;      // the CTA's points of the coefficient planes (L.smc)
  // the control warp (the CTA's last) takes no share of the vector work: its last thread
  // runs the Givens / least-squares update of each step while the other warps already
  // stage and apply the next step's stencil, so the update is off the critical path
  const bool ctl = threadIdx.x == blockDim.x - 1;
  const long nwk = blockDim.x - 32;                                   // worker threads
  const long tw = threadIdx.x < nwk ? threadIdx.x : (long)1 << 40;    // this thread's first point (none: ctl warp)
  const bool cgs2 = ce_S.cgs2 && s <= CE_CGS_MAX && s + 1 <= (int)(blockDim.x >> 5) - 1;
  if (ctl) {
    R->steps = s;
    R->k = 0;
    R->cur = kStopped;
  }
  double beta = 0.0, sc_next = 0.0;
  int cur = kStopped;
  cplx hcol = mk(0.0, 0.0);
  {
    double v[1];
    const cplx* src = b;
    if (x) {
      double red[3];
      ce_stencil<IN_PLAIN, OUT_RESID, RED_NORM>(c, L.A, x, 1.0, nullptr, nullptr, b, L.w[1], nullptr, red);
      v[0] = red[0];
      src = L.w[1];  // written by this CTA's own points (the point partition of ce_stencil)
    }
    double nn = 0.0;
    for (long p = tw; p < np; p += nwk) {
      const cplx y = ldm(src, own0 + p);
      wb[rs + p] = y;  // w[1] = r : the "previous" buffer of step 0
      nn += y.x * y.x + y.y * y.y;
    }
    if (cs) {  // stage the own points of the nofs coefficient planes once for the s stencils
      for (int o = 0; o < L.A.nofs; ++o)
        for (long p = tw; p < np; p += nwk) cs[(long)o * rs + p] = ldk(L.A.coef, (long)o * N + own0 + p);
    }  // (read after the staging barrier of step 0)
    if (!x) v[0] = nn;
    ce_allreduce<1>(c, v);
    if (ctl) relax_beta(R, v[0]);
    // every thread holds the all-reduced value: the branch state and the scale are formed
    // locally (the same IEEE operations as relax_beta / relax_step_sm), so no thread waits
    // for thread 0's control update — it is read back only after the loop
    beta = sqrt(v[0]);
    cur = (beta == 0.0 || s < 1) ? kStopped : 0;
    sc_next = 1.0 / beta;
  }
  for (int j = 0; j < s; ++j) {
    if (cur != j) break;
    const double sc = sc_next;
    cplx* wp = wb + (long)((j + 1) % 2) * rs;  // previous Arnoldi vector (step 0: r)
    cplx* w = wb + (long)(j % 2) * rs;
    cplx* Vj = Vb + (long)j * rs;
    // CGS2 from the 5th step on: two batched all-reduces (~2 us each) replace MGS's j + 2
    // (~1.7 us each); below that MGS is cheaper (measured)
    const bool cg = cgs2 && j >= CE_CGS_FROM;
    {
      CEProfScope prof_(c, 5);
      const bool big = N > 8192;
      CEProfScope prof_st_(ce_prof(), big ? 18 : 22);
      // V[j] = wp * sc (own points); tile = D^-1 (.) (wp * sc) on points [tb, tb + tn)
      for (long q = tw; q < tn; q += nwk) {
        const long g = tb + q;
        cplx v;
        if (g >= own0 && g < own1) {
          v = cscale(wp[g - own0], sc);
          Vj[g - own0] = v;
        } else {  // halo point owned by another CTA: its previous w over DSMEM
          const unsigned owner = (unsigned)(g / rs);
          const cplx* rw = wb + (long)((j + 1) % 2) * rs + (g - (long)owner * rs);
          v = cscale(ce_remote_c(rw, owner), sc);
        }
        tile[q] = cmul_np(ldk(L.dinv, g), v);
      }
      if (threadIdx.x < blockDim.x - 32) ce_worker_sync();  // the control warp neither stages nor applies
      prof_st_.stop();
      CEProfScope prof_rows_(ce_prof(), big ? 20 : 24);
      double red[2] = {0.0, 0.0};
      const cplx* V0 = Vb;
      if (cg) V0 = Vj;  // the epilogue's dot is discarded: batched dots follow
      if (L.A.coef32) {
        if (L.A.nofs == 21)
          sm_stencil_rows<21, true>(c, L.A, tile, own0, own1, tb, w, V0, red, tw, nwk);
        else if (L.A.nofs == 9)
          sm_stencil_rows<9, true>(c, L.A, tile, own0, own1, tb, w, V0, red, tw, nwk);
        else
          sm_stencil_rows<0, true>(c, L.A, tile, own0, own1, tb, w, V0, red, tw, nwk);
      } else {
        switch (L.A.nofs) {
          case 5: sm_stencil_rows<5, false>(c, L.A, tile, own0, own1, tb, w, V0, red, tw, nwk, cs, rs); break;
          case 9: sm_stencil_rows<9, false>(c, L.A, tile, own0, own1, tb, w, V0, red, tw, nwk, cs, rs); break;
          case 21: sm_stencil_rows<21, false>(c, L.A, tile, own0, own1, tb, w, V0, red, tw, nwk, cs, rs); break;
          default: sm_stencil_rows<0, false>(c, L.A, tile, own0, own1, tb, w, V0, red, tw, nwk); break;
        }
      }
      if (!cg) {
        double v[2] = {red[0], red[1]};
        ce_allreduce<2>(c, v);
        hcol = mk(v[0], v[1]);
        if (ctl) R->H[0 * RMAX + j] = hcol;
      }
    }
    if (cg) {
      // CGS2 (two batched projections; algebraically the MGS loop below):
      // h = V^H w ; w' = w - V h ; c = V^H w', ||w'||^2 ; w'' = w' - V c ;
      // H[:, j] = h + c ; ||w''||^2 = ||w'||^2 - |c|^2 (c is at rounding level of ||w'||:
      // no cancellation; an explicit norm when it is not).  Intra-CTA syncs are worker-only.
      CEProfScope prof_cg_(c, 30);
      const int nd = j + 1;
      const cplx* hv = reinterpret_cast<const cplx*>(ce_S.rout);
      CEProfScope ps1(ce_prof(), 32);
      if (threadIdx.x < blockDim.x - 32) {  // worker warps
        ce_worker_sync();  // w of every own point
        ce_dots_cta(Vb, rs, nd, w, np, false);
      }
      ps1.stop();
      CEProfScope ps2(ce_prof(), 34);
      ce_allreduce_cta(c, 2 * nd);
      ps2.stop();
      CEProfScope ps3(ce_prof(), 36);
      if (ctl)
        for (int i = 0; i < nd; ++i) R->H[i * RMAX + j] = hv[i];
      for (long p = tw; p < np; p += nwk) {
        cplx y = w[p];
        for (int i = 0; i < nd; ++i) y = csub(y, cmul_np(hv[i], Vb[(long)i * rs + p]));
        w[p] = y;
      }
      ps3.stop();
      CEProfScope ps4(ce_prof(), 38);
      if (threadIdx.x < blockDim.x - 32) {  // worker warps
        ce_worker_sync();  // w' complete
        ce_dots_cta(Vb, rs, nd, w, np, true);
      }
      ps4.stop();
      CEProfScope ps5(ce_prof(), 40);
      ce_allreduce_cta(c, 2 * nd + 1);
      ps5.stop();
      CEProfScope ps6(ce_prof(), 42);
      double cc = 0.0;
      for (int i = 0; i < nd; ++i) cc += hv[i].x * hv[i].x + hv[i].y * hv[i].y;
      const double n2 = ce_S.rout[2 * nd];
      double nn = 0.0;
      for (long p = tw; p < np; p += nwk) {
        cplx y = w[p];
        for (int i = 0; i < nd; ++i) y = csub(y, cmul_np(hv[i], Vb[(long)i * rs + p]));
        w[p] = y;
        nn += y.x * y.x + y.y * y.y;
      }
      if (ctl)
        for (int i = 0; i < nd; ++i) R->H[i * RMAX + j] = cadd(R->H[i * RMAX + j], hv[i]);
      ps6.stop();
      CEProfScope ps7(ce_prof(), 44);
      double hn2;
      if (cc <= 1e-8 * n2) {
        hn2 = n2 - cc;
        CE_SYNC(c);  // w'' of every CTA before the neighbours read its halo points
      } else {       // heavy cancellation: the explicit norm (its all-reduce is the barrier)
        double v[1] = {nn};
        ce_allreduce<1>(c, v);
        hn2 = v[0];
      }
      if (ctl) {  // Givens, least squares (the control thread)
        CEProfScope prof_(ce_prof_ctl(), 3);
        relax_step_sm(R, j, hn2);
      }
      const double hn = sqrt(hn2);
      const bool stop = (hn <= kBreakdownEps * beta) || (j + 1 >= s);  // helmadr/krylov.py:113-114
      cur = stop ? kStopped : j + 1;
      sc_next = 1.0 / hn;
      continue;
    }
    for (int i = 0; i < j; ++i) {
      const cplx h = hcol;  // H[i][j], the previous all-reduce
      const cplx* Vi = Vb + (long)i * rs;
      const cplx* Vi1 = Vb + (long)(i + 1) * rs;
      double v[2] = {0.0, 0.0};
      for (long p = tw; p < np; p += nwk) {
        const cplx y = csub(w[p], cmul_np(h, Vi[p]));
        w[p] = y;
        const cplx uu = Vi1[p];
        v[0] += uu.x * y.x + uu.y * y.y;
        v[1] += uu.x * y.y - uu.y * y.x;
      }
      ce_allreduce<2>(c, v);
      hcol = mk(v[0], v[1]);
      if (ctl) R->H[(i + 1) * RMAX + j] = hcol;
    }
    {
      const cplx h = hcol;  // H[j][j]
      double v[1] = {0.0};
      for (long p = tw; p < np; p += nwk) {
        const cplx y = csub(w[p], cmul_np(h, Vj[p]));
        w[p] = y;
        v[0] += y.x * y.x + y.y * y.y;
      }
      ce_allreduce<1>(c, v);
      if (ctl) {  // Givens, least squares (the control thread)
        CEProfScope prof_(ce_prof_ctl(), 3);
        relax_step_sm(R, j, v[0]);
      }
      const double hn = sqrt(v[0]);
      const bool stop = (hn <= kBreakdownEps * beta) || (j + 1 >= s);  // helmadr/krylov.py:113-114
      cur = stop ? kStopped : j + 1;
      sc_next = 1.0 / hn;
    }
  }
  __syncthreads();  // the control thread's y / k
  // xo = x + dinv (.) (V[:k]^T y)   (own points)
  const int k = R->k;
  {
    CEProfScope prof_lc_(c, 14);
    for (long p = tw; p < np; p += nwk) {
      cplx t = mk(0.0, 0.0);
      for (int i = 0; i < k; ++i) t = cadd(t, cmul_np(Vb[(long)i * rs + p], R->y[i]));
      t = cmul_np(ldk(L.dinv, own0 + p), t);
      xo[own0 + p] = x ? cadd(ldm(x, own0 + p), t) : cadd(mk(0.0, 0.0), t);
    }
  }
  CE_SYNC(c);
}

__device__ __forceinline__ void ce_relax_any(CEC& c, const CELevel& L, const cplx* b, const cplx* x, cplx* xo,
                                             int s) {
  if (L.smr)
    ce_relax_sm(c, L, b, x, xo, s);
  else
    ce_relax(c, L, b, x, xo, s);
}

// ---------------------------------------------------------------------------
// transfer operators (bit-exact orders, see kernels.cu)
// ---------------------------------------------------------------------------
__device__ __noinline__ void ce_restrict(CEC& c, int n1f, int n2f, int n3f, const cplx* r, cplx* rc) {
  CEProfScope prof_(c, 12);
  const int n1c = (n1f - 1) / 2 + 1, n2c = (n2f - 1) / 2 + 1, n3c = (n3f - 1) / 2 + 1;
  const long Nc = (long)n1c * n2c * n3c;
  const int c3lo = n3f > 1 ? -1 : 0, c3hi = n3f > 1 ? 1 : 0;
  for (long q = ce_gtid(); q < Nc; q += ce_gstride()) {
    const int I1 = (int)(q / ((long)n2c * n3c));
    const int rem = (int)(q - (long)I1 * n2c * n3c);
    const int I2 = rem / n3c, I3 = rem - (rem / n3c) * n3c;
    cplx acc = mk(0.0, 0.0);
    for (int a = -1; a <= 1; ++a) {
      const int f1 = 2 * I1 + a;
      if (f1 < 0 || f1 >= n1f) continue;
      const double w1 = a == 0 ? 1.0 : 0.5;
      for (int bb = -1; bb <= 1; ++bb) {
        const int f2 = 2 * I2 + bb;
        if (f2 < 0 || f2 >= n2f) continue;
        const double w12 = w1 * (bb == 0 ? 1.0 : 0.5);
        for (int cc = c3lo; cc <= c3hi; ++cc) {
          const int f3 = 2 * I3 + cc;
          if (f3 < 0 || f3 >= n3f) continue;
          const double w = w12 * (cc == 0 ? 1.0 : 0.5);
          acc = cadd(acc, cmul_sp(mk(w, 0.0), ldm(r, ((long)f1 * n2f + f2) * n3f + f3)));
        }
      }
    }
    rc[q] = acc;
  }
}

__device__ __forceinline__ int ce_parents(int f, int* p, double& w) {
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

__device__ __noinline__ void ce_prolong_add(CEC& c, int n1f, int n2f, int n3f, const cplx* ec, cplx* x) {
  CEProfScope prof_(c, 12);
  const int n2c = (n2f - 1) / 2 + 1, n3c = (n3f - 1) / 2 + 1;
  const int n23 = n2f * n3f;
  const long Nf = (long)n1f * n23;
  for (long f = ce_gtid(); f < Nf; f += ce_gstride()) {
    const int f1 = (int)(f / n23);
    const int rem = (int)(f - (long)f1 * n23);
    const int f2 = rem / n3f, f3 = rem - (rem / n3f) * n3f;
    int c1[2], c2[2], c3[2];
    double w1, w2, w3;
    const int m1 = ce_parents(f1, c1, w1), m2 = ce_parents(f2, c2, w2), m3 = ce_parents(f3, c3, w3);
    cplx p = mk(0.0, 0.0);
    for (int a = 0; a < m1; ++a)
      for (int bb = 0; bb < m2; ++bb)
        for (int cc = 0; cc < m3; ++cc)
          p = cadd(p, cmul_sp(mk(w1 * w2 * w3, 0.0), ldm(ec, ((long)c1[a] * n2c + c2[bb]) * n3c + c3[cc])));
    x[f] = cadd(ldm(x, f), p);
  }
}

// ---------------------------------------------------------------------------
// K-cycle recursion (helmadr/multigrid.py:132-171) and the inner FGMRES(2)
// (helmadr/multigrid.py:159-167 with helmadr/krylov.py:122-242).  Templated on
// the recursion depth so the compiler sees no runtime recursion.
// ---------------------------------------------------------------------------
template <int D>
__device__ void ce_kcycle(CEC& c, int l, const cplx* b, cplx* xo);

// one Arnoldi column j of the inner FGMRES: w = A z against basis B[0..j]
__device__ __noinline__ void ce_arnoldi(CEC& c, FgCtl2* f, const CELevel& L, int j, const cplx* z, const cplx* B0,
                           const cplx* B1) {
  const long n = L.N;
  const cplx* B[2] = {B0, B1};
  {
    double red[3];
    ce_stencil<IN_PLAIN, OUT_APPLY, RED_NORM | RED_DOT>(c, L.A, z, 1.0, nullptr, nullptr, nullptr, L.fw, B0, red);
    double v[3] = {red[0], red[1], red[2]};
    ce_allreduce<3>(c, v);
    if (threadIdx.x == 0) {
      f->w0 = sqrt(v[0]);
      f->H[0 * 2 + j] = mk(v[1], v[2]);
    }
    __syncthreads();
  }
  for (int i = 0; i < j; ++i) {
    double v[2];
    ce_axpy<RED_DOT>(c, n, L.fw, f->H[i * 2 + j], B[i], B[i + 1], v);
    ce_allreduce<2>(c, v);
    if (threadIdx.x == 0) f->H[(i + 1) * 2 + j] = mk(v[0], v[1]);
    __syncthreads();
  }
  {
    double v2[2];
    ce_axpy<RED_NORM>(c, n, L.fw, f->H[j * 2 + j], B[j], nullptr, v2);
    double v[1] = {v2[0]};
    ce_allreduce<1>(c, v);
    if (threadIdx.x == 0) {
      f->wn = sqrt(v[0]);
      f->reo = (f->wn < kReorthRatio * f->w0) ? 1 : 0;  // helmadr/krylov.py:178-179
      if (!f->reo) {
        CEProfScope prof_(c, 28);
        fg_post_sm(f, j);
      }
    }
    __syncthreads();
  }
  if (f->reo) {  // one re-orthogonalisation pass (helmadr/krylov.py:180-184)
    {
      double v[2];
      ce_dot(c, n, B0, L.fw, v);
      ce_allreduce<2>(c, v);
      if (threadIdx.x == 0) {
        f->corr[0] = mk(v[0], v[1]);
        f->H[0 * 2 + j] = cadd(f->H[0 * 2 + j], f->corr[0]);
      }
      __syncthreads();
    }
    for (int i = 0; i < j; ++i) {
      double v[2];
      ce_axpy<RED_DOT>(c, n, L.fw, f->corr[i], B[i], B[i + 1], v);
      ce_allreduce<2>(c, v);
      if (threadIdx.x == 0) {
        f->corr[i + 1] = mk(v[0], v[1]);
        f->H[(i + 1) * 2 + j] = cadd(f->H[(i + 1) * 2 + j], f->corr[i + 1]);
      }
      __syncthreads();
    }
    double v2[2];
    ce_axpy<RED_NORM>(c, n, L.fw, f->corr[j], B[j], nullptr, v2);
    double v[1] = {v2[0]};
    ce_allreduce<1>(c, v);
    if (threadIdx.x == 0) {
      f->wn = sqrt(v[0]);
      fg_post_sm(f, j);
    }
    __syncthreads();
  }
}

template <int D>
__device__ void ce_inner(CEC& c, int ci) {
  CEShared* S = &ce_S;
  const CELevel& C = S->lv[ci];
  FgCtl2* f = &S->fg[ci];
  const long n = C.N;
  if (threadIdx.x == 0) {
    f->tol = S->coarse_tol;
    f->reo = 0;
  }
  {
    double v[1] = {ce_scale(c, n, C.fb, 1.0, false, nullptr)};
    ce_allreduce<1>(c, v);
    if (threadIdx.x == 0) fg_init(f, v[0]);
    __syncthreads();
  }
  if (f->path == FG_ZERO) {
    for (long p = ce_gtid(); p < n; p += ce_gstride()) C.fx[p] = mk(0.0, 0.0);
    CE_SYNC(c);
    return;
  }
  ce_scale(c, n, C.fb, f->inv_r, true, C.fV0);
  CE_SYNC(c);
  ce_kcycle<D>(c, ci, C.fV0, C.fZ0);
  ce_arnoldi(c, f, C, 0, C.fZ0, C.fV0, nullptr);
  if (f->path == FG_BRK) {  // early exit after iteration 1: x = Z0 y0, r = b - A x
    const int k = f->k;
    const cplx y0 = f->y[0];
    for (long p = ce_gtid(); p < n; p += ce_gstride())
      C.fx[p] = (k >= 1) ? cadd(mk(0.0, 0.0), cmul_np(ldm(C.fZ0, p), y0)) : mk(0.0, 0.0);
    CE_SYNC(c);
    double red[3];
    ce_stencil<IN_PLAIN, OUT_RESID, RED_NORM>(c, C.A, C.fx, 1.0, nullptr, nullptr, C.fb, C.fr, nullptr, red);
    double v[1] = {red[0]};
    ce_allreduce<1>(c, v);
    if (threadIdx.x == 0) fg_res(f, v[0]);
    __syncthreads();
  }
  const int path = f->path;
  if (path == FG_CONT || path == FG_RST) {
    if (path == FG_CONT)
      ce_scale(c, n, C.fw, f->inv_w, true, C.fu);
    else
      ce_scale(c, n, C.fr, f->inv_r, true, C.fu);
    CE_SYNC(c);
    ce_kcycle<D>(c, ci, C.fu, C.fZ1);
    if (path == FG_CONT)
      ce_arnoldi(c, f, C, 1, C.fZ1, C.fV0, C.fu);
    else
      ce_arnoldi(c, f, C, 0, C.fZ1, C.fu, nullptr);
  }
  if (f->path == FG_FIN) {
    const int k = f->k, cyc = f->cycle;
    const cplx y0 = f->y[0], y1 = f->y[1];
    for (long p = ce_gtid(); p < n; p += ce_gstride()) {
      cplx out;
      if (cyc == 0) {
        cplx t = mk(0.0, 0.0);
        if (k >= 1) t = cadd(t, cmul_np(ldm(C.fZ0, p), y0));
        if (k >= 2) t = cadd(t, cmul_np(ldm(C.fZ1, p), y1));
        out = cadd(mk(0.0, 0.0), t);
      } else {
        const cplx xp = ldm(C.fx, p);
        out = (k >= 1) ? cadd(xp, cmul_np(ldm(C.fZ1, p), y0)) : xp;
      }
      C.fx[p] = out;
    }
    CE_SYNC(c);
  }
}

template <int D>
__device__ void ce_kcycle(CEC& c, int l, const cplx* b, cplx* xo) {
  if constexpr (D < CE_MAXLEV) {
    CEShared* S = &ce_S;
    const CELevel& L = S->lv[l];
    const CELevel& C = S->lv[l + 1];
    ce_relax_any(c, L, b, nullptr, xo, L.s);
    {
      double red[3];
      ce_stencil<IN_PLAIN, OUT_RESID, RED_NONE>(c, L.A, xo, 1.0, nullptr, nullptr, b, L.r, nullptr, red);
      CE_SYNC(c);
    }
    ce_restrict(c, L.A.n1, L.A.n2, L.A.n3, L.r, C.fb);
    CE_SYNC(c);
    if (l + 1 == S->nlev - 1)
      ce_relax_any(c, C, C.fb, nullptr, C.fx, C.s);  // the level's min(coarse_steps, N)
    else
      ce_inner<D + 1>(c, l + 1);
    ce_prolong_add(c, L.A.n1, L.A.n2, L.A.n3, C.fx, xo);
    CE_SYNC(c);
    ce_relax_any(c, L, b, xo, xo, L.s);
  }
}

__global__ void __launch_bounds__(CE_THREADS, 1)
    k_cluster_engine(const CEDesc* __restrict__ d, int mode, int l0, const cplx* b, cplx* xo, const int* active,
                     int prof) {
  pdl_enter();
  if (active && *((volatile const int*)active) == 0) return;
  CEShared& S = ce_S;
  // level descriptors into shared memory
  {
    const int nw = (int)(sizeof(CELevel) * CE_MAXLEV / sizeof(int));
    const int* src = reinterpret_cast<const int*>(d->lv);
    int* dst = reinterpret_cast<int*>(S.lv);
    for (int i = threadIdx.x; i < nw; i += blockDim.x) dst[i] = src[i];
    if (threadIdx.x == 0) {
      S.nlev = d->nlev;
      S.coarse_steps = d->coarse_steps;
      S.coarse_tol = d->coarse_tol;
      S.prof_on = prof & 1;
      S.cgs2 = (prof >> 1) & 1;
    }
    if ((threadIdx.x & 31) == 0) S.ph[threadIdx.x >> 5] = 0;
  }
  __syncthreads();
  CEC c;
  const long long t_start = clock64();
  if (mode == 0) {
    ce_kcycle<0>(c, l0, b, xo);
  } else if (mode == 1) {
    ce_inner<0>(c, l0);
  } else {
    const CELevel& C = S.lv[l0];
    ce_relax_any(c, C, C.fb, nullptr, C.fx, C.s);
  }
  ce_sync();  // no CTA exits while another may still read its shared memory
  if (unsigned long long* pr = ce_prof()) {
    pr[0] += clock64() - t_start;
    pr[7] += 1;
  }
}

int ce_profile_read(unsigned long long* out, int reset) {
  cudaError_t e = cudaMemcpyFromSymbol(out, g_ce_prof, sizeof(unsigned long long) * CE_NPROF);
  if (e != cudaSuccess) return (int)e;
  if (reset) {
    unsigned long long z[CE_NPROF] = {0};
    e = cudaMemcpyToSymbol(g_ce_prof, z, sizeof(z));
  }
  return (int)e;
}

int g_ce_prof_on = 0;
int g_ce_cgs2 = 1;

extern int g_ce_prof_on;
void launch_cluster_engine(cudaStream_t s, const CEDesc* d, int mode, int l0, const cplx* b, cplx* xo,
                           const int* active, int ctas, size_t tile_bytes) {
  ++g_launch_count;
  static bool init = false;
  static size_t max_tile = 0;
  if (!init) {
    cudaFuncSetAttribute(k_cluster_engine, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    init = true;
  }
  if (tile_bytes > max_tile) {
    cudaFuncSetAttribute(k_cluster_engine, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tile_bytes);
    max_tile = tile_bytes;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = dim3(CE_THREADS);
  cfg.dynamicSmemBytes = tile_bytes;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = ctas;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = g_pdl ? 2 : 1;
  cudaLaunchKernelEx(&cfg, k_cluster_engine, d, mode, l0, b, xo, active, (g_ce_prof_on ? 1 : 0) | (g_ce_cgs2 ? 2 : 0));
}

}  // namespace hadr
