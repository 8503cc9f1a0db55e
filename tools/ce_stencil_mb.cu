// Microbenchmark: the cluster engine's 129^2 coarse stencil (21-offset Galerkin operator,
// complex128, row slabs over a 16-CTA cluster) — how fast can one CTA stream its
// ~390 KB coefficient block from L2 and apply it?  Variants:
//   0: flat per-point loop, one 21-load chunk per point (the engine's original code)
//   1: register-blocked, KP points x CH planes of loads in flight (KP=3, CH=3)
//   2: register-blocked KP=3, CH=7
//   3: bulk-async (cp.async.bulk) plane segments into a 3-stage shared-memory ring
//      (mbarrier completion), every thread applies the staged plane to its points
//   4: like 3 with 2-stage ring of 2 planes
// Each rep: stage the input tile (own rows + 2 halo rows each side) from global, apply,
// write y, cluster barrier.  Time per rep from CUDA events over the whole launch.
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a --fmad=false -o ce_mb tools/ce_stencil_mb.cu
#include <cstdio>
#include <cuda_runtime.h>
#include <vector>

typedef double2 cplx;
__device__ __forceinline__ cplx mk(double r, double i) { return make_double2(r, i); }
__device__ __forceinline__ cplx cmul_sp(cplx a, cplx b) {
  return mk(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)), __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}
__device__ __forceinline__ cplx cadd(cplx a, cplx b) { return mk(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y)); }

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e = (x);                                                       \
    if (e != cudaSuccess) {                                                    \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      return 1;                                                                \
    }                                                                          \
  } while (0)

constexpr int NO = 21;
__constant__ int c_d1[NO], c_d2[NO];

__device__ __forceinline__ void csync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

extern __shared__ __align__(128) unsigned char smraw[];

template <int KP, int CH>
__device__ __forceinline__ void blocked(const cplx* __restrict__ coef, const cplx* tile, int n1, int n2, int t0,
                                        long own0, long own1, cplx* y, double& chk) {
  const long N = (long)n1 * n2;
  long kk[KP];
  int i1[KP], i2[KP];
  bool live[KP];
#pragma unroll
  for (int p = 0; p < KP; ++p) {
    kk[p] = own0 + threadIdx.x + (long)p * blockDim.x;
    live[p] = kk[p] < own1;
    const long k = live[p] ? kk[p] : own0;
    i1[p] = (int)(k / n2);
    i2[p] = (int)(k - (long)i1[p] * n2);
  }
  cplx acc[KP];
#pragma unroll
  for (int p = 0; p < KP; ++p) acc[p] = mk(0, 0);
#pragma unroll
  for (int o0 = 0; o0 < NO; o0 += CH) {
    cplx cv[KP][CH];
#pragma unroll
    for (int p = 0; p < KP; ++p)
#pragma unroll
      for (int q = 0; q < CH; ++q)
        if (o0 + q < NO) cv[p][q] = __ldg(coef + (long)(o0 + q) * N + (live[p] ? kk[p] : own0));
#pragma unroll
    for (int p = 0; p < KP; ++p)
#pragma unroll
      for (int q = 0; q < CH; ++q) {
        const int o = o0 + q;
        if (o < NO) {
          const int j1 = i1[p] + c_d1[o], j2 = i2[p] + c_d2[o];
          const bool ok = j1 >= 0 && j1 < n1 && j2 >= 0 && j2 < n2;
          const cplx v = tile[ok ? (long)(j1 - t0) * n2 + j2 : 0];
          const cplx t = cadd(acc[p], cmul_sp(cv[p][q], v));
          acc[p] = ok ? t : acc[p];
        }
      }
  }
#pragma unroll
  for (int p = 0; p < KP; ++p)
    if (live[p]) {
      y[kk[p]] = acc[p];
      chk += acc[p].x;
    }
}

__device__ __forceinline__ void flat(const cplx* __restrict__ coef, const cplx* tile, int n1, int n2, int t0,
                                     long own0, long own1, cplx* y, double& chk) {
  const long N = (long)n1 * n2;
  for (long k = own0 + threadIdx.x; k < own1; k += blockDim.x) {
    const int i1 = (int)(k / n2), i2 = (int)(k - (long)i1 * n2);
    cplx cv[NO];
#pragma unroll
    for (int o = 0; o < NO; ++o) cv[o] = __ldg(coef + (long)o * N + k);
    cplx acc = mk(0, 0);
#pragma unroll
    for (int o = 0; o < NO; ++o) {
      const int j1 = i1 + c_d1[o], j2 = i2 + c_d2[o];
      const bool ok = j1 >= 0 && j1 < n1 && j2 >= 0 && j2 < n2;
      const cplx v = tile[ok ? (long)(j1 - t0) * n2 + j2 : 0];
      const cplx t = cadd(acc, cmul_sp(cv[o], v));
      acc = ok ? t : acc;
    }
    y[k] = acc;
    chk += acc.x;
  }
}

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned cnt) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared.b64 P, [%0], %1;\n@!P bra W;\n}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// TMA-staged: NS stages of PPS planes; stage s holds planes [s*PPS, ...) of the CTA's segment
template <int NS, int PPS>
__device__ void staged(const cplx* __restrict__ coef, const cplx* tile, int n1, int n2, int t0, long own0, long own1,
                       cplx* y, double& chk, cplx* ring, unsigned long long* bars, unsigned& phase_bits) {
  const long N = (long)n1 * n2;
  const long np = own1 - own0;
  const unsigned seg = (unsigned)(np * sizeof(cplx));
  constexpr int KP = 3;
  long kk[KP];
  int i1[KP], i2[KP];
  bool live[KP];
  cplx acc[KP];
#pragma unroll
  for (int p = 0; p < KP; ++p) {
    kk[p] = own0 + threadIdx.x + (long)p * blockDim.x;
    live[p] = kk[p] < own1;
    const long k = live[p] ? kk[p] : own0;
    i1[p] = (int)(k / n2);
    i2[p] = (int)(k - (long)i1[p] * n2);
    acc[p] = mk(0, 0);
  }
  constexpr int NG = (NO + PPS - 1) / PPS;  // plane groups
  auto issue = [&](int g) {
    const int st = g % NS;
    const int np_g = min(PPS, NO - g * PPS);
    mbar_expect_tx(&bars[st], seg * np_g);
    for (int q = 0; q < np_g; ++q)
      bulk_g2s(ring + ((long)st * PPS + q) * np, coef + (long)(g * PPS + q) * N + own0, seg, &bars[st]);
  };
  if (threadIdx.x == 0)
    for (int g = 0; g < NS && g < NG; ++g) issue(g);
  for (int g = 0; g < NG; ++g) {
    const int st = g % NS;
    mbar_wait(&bars[st], (phase_bits >> st) & 1u);
    const int np_g = min(PPS, NO - g * PPS);
    for (int q = 0; q < np_g; ++q) {
      const int o = g * PPS + q;
      const cplx* cp = ring + ((long)st * PPS + q) * np;
#pragma unroll
      for (int p = 0; p < KP; ++p) {
        const int j1 = i1[p] + c_d1[o], j2 = i2[p] + c_d2[o];
        const bool ok = live[p] && j1 >= 0 && j1 < n1 && j2 >= 0 && j2 < n2;
        const cplx cvv = cp[live[p] ? kk[p] - own0 : 0];
        const cplx v = tile[ok ? (long)(j1 - t0) * n2 + j2 : 0];
        const cplx t = cadd(acc[p], cmul_sp(cvv, v));
        acc[p] = ok ? t : acc[p];
      }
    }
    phase_bits ^= 1u << st;
    __syncthreads();  // stage st consumed by every thread
    if (threadIdx.x == 0 && g + NS < NG) issue(g + NS);
  }
#pragma unroll
  for (int p = 0; p < KP; ++p)
    if (live[p]) {
      y[kk[p]] = acc[p];
      chk += acc[p].x;
    }
}

__global__ void __launch_bounds__(512, 1) k_bench(int variant, const cplx* __restrict__ coef, const cplx* x, cplx* y,
                                                  int n1, int n2, int reps, double* out) {
  const int C = gridDim.x, rank = blockIdx.x;
  const int R = (n1 + C - 1) / C;
  const int r0 = min(n1, rank * R), r1 = min(n1, r0 + R);
  const int t0 = max(0, r0 - 2), t1 = min(n1, r1 + 2);
  const long own0 = (long)r0 * n2, own1 = (long)r1 * n2;
  cplx* tile = (cplx*)smraw;
  const long tn = (long)(t1 - t0) * n2;
  cplx* ring = tile + ((long)(R + 4) * n2 + 7) / 8 * 8;
  __shared__ unsigned long long bars[4];
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  unsigned phase_bits = 0;
  double chk = 0;
  for (int r = 0; r < reps; ++r) {
    for (long p = threadIdx.x; p < tn; p += blockDim.x) tile[p] = __ldcg(x + (long)t0 * n2 + p);
    __syncthreads();
    switch (variant) {
      case 0: flat(coef, tile, n1, n2, t0, own0, own1, y, chk); break;
      case 1: blocked<3, 3>(coef, tile, n1, n2, t0, own0, own1, y, chk); break;
      case 2: blocked<3, 7>(coef, tile, n1, n2, t0, own0, own1, y, chk); break;
      case 3: staged<3, 1>(coef, tile, n1, n2, t0, own0, own1, y, chk, ring, bars, phase_bits); break;
      case 4: staged<2, 2>(coef, tile, n1, n2, t0, own0, own1, y, chk, ring, bars, phase_bits); break;
      case 5: staged<4, 1>(coef, tile, n1, n2, t0, own0, own1, y, chk, ring, bars, phase_bits); break;
    }
    __syncthreads();
    csync();
  }
  if (chk == 12345.678) out[0] = chk;
}

// ---- all-reduce floor: push version (as cluster_engine.cu), NV doubles, no work between ----
struct ARS {
  double pslot[2][16][4];
  double bsum[4 * 32];
};
__device__ __forceinline__ void st_remote(double* p, unsigned rank, double v) {
  unsigned long long in = reinterpret_cast<unsigned long long>(p), out;
  asm volatile("mapa.u64 %0, %1, %2;" : "=l"(out) : "l"(in), "r"(rank));
  *reinterpret_cast<volatile double*>(out) = v;
}
template <int NV>
__device__ __forceinline__ void allred(ARS* S, int& ph, double (&v)[NV], int sync_first) {
#pragma unroll
  for (int q = 0; q < NV; ++q)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[q] += __shfl_xor_sync(0xffffffffu, v[q], o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const unsigned rank = blockIdx.x, C = gridDim.x;
  if (sync_first) {
    if (lane == 0)
#pragma unroll
      for (int q = 0; q < NV; ++q) S->bsum[q * 32 + wid] = v[q];
    __syncthreads();
    if (wid == 0) {
      const int nw = blockDim.x >> 5;
#pragma unroll
      for (int q = 0; q < NV; ++q) {
        double t = lane < nw ? S->bsum[q * 32 + lane] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (lane < (int)C) st_remote(&S->pslot[ph][rank][q], lane, t);
      }
    }
  } else {  // no block barrier: only warp 0 contributes (floor of the cluster part)
    if (wid == 0)
#pragma unroll
      for (int q = 0; q < NV; ++q)
        if (lane < (int)C) st_remote(&S->pslot[ph][rank][q], lane, v[q]);
  }
  csync();
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    double t = lane < (int)C ? S->pslot[ph][lane][q] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    v[q] = t;
  }
  ph ^= 1;
}
// pull version (the engine's round-1 all-reduce): block sum -> own slot -> barrier -> warp 0
// reads the 16 remote slots -> smem -> __syncthreads
struct ARP {
  double slot[2][4];
  double tot[4];
  double bsum[4 * 32];
};
__device__ __forceinline__ double ld_remote(const double* p, unsigned rank) {
  unsigned long long in = reinterpret_cast<unsigned long long>(p), out;
  asm volatile("mapa.u64 %0, %1, %2;" : "=l"(out) : "l"(in), "r"(rank));
  return *reinterpret_cast<const volatile double*>(out);
}
template <int NV>
__device__ __forceinline__ void allred_pull(ARP* S, int& ph, double (&v)[NV]) {
#pragma unroll
  for (int q = 0; q < NV; ++q)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[q] += __shfl_xor_sync(0xffffffffu, v[q], o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const unsigned C = gridDim.x;
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < NV; ++q) S->bsum[q * 32 + wid] = v[q];
  __syncthreads();
  if (wid == 0) {
    const int nw = blockDim.x >> 5;
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      double t = lane < nw ? S->bsum[q * 32 + lane] : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      if (lane == 0) S->slot[ph][q] = t;
    }
  }
  csync();
  if (wid == 0) {
    double t[NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) t[q] = lane < (int)C ? ld_remote(&S->slot[ph][q], lane) : 0.0;
#pragma unroll
    for (int q = 0; q < NV; ++q) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t[q] += __shfl_xor_sync(0xffffffffu, t[q], o);
      if (lane == 0) S->tot[q] = t[q];
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < NV; ++q) v[q] = S->tot[q];
  ph ^= 1;
}

// st.async version: the pushes land in the remote CTA's slots and complete_tx its mbarrier;
// no cluster barrier.  WARPS: 0 -> warp 0 pushes the block sum (after __syncthreads);
// 1 -> every warp pushes its own partial (no block barrier), every warp sums 16 x nw slots.
struct ARA {
  double slot[2][16 * 16][4];
  double bsum[4 * 32];
  unsigned long long bar[2];
};
__device__ __forceinline__ void st_async_f64(double* remote_local_addr, unsigned rank, double v,
                                             unsigned long long* bar_local) {
  unsigned a = (unsigned)__cvta_generic_to_shared(remote_local_addr), b = (unsigned)__cvta_generic_to_shared(bar_local);
  unsigned ra, rb;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(b), "r"(rank));
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(ra), "d"(v), "r"(rb)
               : "memory");
}
template <int NV, int ALLW>
__device__ __forceinline__ void allred_async(ARA* S, int& k, double (&v)[NV]) {
#pragma unroll
  for (int q = 0; q < NV; ++q)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[q] += __shfl_xor_sync(0xffffffffu, v[q], o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const unsigned C = gridDim.x, rank = blockIdx.x;
  const int ph = k & 1;
  const unsigned par = (k >> 1) & 1;
  if (threadIdx.x == 0) {
    const unsigned bytes = (ALLW ? C * nw : C) * NV * 8;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                     (unsigned)__cvta_generic_to_shared(&S->bar[ph])),
                 "r"(bytes)
                 : "memory");
  }
  if (ALLW) {
    if (lane < (int)C)
#pragma unroll
      for (int q = 0; q < NV; ++q) st_async_f64(&S->slot[ph][rank * nw + wid][q], lane, v[q], &S->bar[ph]);
  } else {
    if (lane == 0)
#pragma unroll
      for (int q = 0; q < NV; ++q) S->bsum[q * 32 + wid] = v[q];
    __syncthreads();
    if (wid == 0) {
#pragma unroll
      for (int q = 0; q < NV; ++q) {
        double t = lane < nw ? S->bsum[q * 32 + lane] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (lane < (int)C) st_async_f64(&S->slot[ph][rank][q], lane, t, &S->bar[ph]);
      }
    }
  }
  asm volatile(
      "{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W;\n}\n" ::"r"(
          (unsigned)__cvta_generic_to_shared(&S->bar[ph])),
      "r"(par)
      : "memory");
  const int ns = ALLW ? C * nw : C;
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    double t = 0.0;
    for (int i = lane; i < ns; i += 32) t += S->slot[ph][i][q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    v[q] = t;
  }
  ++k;
}

__global__ void __launch_bounds__(512, 1) k_allred(int variant, int reps, double* out) {
  __shared__ ARS S;
  __shared__ ARP SP;
  __shared__ ARA SA;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&SA.bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  csync();
  int ph = 0;
  double v[2] = {threadIdx.x * 1e-3, blockIdx.x * 1.0};
  for (int r = 0; r < reps; ++r) {
    if (variant == 0) allred<2>(&S, ph, v, 1);
    else if (variant == 1) allred<2>(&S, ph, v, 0);
    else if (variant == 2) csync();
    else if (variant == 3) allred_pull<2>(&SP, ph, v);
    else if (variant == 4) allred_async<2, 0>(&SA, ph, v);
    else allred_async<2, 1>(&SA, ph, v);
    v[0] *= 0.5;
    v[1] *= 0.5;
  }
  csync();
  if (v[0] == 12345.678) out[0] = v[1];
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 129;
  if (n == 0) {  // all-reduce floor
    double* o;
    CK(cudaMalloc(&o, 8));
    CK(cudaFuncSetAttribute(k_allred, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    const char* names[6] = {"push all-reduce (block sum + DSMEM push + barrier + local sum)",
                            "warp-0 push only (no __syncthreads)", "cluster barrier alone",
                            "pull all-reduce (round 1: barrier + remote reads + __syncthreads)",
                            "st.async + mbarrier, block sum pushed by warp 0",
                            "st.async + mbarrier, every warp pushes its partial"};
    for (int v = 0; v < 6; ++v)
      for (int threads : {512, 256}) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(16);
        cfg.blockDim = dim3(threads);
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 16;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        const int reps = 20000;
        CK(cudaLaunchKernelEx(&cfg, k_allred, v, 100, o));
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        CK(cudaEventRecord(e0));
        CK(cudaLaunchKernelEx(&cfg, k_allred, v, reps, o));
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        printf("%s, %d threads: %.3f us\n", names[v], threads, ms * 1e3 / reps);
      }
    return 0;
  }
  const int reps = 200;
  const long N = (long)n * n;
  int d1[NO], d2[NO], q = 0;
  for (int a = -2; a <= 2; ++a)
    for (int b = -2; b <= 2; ++b)
      if (!(abs(a) == 2 && abs(b) == 2)) d1[q] = a, d2[q] = b, ++q;
  CK(cudaMemcpyToSymbol(c_d1, d1, sizeof(d1)));
  CK(cudaMemcpyToSymbol(c_d2, d2, sizeof(d2)));
  std::vector<cplx> h(NO * N);
  for (long i = 0; i < NO * N; ++i) h[i] = make_double2((i % 7) * 0.1, (i % 5) * 0.2);
  cplx *coef, *x, *y;
  double* out;
  CK(cudaMalloc(&coef, NO * N * sizeof(cplx)));
  CK(cudaMalloc(&x, N * sizeof(cplx)));
  CK(cudaMalloc(&y, N * sizeof(cplx)));
  CK(cudaMalloc(&out, 8));
  CK(cudaMemcpy(coef, h.data(), NO * N * sizeof(cplx), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(x, h.data(), N * sizeof(cplx), cudaMemcpyHostToDevice));
  const int C = 16;
  const int R = (n + C - 1) / C;
  const size_t tile_b = ((size_t)(R + 4) * n + 7) / 8 * 8 * sizeof(cplx);
  const size_t seg_b = (size_t)R * n * sizeof(cplx);
  CK(cudaFuncSetAttribute(k_bench, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CK(cudaFuncSetAttribute(k_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  printf("n=%d rows/CTA=%d coef bytes/CTA=%.1f KB tile=%.1f KB\n", n, R, NO * seg_b / 1024.0, tile_b / 1024.0);
  std::vector<cplx> ref(N), got(N);
  for (int v = 0; v <= 5; ++v) {
    size_t smem = tile_b + (v == 3 ? 3 : v == 4 ? 4 : v == 5 ? 4 : 0) * seg_b;
    if (smem > 200 * 1024) {
      printf("variant %d needs %.1f KB smem: skipped\n", v, smem / 1024.0);
      continue;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(C);
    cfg.blockDim = dim3(512);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, k_bench, v, (const cplx*)coef, (const cplx*)x, y, n, n, 5, out));
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0));
    CK(cudaLaunchKernelEx(&cfg, k_bench, v, (const cplx*)coef, (const cplx*)x, y, n, n, reps, out));
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    CK(cudaMemcpy(got.data(), y, N * sizeof(cplx), cudaMemcpyDeviceToHost));
    if (v == 0) ref = got;
    double diff = 0;
    for (long i = 0; i < N; ++i) diff += fabs(got[i].x - ref[i].x) + fabs(got[i].y - ref[i].y);
    printf("variant %d: %.2f us per rep (stage tile + stencil + cluster barrier), diff vs 0: %g\n", v,
           ms * 1e3 / reps, diff);
  }
  return 0;
}
