// Shared device helpers for the amplitude-solve kernels (sm_100a).
//
// Complex values are stored interleaved (re, im) as double2 — the memory
// layout of numpy complex128, so host buffers copy in without repacking.
//
// Two complex multiplies are provided because the reference gets its
// arithmetic from two different places and we reproduce both bit for bit:
//   cmul_sp : scipy sparsetools' complex_wrapper (no FMA contraction):
//             re = ar*br - ai*bi, im = ar*bi + ai*br   — csr_matvec / csc_matvec
//   cmul_np : numpy's SIMD complex multiply on x86-64 (measured in this image):
//             re = fma(ar, br, -(ai*bi)), im = fma(ar, bi, ai*br)
//             — every "array * array" / "scalar * array" in helmadr/krylov.py
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#ifndef HADR_MAX_OFS
#define HADR_MAX_OFS 125  // offsets in the 5x5(x5) box: 2D unions reach 21, 3D coarse upwind 81
#endif

typedef double2 cplx;

__host__ __device__ __forceinline__ cplx mk(double r, double i) { return make_double2(r, i); }

__device__ __forceinline__ cplx cmul_sp(cplx a, cplx b) {
  return mk(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
            __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}
__device__ __forceinline__ cplx cmul_np(cplx a, cplx b) {
  return mk(__fma_rn(a.x, b.x, -__dmul_rn(a.y, b.y)), __fma_rn(a.x, b.y, __dmul_rn(a.y, b.x)));
}
__device__ __forceinline__ cplx cadd(cplx a, cplx b) { return mk(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y)); }
__device__ __forceinline__ cplx csub(cplx a, cplx b) { return mk(__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y)); }
__device__ __forceinline__ cplx cscale(cplx a, double s) { return mk(__dmul_rn(a.x, s), __dmul_rn(a.y, s)); }
__device__ __forceinline__ cplx cconj(cplx a) { return mk(a.x, -a.y); }
// numpy complex division (Smith's algorithm, no FMA; numpy loops.c.src)
__host__ __device__ __forceinline__ cplx cdiv_np(cplx a, cplx b) {
  double br = b.x, bi = b.y;
  double abr = br < 0 ? -br : br, abi = bi < 0 ? -bi : bi;
  if (abr >= abi) {
    if (abr == 0 && abi == 0) return mk(a.x / abr, a.y / abr);
    double rat = bi / br;
    double scl = 1.0 / (br + bi * rat);
    return mk((a.x + a.y * rat) * scl, (a.y - a.x * rat) * scl);
  }
  double rat = br / bi;
  double scl = 1.0 / (bi + br * rat);
  return mk((a.x * rat + a.y) * scl, (a.y * rat - a.x) * scl);
}
__host__ __device__ __forceinline__ double cabs2(cplx a) { return a.x * a.x + a.y * a.y; }

// ---------------------------------------------------------------------------
// Device-side gating: a kernel runs iff (*active != 0) and (mask >> *var) & 1.
// Either pointer may be null (= unconditional).  Gates carry the data-dependent
// branches of the reference (breakdown, re-orthogonalisation, early exits) so
// that a whole K-cycle can be captured once as a CUDA graph with no host sync.
// ---------------------------------------------------------------------------
struct Gate {
  const int* active;
  const int* var;
  unsigned mask;
  const int* var2;
  unsigned mask2;
};
__host__ __device__ __forceinline__ Gate gate_always() { return Gate{nullptr, nullptr, 0u, nullptr, 0u}; }
__host__ __device__ __forceinline__ Gate gate_on(const int* active) { return Gate{active, nullptr, 0u, nullptr, 0u}; }
__host__ __device__ __forceinline__ Gate gate_var(const int* active, const int* var, unsigned mask) {
  return Gate{active, var, mask, nullptr, 0u};
}
__host__ __device__ __forceinline__ Gate gate_var2(const int* active, const int* var, unsigned mask, const int* var2,
                                                   unsigned mask2) {
  return Gate{active, var, mask, var2, mask2};
}
__device__ __forceinline__ bool gate_bit(const int* var, unsigned mask) {
  if (!var) return true;
  int v = *((volatile const int*)var);
  if (v < 0 || v > 31) return false;
  return (mask >> v) & 1u;
}
__device__ __forceinline__ bool gate_open(const Gate& g) {
  if (g.active && *((volatile const int*)g.active) == 0) return false;
  return gate_bit(g.var, g.mask) && gate_bit(g.var2, g.mask2);
}

// ---------------------------------------------------------------------------
// Grid reductions: every block writes NV partial sums, the last block to
// arrive (atomic ticket) sums the partials in a fixed order — deterministic for
// a fixed grid size — and then runs the caller's scalar epilogue.
// ---------------------------------------------------------------------------
struct RedScratch {
  double* partials;   // >= max_blocks * 4
  unsigned* ticket;   // one counter, reset by the last block
};

constexpr int kThreads = 256;

template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* sm /* NV*32 */) {
#pragma unroll
  for (int q = 0; q < NV; ++q) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[q] += __shfl_xor_sync(0xffffffffu, v[q], o);
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q) sm[q * 32 + wid] = v[q];
  }
  __syncthreads();
  if (wid == 0) {
    const int nw = blockDim.x >> 5;
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      double t = lane < nw ? sm[q * 32 + lane] : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      v[q] = t;
    }
  }
  __syncthreads();
}

// Returns true in the (whole) last block; `out` then holds the grid totals.
template <int NV>
__device__ __forceinline__ bool grid_sum(double (&v)[NV], RedScratch rs, double (&out)[NV]) {
  __shared__ double sm[NV * 32];
  __shared__ int last;
  block_sum<NV>(v, sm);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q) rs.partials[blockIdx.x * NV + q] = v[q];
    __threadfence();
    unsigned t = atomicAdd(rs.ticket, 1u);
    last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return false;
  __threadfence();
  double acc[NV];
#pragma unroll
  for (int q = 0; q < NV; ++q) acc[q] = 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) {
#pragma unroll
    for (int q = 0; q < NV; ++q) acc[q] += ((volatile double*)rs.partials)[b * NV + q];
  }
  block_sum<NV>(acc, sm);
  __shared__ double tot[NV];
  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q) tot[q] = acc[q];
    *rs.ticket = 0u;
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < NV; ++q) out[q] = tot[q];
  return true;
}

// Programmatic dependent launch (PDL): solve-phase kernels are launched with
// programmatic stream serialization, so the next kernel of the chain is scheduled
// while this one runs; every such kernel first waits for its predecessor's
// completion (griddepcontrol.wait: full completion + memory visibility) and then
// allows its own successor to launch.  Both are no-ops without the attribute.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;\n\tgriddepcontrol.launch_dependents;" ::: "memory");
}

#define HADR_CUDA(call)                                                     \
  do {                                                                      \
    cudaError_t e_ = (call);                                                \
    if (e_ != cudaSuccess) throw hadr::CudaError(e_, #call, __FILE__, __LINE__); \
  } while (0)
