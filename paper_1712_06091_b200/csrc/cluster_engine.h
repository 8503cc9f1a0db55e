// Cluster engine interface (cluster_engine.cu).
#pragma once
#include "kernels.cuh"

namespace hadr {

constexpr int CE_MAXLEV = 6;      // levels a single engine launch may span
#ifndef HADR_CE_THREADS
#define HADR_CE_THREADS 384  // 11 worker warps + the control warp; 168 registers per thread (512: 128, spills)
#endif
constexpr int CE_THREADS = HADR_CE_THREADS;  // threads per CTA
constexpr int CE_CTAS = 16;       // CTAs in the (single, non-portable) cluster

// Device-resident description of one multigrid level for the engine.
struct CELevel {
  StencilDev A;
  const cplx* dinv;
  long N;
  int s;    // relaxation length
  int smr;  // 1: the relaxation runs out of shared memory (ce_relax_sm; see ce_relax_sm_bytes)
  int smc;  // 1: ... and stages the CTA's rows of the coefficient planes there too (ce_relax_smc_bytes)
  cplx* r;
  cplx* V[RMAX + 1];
  cplx* w[2];
  cplx *fb, *fx, *fV0, *fu, *fZ0, *fZ1, *fw, *fr;
};

struct CEDesc {
  int nlev;          // levels described (index 0 = the hierarchy's level `base`)
  int coarse_steps;
  double coarse_tol;
  CELevel lv[CE_MAXLEV];
};

// mode 0: k_cycle(l0, b -> xo) with x = 0
// mode 1: inner FGMRES(2) at level l0 (lv[l0].fb -> lv[l0].fx)
// mode 2: coarsest relaxation at level l0 (lv[l0].fb -> lv[l0].fx)
// phase counters [total cyc, allreduce cyc, n, epilogue cyc, n, stencil cyc, n, launches]
int ce_profile_read(unsigned long long* out, int reset);
extern int g_ce_prof_on;
extern int g_ce_cgs2;  // engine relaxations orthogonalise by CGS2 (batched reductions) instead of MGS
void launch_cluster_engine(cudaStream_t s, const CEDesc* d, int mode, int l0, const cplx* b, cplx* xo,
                           const int* active, int ctas, size_t tile_bytes);
// The engine partitions a level of N points by POINTS: CTA r owns [r ppc, (r+1) ppc),
// ppc = ceil(N / ctas) (a row partition left 129^2 at 9 rows = 1161 points on most CTAs
// against a mean of 1040); a stencil's input tile adds `halo` points on each side.
inline long ce_ppc(long N, int ctas) { return (N + ctas - 1) / ctas; }
// dynamic shared memory for the stencil input tile of a level
inline size_t ce_tile_bytes(long N, int halo, int ctas) {
  return (size_t)(ce_ppc(N, ctas) + 2L * halo) * sizeof(cplx);
}
// shared-memory relaxation with s steps: per CTA the input tile, the basis V[0..s] and two
// w buffers of its own points
inline size_t ce_relax_sm_bytes(long N, int halo, int s, int ctas) {
  return ce_tile_bytes(N, halo, ctas) + (size_t)ce_ppc(N, ctas) * (s + 3) * sizeof(cplx);
}
// ... plus the CTA's points of the nofs coefficient planes (complex128)
inline size_t ce_relax_smc_bytes(long N, int halo, int s, int nofs, int ctas) {
  return ce_relax_sm_bytes(N, halo, s, ctas) + (size_t)ce_ppc(N, ctas) * nofs * sizeof(cplx);
}
constexpr size_t CE_SMEM_BUDGET = 190 * 1024;  // dynamic shared memory the engine may request

}  // namespace hadr
