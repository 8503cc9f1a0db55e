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
// dynamic shared memory for the stencil row tiles of levels with n1 x n2 points
inline size_t ce_tile_bytes(int n1, int n2, int ctas) {
  return (size_t)((n1 + ctas - 1) / ctas + 4) * n2 * sizeof(cplx);
}
// shared-memory relaxation of a level with n1 rows of n23 points and s steps: per CTA the
// input tile (rows + 4 halo rows), the basis V[0..s] and two w buffers of its own rows
inline size_t ce_relax_sm_bytes(int n1, long n23, int s, int ctas) {
  const long rows = (n1 + ctas - 1) / ctas;
  return (size_t)(rows * (s + 3) + rows + 4) * n23 * sizeof(cplx);
}
// ... plus the CTA's rows of the nofs coefficient planes (complex128)
inline size_t ce_relax_smc_bytes(int n1, long n23, int s, int nofs, int ctas) {
  const long rows = (n1 + ctas - 1) / ctas;
  return ce_relax_sm_bytes(n1, n23, s, ctas) + (size_t)rows * n23 * nofs * sizeof(cplx);
}
constexpr size_t CE_SMEM_BUDGET = 190 * 1024;  // dynamic shared memory the engine may request

}  // namespace hadr
