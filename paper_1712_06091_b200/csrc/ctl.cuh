// Device-resident control blocks for the Krylov state machines.
//
// The reference's data-dependent branches (helmadr/krylov.py:96-97, 113-114,
// 177-193, 212; helmadr/multigrid.py:159-167 with the 0.1 early exit) are
// decided on the device by single-thread epilogues that run in the last block
// of each reduction kernel, and are consumed by later kernels through Gates.
#pragma once
#include "common.cuh"

namespace hadr {

constexpr int RMAX = 16;   // max Jacobi-GMRES relaxation length (coarsest default 10)
constexpr int MMAX = 16;   // max FGMRES restart length
constexpr int kStopped = 31;
constexpr double kBreakdownEps = 1e-14;                    // helmadr/krylov.py:13
constexpr double kReorthRatio = 0.70710678118654757;       // 1/sqrt(2), helmadr/krylov.py:12

// Jacobi-preconditioned GMRES(s) relaxation (helmadr/krylov.py:91-119).
struct RelaxCtl {
  int cur;        // gate var: next step index; kStopped when finished / broken down
  int k;          // completed Arnoldi steps
  int steps;      // s = min(steps, n)
  int pad_;
  double beta;
  double inv_beta;
  double inv_hn;  // 1/H[j+1,j] of the last step: V_{j+1} = w * inv_hn
  double pad2_;
  cplx H[(RMAX + 1) * RMAX];  // raw Arnoldi Hessenberg, H[i*RMAX + j]
  cplx R[(RMAX + 1) * RMAX];  // Givens-rotated copy
  cplx cs[RMAX], sn[RMAX];
  cplx g[RMAX + 1];
  cplx y[RMAX];
};

// Flexible GMRES state (helmadr/krylov.py:122-242).  Used in full on the device
// for the inner FGMRES(2) of the K-cycle, and as the Arnoldi scratch of the
// host-driven outer FGMRES.
enum FgPath : int {
  FG_A = 0,        // first iteration of the first cycle
  FG_CONT = 1,     // second iteration of the first cycle (no early exit)
  FG_BRK = 2,      // early exit after iteration 1 -> finalize k=1, residual, maybe restart
  FG_RST = 3,      // restart cycle with m = 1
  FG_FIN = 4,      // cycle complete -> finalize
  FG_DONE = 5,     // x final
  FG_ZERO = 6,     // ||b|| == 0 -> x = 0
};

template <int MM>
struct FgCtlT {
  int path;       // gate var (inner solver)
  int reo;        // gate var: 1 = re-orthogonalisation pass needed
  int it;
  int k;
  int cycle;      // 0 first cycle, 1 restart cycle
  int broke;
  int note;       // 1 = non-finite Arnoldi vector
  int nhist;
  double bnorm, target, rnorm, inv_r;
  double w0, wn, inv_w, tol;
  cplx corr[MM + 1];
  cplx H[(MM + 1) * MM];   // H[i*MM + j], rotated in place as in the reference
  cplx cs[MM], sn[MM];
  cplx g[MM + 1];
  cplx y[MM];
  double hist[8];
  static constexpr int LD = MM;
};
using FgCtl = FgCtlT<MMAX>;   // outer solver scratch / graph-path inner solver
using FgCtl2 = FgCtlT<2>;     // inner FGMRES(2) inside the cluster engine

}  // namespace hadr
