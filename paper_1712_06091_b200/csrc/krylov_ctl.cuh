// Scalar control logic of the Krylov solvers (Givens, least squares, the
// reference's branch decisions), shared by the graph-path epilogues
// (kernels.cu) and the cluster engine (cluster_engine.cu).  Runs on one
// thread; the state may live in global or shared memory.
#pragma once
#include "ctl.cuh"

namespace hadr {

// ---------------------------------------------------------------------------
// scalar helpers for the control epilogues (numpy *scalar* arithmetic is plain,
// non-contracted C: use the no-FMA product)
// ---------------------------------------------------------------------------
__device__ __forceinline__ cplx cneg(cplx a) { return mk(-a.x, -a.y); }
__device__ __forceinline__ double cabs_d(cplx a) { return hypot(a.x, a.y); }

// The state may live in global memory (graph-path epilogues): every routine
// first copies what it needs into registers/local memory with independent
// loads, computes there, and writes the results back — no chain of dependent
// global round trips.

// Givens update of column j (helmadr/krylov.py:195-208) on a local column
// col[0..j+1]; rotations 0..j-1 are given, rotation j is produced.
__device__ __forceinline__ void givens_col(cplx* col, const cplx* csl, const cplx* snl, cplx& csj, cplx& snj, cplx& gj,
                                           cplx& gj1, int j) {
  for (int i = 0; i < j; ++i) {
    const cplx hij = col[i], hi1 = col[i + 1];
    const cplx t = cadd(cmul_sp(csl[i], hij), cmul_sp(snl[i], hi1));
    col[i + 1] = cadd(cmul_sp(cneg(cconj(snl[i])), hij), cmul_sp(cconj(csl[i]), hi1));
    col[i] = t;
  }
  const cplx a = col[j], b = col[j + 1];
  const double aa = cabs_d(a), bb = cabs_d(b);
  const double den = sqrt(aa * aa + bb * bb);
  if (den == 0.0) {
    csj = mk(1.0, 0.0);
    snj = mk(0.0, 0.0);
  } else {
    csj = cdiv_np(cconj(a), mk(den, 0.0));
    snj = cdiv_np(cconj(b), mk(den, 0.0));
  }
  col[j] = cadd(cmul_sp(csj, a), cmul_sp(snj, b));
  col[j + 1] = mk(0.0, 0.0);
  const cplx g = gj;
  gj1 = cmul_sp(cneg(cconj(snj)), g);
  gj = cmul_sp(csj, g);
}

template <int LD>
__device__ void givens_step(cplx* H, cplx* cs, cplx* sn, cplx* g, int j) {
  cplx col[LD + 1], csl[LD], snl[LD];
  for (int i = 0; i <= j + 1; ++i) col[i] = H[i * LD + j];
  for (int i = 0; i < j; ++i) {
    csl[i] = cs[i];
    snl[i] = sn[i];
  }
  cplx gj = g[j], gj1, csj, snj;
  givens_col(col, csl, snl, csj, snj, gj, gj1, j);
  for (int i = 0; i <= j + 1; ++i) H[i * LD + j] = col[i];
  cs[j] = csj;
  sn[j] = snj;
  g[j] = gj;
  g[j + 1] = gj1;
}

// Upper-triangular solve R[:k,:k] y = g[:k], column-oriented like LAPACK ?trsm.
template <int LD>
__device__ void backsolve(const cplx* R, const cplx* g, cplx* y, int k) {
  cplx Rl[LD * LD], yl[LD];
  for (int j = 0; j < k; ++j)
    for (int i = 0; i <= j; ++i) Rl[i * LD + j] = R[i * LD + j];
  for (int i = 0; i < k; ++i) yl[i] = g[i];
  for (int j = k - 1; j >= 0; --j) {
    yl[j] = cdiv_np(yl[j], Rl[j * LD + j]);
    for (int i = 0; i < j; ++i) yl[i] = csub(yl[i], cmul_sp(yl[j], Rl[i * LD + j]));
  }
  for (int i = 0; i < k; ++i) y[i] = yl[i];
}

// ---- Jacobi-GMRES relaxation control (helmadr/krylov.py:91-119) ----
static __device__ void relax_beta(RelaxCtl* c, double ss) {
  double beta = sqrt(ss);
  c->beta = beta;
  c->k = 0;
  for (int i = 0; i <= RMAX; ++i) c->g[i] = mk(0.0, 0.0);
  if (beta == 0.0 || c->steps < 1) {  // helmadr/krylov.py:96-97
    c->cur = kStopped;
    return;
  }
  c->inv_beta = 1.0 / beta;
  c->g[0] = mk(beta, 0.0);
  c->cur = 0;
}

static __device__ void relax_step(RelaxCtl* c, int j, double ss) {
  const double hn = sqrt(ss);
  const double beta = c->beta;
  const int steps = c->steps;
  cplx col[RMAX + 1], csl[RMAX], snl[RMAX];
  for (int i = 0; i <= j; ++i) col[i] = c->H[i * RMAX + j];
  col[j + 1] = mk(hn, 0.0);
  for (int i = 0; i < j; ++i) {
    csl[i] = c->cs[i];
    snl[i] = c->sn[i];
  }
  cplx gj = c->g[j], gj1, csj, snj;
  c->H[(j + 1) * RMAX + j] = mk(hn, 0.0);
  givens_col(col, csl, snl, csj, snj, gj, gj1, j);
  for (int i = 0; i <= j + 1; ++i) c->R[i * RMAX + j] = col[i];
  c->cs[j] = csj;
  c->sn[j] = snj;
  c->g[j] = gj;
  c->g[j + 1] = gj1;
  c->k = j + 1;
  const bool stop = (hn <= kBreakdownEps * beta) || (j + 1 >= steps);  // helmadr/krylov.py:113-114
  if (!stop) {
    c->inv_hn = 1.0 / hn;
    c->cur = j + 1;
    return;
  }
  c->cur = kStopped;
  backsolve<RMAX>(c->R, c->g, c->y, j + 1);
}

// ---- the same control with the state in SHARED memory (cluster engine) ----
// No local copies (the local-array versions above cost a 6 KB stack frame and
// L1/L2 round trips per element); identical arithmetic in identical order, so
// the results are bit-identical to givens_col / backsolve.
template <int LD>
__device__ __forceinline__ void givens_col_sm(const cplx* H, cplx* R, const cplx* cs, const cplx* sn, cplx hnext,
                                              cplx& csj, cplx& snj, cplx& gj, cplx& gj1, int j) {
  // column j of H (rows 0..j; row j+1 = hnext), rotated by cs/sn[0..j-1] into R
  cplx a = H[j];  // H[0 * LD + j]
  for (int i = 0; i < j; ++i) {
    const cplx b = H[(i + 1) * LD + j];
    const cplx ci = cs[i], si = sn[i];
    const cplx t = cadd(cmul_sp(ci, a), cmul_sp(si, b));
    a = cadd(cmul_sp(cneg(cconj(si)), a), cmul_sp(cconj(ci), b));
    R[i * LD + j] = t;
  }
  const cplx b = hnext;
  const double aa = cabs_d(a), bb = cabs_d(b);
  const double den = sqrt(aa * aa + bb * bb);
  if (den == 0.0) {
    csj = mk(1.0, 0.0);
    snj = mk(0.0, 0.0);
  } else {
    csj = cdiv_np(cconj(a), mk(den, 0.0));
    snj = cdiv_np(cconj(b), mk(den, 0.0));
  }
  R[j * LD + j] = cadd(cmul_sp(csj, a), cmul_sp(snj, b));
  R[(j + 1) * LD + j] = mk(0.0, 0.0);
  const cplx g = gj;
  gj1 = cmul_sp(cneg(cconj(snj)), g);
  gj = cmul_sp(csj, g);
}

template <int LD>
__device__ void backsolve_sm(const cplx* R, const cplx* g, cplx* y, int k) {
  for (int i = 0; i < k; ++i) y[i] = g[i];
  for (int j = k - 1; j >= 0; --j) {
    const cplx yj = cdiv_np(y[j], R[j * LD + j]);
    y[j] = yj;
    for (int i = 0; i < j; ++i) y[i] = csub(y[i], cmul_sp(yj, R[i * LD + j]));
  }
}

static __device__ void relax_step_sm(RelaxCtl* c, int j, double ss) {
  const double hn = sqrt(ss);
  const double beta = c->beta;
  const int steps = c->steps;
  c->H[(j + 1) * RMAX + j] = mk(hn, 0.0);
  cplx gj = c->g[j], gj1, csj, snj;
  givens_col_sm<RMAX>(c->H, c->R, c->cs, c->sn, mk(hn, 0.0), csj, snj, gj, gj1, j);
  c->cs[j] = csj;
  c->sn[j] = snj;
  c->g[j] = gj;
  c->g[j + 1] = gj1;
  c->k = j + 1;
  const bool stop = (hn <= kBreakdownEps * beta) || (j + 1 >= steps);  // helmadr/krylov.py:113-114
  if (!stop) {
    c->inv_hn = 1.0 / hn;
    c->cur = j + 1;
    return;
  }
  c->cur = kStopped;
  backsolve_sm<RMAX>(c->R, c->g, c->y, j + 1);
}

// ---- inner FGMRES(2) control (helmadr/krylov.py:142-231, helmadr/multigrid.py:159-167) ----
template <class F>
__device__ void fg_init(F* f, double ss) {
  double bn = sqrt(ss);
  f->bnorm = bn;
  f->it = 0;
  f->k = 0;
  f->cycle = 0;
  f->broke = 0;
  f->note = 0;
  f->reo = 0;
  f->nhist = 0;
  for (int i = 0; i < (F::LD + 1) * F::LD; ++i) f->H[i] = mk(0.0, 0.0);
  for (int i = 0; i <= F::LD; ++i) f->g[i] = mk(0.0, 0.0);
  if (bn == 0.0) {  // helmadr/krylov.py:143-145
    f->path = FG_ZERO;
    return;
  }
  f->rnorm = bn;  // r = b - A*0 = b
  f->target = f->tol * bn;
  f->g[0] = mk(bn, 0.0);
  f->inv_r = 1.0 / bn;
  f->path = FG_A;
}

template <class F>
__device__ void fg_solve_y(F* f) {
  int k = f->k;
  if (k == 1) {
    f->y[0] = cdiv_np(f->g[0], f->H[0]);  // g[:1] / H[0, 0]
  } else if (k > 1) {
    backsolve<F::LD>(f->H, f->g, f->y, k);  // np.linalg.solve on the rotated (triangular) H
  }
}

template <class F>
__device__ void fg_post(F* f, int j) {
  constexpr int LD = F::LD;
  f->reo = 0;
  const double wn = f->wn;
  f->H[(j + 1) * LD + j] = mk(wn, 0.0);
  if (!isfinite(wn)) {  // helmadr/krylov.py:186-190
    f->note = 1;
    f->broke = 1;
    f->k = j;
  } else {
    const bool lucky = wn <= kBreakdownEps * fmax(f->bnorm, 1e-300);
    if (!lucky) f->inv_w = 1.0 / wn;
    cplx col[LD + 1], csl[LD], snl[LD];
    for (int i = 0; i <= j; ++i) col[i] = f->H[i * LD + j];
    col[j + 1] = mk(wn, 0.0);
    for (int i = 0; i < j; ++i) {
      csl[i] = f->cs[i];
      snl[i] = f->sn[i];
    }
    cplx gj = f->g[j], gj1, csj, snj;
    const double target = f->target;
    const int cycle = f->cycle;
    givens_col(col, csl, snl, csj, snj, gj, gj1, j);
    for (int i = 0; i <= j + 1; ++i) f->H[i * LD + j] = col[i];
    f->cs[j] = csj;
    f->sn[j] = snj;
    f->g[j] = gj;
    f->g[j + 1] = gj1;
    f->it += 1;
    f->k = j + 1;
    const double h = cabs_d(gj1);
    if (f->nhist < 8) f->hist[f->nhist++] = h;
    const bool stop = lucky || h <= target;
    if (cycle == 0 && j == 0 && !stop) {  // m = 2: second iteration of the first cycle
      f->path = FG_CONT;
      return;
    }
  }
  fg_solve_y(f);
  f->path = (f->cycle == 0 && j == 0) ? FG_BRK : FG_FIN;
}

// fg_post with shared-memory state: H is rotated in place (R == H), as the reference does
template <class F>
__device__ void fg_post_sm(F* f, int j) {
  constexpr int LD = F::LD;
  f->reo = 0;
  const double wn = f->wn;
  f->H[(j + 1) * LD + j] = mk(wn, 0.0);
  if (!isfinite(wn)) {  // helmadr/krylov.py:186-190
    f->note = 1;
    f->broke = 1;
    f->k = j;
  } else {
    const bool lucky = wn <= kBreakdownEps * fmax(f->bnorm, 1e-300);
    if (!lucky) f->inv_w = 1.0 / wn;
    cplx gj = f->g[j], gj1, csj, snj;
    givens_col_sm<LD>(f->H, f->H, f->cs, f->sn, mk(wn, 0.0), csj, snj, gj, gj1, j);
    f->cs[j] = csj;
    f->sn[j] = snj;
    f->g[j] = gj;
    f->g[j + 1] = gj1;
    f->it += 1;
    f->k = j + 1;
    const double h = cabs_d(gj1);
    if (f->nhist < 8) f->hist[f->nhist++] = h;
    const bool stop = lucky || h <= f->target;
    if (f->cycle == 0 && j == 0 && !stop) {  // m = 2: second iteration of the first cycle
      f->path = FG_CONT;
      return;
    }
  }
  const int k = f->k;
  if (k == 1)
    f->y[0] = cdiv_np(f->g[0], f->H[0]);
  else if (k > 1)
    backsolve_sm<LD>(f->H, f->g, f->y, k);
  f->path = (f->cycle == 0 && j == 0) ? FG_BRK : FG_FIN;
}

template <class F>
__device__ void fg_res(F* f, double ss) {
  double rn = sqrt(ss);
  f->rnorm = rn;
  if (f->broke) {
    f->path = FG_DONE;
    return;
  }
  if (f->it < 2 && rn > f->target) {  // while it < maxiter and rnorm > target: restart with m = 1
    f->path = FG_RST;
    f->cycle = 1;
    f->k = 0;
    for (int i = 0; i < (F::LD + 1) * F::LD; ++i) f->H[i] = mk(0.0, 0.0);
    for (int i = 0; i <= F::LD; ++i) f->g[i] = mk(0.0, 0.0);
    f->g[0] = mk(rn, 0.0);
    f->inv_r = 1.0 / rn;
  } else {
    f->path = FG_DONE;
  }
}


}  // namespace hadr
