// extern "C" boundary (include/hadr.h).  Plain pointers and sizes only.
#include <cstring>
#include <string>

#include "../../include/hadr.h"
#include "dist.h"
#include "engine.h"

using namespace hadr;

struct hadr_op_s {
  Op* op;
  bool own;
};
struct hadr_hier_s {
  Hier* h;
  std::vector<hadr_op_s> level_handles;
};

static thread_local std::string g_err;

template <class F>
static int guarded(F&& f) {
  try {
    f();
    return HADR_OK;
  } catch (const ValueError& e) {
    g_err = e.what();
    return HADR_EVALUE;
  } catch (const CudaError& e) {
    g_err = e.what();
    return HADR_ECUDA;
  } catch (const std::exception& e) {
    g_err = e.what();
    return HADR_ERUNTIME;
  } catch (...) {
    g_err = "unknown error";
    return HADR_ERUNTIME;
  }
}

// Device view of a complex vector: borrowed (on_device) or a staged copy.
struct DevVec {
  cplx* p = nullptr;
  bool owned = false;
  long n = 0;
  DevVec(const double* src, long n_, int on_device, bool copy_in) : n(n_) {
    if (on_device || (copy_in && !src)) {
      p = (cplx*)src;
    } else {
      p = dalloc<cplx>(n);
      owned = true;
      if (copy_in && src) {
        Ctx& c = Ctx::get();
        HADR_CUDA(cudaMemcpyAsync(p, src, n * sizeof(cplx), cudaMemcpyHostToDevice, c.stream));
      }
    }
  }
  void copy_out(double* dst) {
    if (!owned) return;
    Ctx& c = Ctx::get();
    HADR_CUDA(cudaMemcpyAsync(dst, p, n * sizeof(cplx), cudaMemcpyDeviceToHost, c.stream));
  }
  ~DevVec() {
    if (owned) dfree(p);
  }
};

static hadr_op wrap(Op* op, bool own = true) { return new hadr_op_s{op, own}; }

namespace hadr {
void accuracy_stats(long n, const cplx* u, const cplx* ref, double floor_in, double* err_dev, double* floor_out,
                    long long* count_out, const long long* idx, int nidx, double* vals_out);  // accuracy.cu
int64_t fast_march(int dim, const int* n, const double* h, const double* tau0, const double* const* g0,
                   const double* kappa, const int* src, int order, double* tau1_out);  // eikonal.cpp
}

// Multi-GPU solve_adr_upwind: slab assembly, slab hierarchy with agglomerated coarse
// levels, distributed FGMRES; every rank passes the global inputs and receives the
// global amplitude (rows gathered from their owners).
static void solve_adr_upwind_dist(int dim, int n1, int n2, int n3, double h1, double h2, double h3, double omega,
                                  const int* bc, int src1, int src2, int src3, const double* ksq, const double* gam,
                                  const double* g1, const double* g2, const double* g3, const double* lap,
                                  const double* qhat, double beta, int levels, int restart, int maxiter, double tol,
                                  double* a_out, Report& r, double* t_setup, int on_device) {
  Ctx& c = Ctx::get();
  Comm* cm = dist_comm();
  const int rk = cm->rank, R = cm->size;
  const SlabPlan plan = slab_plan(n1, n2, n3, levels);
  const int p0 = plan.bounds[rk], nown = plan.bounds[rk + 1] - p0;
  const long n23 = (long)n2 * n3, N = (long)n1 * n23, nloc = (long)nown * n23, hh = (long)kHalo * n23;
  cudaEvent_t e0, e1;
  HADR_CUDA(cudaEventCreate(&e0));
  HADR_CUDA(cudaEventCreate(&e1));
  HADR_CUDA(cudaEventRecord(e0, c.stream));
  Op *H2 = nullptr, *H1 = nullptr, *B = nullptr;
  Hier* hier = nullptr;
  cplx *b = nullptr, *x = nullptr, *full = nullptr;
  auto cleanup = [&]() {
    delete H1;
    delete B;
    delete hier;
    delete H2;
    dfree(b);
    dfree(x);
    dfree(full);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  };
  try {
    H2 = op_assemble_slab(dim, n1, n2, n3, h1, h2, h3, omega, 2, bc, src1, src2, src3, ksq, gam, g1, g2, g3, lap,
                          on_device, p0, nown);
    H1 = op_assemble_slab(dim, n1, n2, n3, h1, h2, h3, omega, 1, bc, src1, src2, src3, ksq, gam, g1, g2, g3, lap,
                          on_device, p0, nown);
    B = op_axpby(mk(1.0 - beta, 0.0), *H2, mk(beta, 0.0), *H1);
    delete H1;
    H1 = nullptr;
    hier = hier_build_dist(B, plan, 10, 0.1);
    delete B;
    B = nullptr;
    HADR_CUDA(cudaEventRecord(e1, c.stream));
    HADR_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    HADR_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    if (t_setup) *t_setup = ms * 1e-3;
    b = dalloc<cplx>(nloc + 2 * hh) + hh;
    x = dalloc<cplx>(nloc + 2 * hh) + hh;
    HADR_CUDA(cudaMemsetAsync(x - hh, 0, (nloc + 2 * hh) * sizeof(cplx), c.stream));
    HADR_CUDA(cudaMemcpyAsync(b, (const cplx*)qhat + (long)p0 * n23, nloc * sizeof(cplx),
                              on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c.stream));
    fgmres(*H2, hier, b, nullptr, x, restart, maxiter, tol, r);
    // gather the owned rows of every rank
    full = on_device ? (cplx*)a_out : dalloc<cplx>(N);
    HADR_CUDA(cudaMemcpyAsync(full + (long)p0 * n23, x, nloc * sizeof(cplx), cudaMemcpyDeviceToDevice, c.stream));
    cm->group_start();
    for (int q = 0; q < R; ++q)
      cm->bcast(full + (long)plan.bounds[q] * n23, (size_t)(plan.bounds[q + 1] - plan.bounds[q]) * n23 * sizeof(cplx),
                q, c.stream);
    cm->group_end();
    if (!on_device) HADR_CUDA(cudaMemcpyAsync(a_out, full, N * sizeof(cplx), cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    if (on_device) full = nullptr;
  } catch (...) {
    if (on_device) full = nullptr;
    cleanup();
    throw;
  }
  cleanup();
}

extern "C" {

const char* hadr_last_error(void) { return g_err.c_str(); }

int hadr_init(int device) {
  return guarded([&] {
    int n = 0;
    HADR_CUDA(cudaGetDeviceCount(&n));
    if (n <= 0) throw std::runtime_error("no CUDA device");
    HADR_CUDA(cudaSetDevice(device));
    Ctx::get();
  });
}

int hadr_device_sync(void) { return guarded([&] { Ctx::get().sync(); }); }

int hadr_device_malloc(void** ptr, size_t bytes) {
  return guarded([&] { *ptr = pool_alloc(bytes); });  // caching allocator: repeated solves do not cudaMalloc
}
int hadr_device_free(void* ptr) {
  return guarded([&] { pool_free(ptr); });
}

int hadr_phase_transform(long long n, const double* q, const double* tau, double omega, int sign, double* out,
                         int on_device) {
  return guarded([&] {
    if (sign != 1 && sign != -1) throw ValueError("sign must be +1 (to_adr) or -1 (to_helmholtz)");
    Ctx& c = Ctx::get();
    DevVec dq(q, n, on_device, true), dout(out, n, on_device, false);
    const double* dt = tau;
    double* tmp = nullptr;
    if (!on_device) {
      tmp = dalloc<double>(n);
      HADR_CUDA(cudaMemcpyAsync(tmp, tau, n * sizeof(double), cudaMemcpyHostToDevice, c.stream));
      dt = tmp;
    }
    launch_phase(c.stream, n, dq.p, dt, omega, sign, dout.p);
    HADR_CUDA(cudaGetLastError());
    dout.copy_out(out);
    c.sync();
    dfree(tmp);
  });
}
int hadr_tau_derivatives(int dim, const int* n, const double* L, const int* src, const double* tau1, double* tau,
                         double* grads, double* lap, int on_device) {
  return guarded([&] {
    if (dim != 2 && dim != 3) throw ValueError("dim must be 2 or 3");
    long N = 1;
    double h[3];
    for (int a = 0; a < dim; ++a) {
      if (n[a] < 4) throw ValueError("tau_derivatives needs at least 4 nodes per axis (one-sided 4-point ends)");
      if (src[a] < 0 || src[a] >= n[a]) throw ValueError("source index outside the grid");
      h[a] = L[a] / (n[a] - 1);  // GridSpec.h = L / (n - 1)
      N *= n[a];
    }
    Ctx& c = Ctx::get();
    const size_t nb = N * sizeof(double);
    const double* t1 = tau1;
    double *tmp = nullptr, *dtau = tau, *dg = grads, *dl = lap;
    if (!on_device) {  // one staging block: tau1 | tau | grads | lap
      tmp = dalloc<double>((size_t)N * (dim + 3));
      HADR_CUDA(cudaMemcpyAsync(tmp, tau1, nb, cudaMemcpyHostToDevice, c.stream));
      t1 = tmp;
      dtau = tau ? tmp + N : nullptr;
      dg = tmp + 2 * N;
      dl = tmp + (2 + dim) * N;
    }
    double* gp[3] = {dg, dg + N, dim == 3 ? dg + 2 * N : nullptr};
    launch_tau_derivs(c.stream, dim, n, h, L, src, t1, dtau, gp, dl);
    HADR_CUDA(cudaGetLastError());
    if (!on_device) {
      if (tau) HADR_CUDA(cudaMemcpyAsync(tau, dtau, nb, cudaMemcpyDeviceToHost, c.stream));
      HADR_CUDA(cudaMemcpyAsync(grads, dg, nb * dim, cudaMemcpyDeviceToHost, c.stream));
      HADR_CUDA(cudaMemcpyAsync(lap, dl, nb, cudaMemcpyDeviceToHost, c.stream));
    }
    c.sync();
    dfree(tmp);
  });
}

int hadr_memcpy(void* dst, const void* src, size_t bytes, int kind) {
  return guarded([&] {
    Ctx& c = Ctx::get();
    cudaMemcpyKind k = kind == 1 ? cudaMemcpyHostToDevice : kind == 2 ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
    HADR_CUDA(cudaMemcpyAsync(dst, src, bytes, k, c.stream));
    c.sync();
  });
}

int hadr_memset(void* dst, int value, size_t bytes) {
  return guarded([&] {
    Ctx& c = Ctx::get();
    HADR_CUDA(cudaMemsetAsync(dst, value, bytes, c.stream));
    c.sync();
  });
}

int hadr_op_from_csr(int n1, int n2, int n3, int64_t nnz, const int64_t* indptr, const int32_t* indices,
                     const double* data, hadr_op* out) {
  return guarded([&] {
    if (n1 < 1 || n2 < 1 || n3 < 1) throw ValueError("grid dimensions must be positive");
    *out = wrap(op_from_csr(n1, n2, n3, nnz, indptr, indices, (const cplx*)data));
  });
}

int hadr_op_from_planes(int n1, int n2, int n3, int n_offsets, const int* offsets, const double* coef, hadr_op* out) {
  return guarded([&] { *out = wrap(op_from_planes(n1, n2, n3, n_offsets, offsets, (const cplx*)coef)); });
}

int hadr_op_info(hadr_op h, int* n1, int* n2, int* n3, int* n_offsets, int* offsets) {
  return guarded([&] {
    const Op* op = h->op;
    *n1 = op->n1;
    *n2 = op->n2;
    *n3 = op->n3;
    *n_offsets = op->nofs;
    for (int o = 0; o < op->nofs; ++o) {
      offsets[3 * o] = op->d1[o];
      offsets[3 * o + 1] = op->d2[o];
      offsets[3 * o + 2] = op->d3[o];
    }
  });
}

int hadr_op_export(hadr_op h, double* coef) {
  return guarded([&] {
    Ctx& c = Ctx::get();
    const Op* op = h->op;
    HADR_CUDA(cudaMemcpyAsync(coef, op->coef, (size_t)op->nofs * op->N * sizeof(cplx), cudaMemcpyDeviceToHost,
                              c.stream));
    c.sync();
  });
}

int hadr_op_apply(hadr_op h, const double* x, double* y, int on_device) {
  return guarded([&] {
    Op* op = h->op;
    if (g_pair_compress && !op->pc_tried) op->pair_compress();  // the fine-level kernel the solver runs
    if (!op->pcode && g_class_compress > (op->n3 > 1 ? 0 : 1) && !op->cc_tried && op->nofs > 13)
      op->class_compress();  // the coarse-level kernel of the hierarchy's graph path
    DevVec dx(x, op->N, on_device, true), dy(y, op->N, on_device, false);
    op_apply(*op, dx.p, dy.p);
    HADR_CUDA(cudaGetLastError());
    dy.copy_out(y);
    Ctx::get().sync();
  });
}

int hadr_op_storage(hadr_op h, int* n_slots, long long* overflow_rows) {
  return guarded([&] {
    *n_slots = h->op->pcode ? h->op->nslot : h->op->ccode ? h->op->nsl : 0;
    if (overflow_rows) *overflow_rows = h->op->ccode ? h->op->mixed_rows : 0;
  });
}

int hadr_op_jacobi(hadr_op h, const double* r, double* z, int on_device) {
  return guarded([&] {
    Op* op = h->op;
    const int ce = op->center();
    if (ce < 0) throw ValueError("jacobi_apply: operator has zero diagonal entries");
    op->inv_diag();  // raises on a zero diagonal (helmadr/krylov.py:71-72)
    DevVec dr(r, op->N, on_device, true), dz(z, op->N, on_device, false);
    launch_cdiv(Ctx::get().stream, op->N, dr.p, op->coef + (long)ce * op->N, dz.p);
    HADR_CUDA(cudaGetLastError());
    dz.copy_out(z);
    Ctx::get().sync();
  });
}

int hadr_op_axpby(double ar, double ai, hadr_op A, double br, double bi, hadr_op B, hadr_op* out) {
  return guarded([&] { *out = wrap(op_axpby(mk(ar, ai), *A->op, mk(br, bi), *B->op)); });
}

int hadr_op_add_diag(hadr_op A, double sr, double si, const double* field, hadr_op* out) {
  return guarded([&] { *out = wrap(op_add_diag_real(*A->op, mk(sr, si), field)); });
}

int hadr_op_similarity(hadr_op A, const double* left, const double* right, hadr_op* out) {
  return guarded([&] { *out = wrap(op_similarity(*A->op, (const cplx*)left, (const cplx*)right)); });
}

int hadr_op_galerkin(hadr_op A, hadr_op* out) {
  return guarded([&] { *out = wrap(op_galerkin(*A->op)); });
}

int hadr_assemble(int dim, int n1, int n2, int n3, double h1, double h2, double h3, double omega, int scheme,
                  const int* bc, int src1, int src2, int src3, const double* kappa_sq, const double* gamma,
                  const double* grad1, const double* grad2, const double* grad3, const double* lap_tau, int on_device,
                  hadr_op* out) {
  return guarded([&] {
    *out = wrap(op_assemble(dim, n1, n2, n3, h1, h2, h3, omega, scheme, bc, src1, src2, src3, kappa_sq, gamma, grad1,
                            grad2, grad3, lap_tau, on_device != 0));
  });
}

int hadr_solve_adr_upwind(int dim, int n1, int n2, int n3, double h1, double h2, double h3, double omega,
                          const int* bc, int src1, int src2, int src3, const double* kappa_sq, const double* gamma,
                          const double* grad1, const double* grad2, const double* grad3, const double* lap_tau,
                          const double* qhat, double beta, int levels, int restart, int maxiter, double tol,
                          double* a_out, hadr_report* rep, double* history, int history_cap, double* t_setup,
                          int on_device) {
  return guarded([&] {
    Ctx& c = Ctx::get();
    if (dim == 2) n3 = 1;
    const long N = (long)n1 * n2 * n3;
    if (dist_comm()) {
      Report r;
      solve_adr_upwind_dist(dim, n1, n2, n3, h1, h2, h3, omega, bc, src1, src2, src3, kappa_sq, gamma, grad1, grad2,
                            grad3, lap_tau, qhat, beta, levels, restart, maxiter, tol, a_out, r, t_setup, on_device);
      rep->iterations = r.iterations;
      rep->converged = r.converged;
      rep->note = r.note;
      rep->bnorm = r.bnorm;
      rep->final_relres = r.final_relres;
      rep->wall_time = r.wall_time;
      rep->device_time = r.device_time;
      rep->ortho_max = r.ortho_max;
      const int nh = (int)r.history.size();
      rep->history_len = nh;
      if (history)
        for (int i = 0; i < nh && i < history_cap; ++i) history[i] = r.history[i];
      return;
    }
    cudaEvent_t e0, e1;
    HADR_CUDA(cudaEventCreate(&e0));
    HADR_CUDA(cudaEventCreate(&e1));
    HADR_CUDA(cudaEventRecord(e0, c.stream));
    // helmadr/drivers.py:153-157: assemble H2up, H1up, blend, hierarchy
    Op* H2 = op_assemble(dim, n1, n2, n3, h1, h2, h3, omega, 2, bc, src1, src2, src3, kappa_sq, gamma, grad1, grad2,
                         grad3, lap_tau, on_device);
    Op* H1 = nullptr;
    Op* B = nullptr;
    Hier* hier = nullptr;
    try {
      H1 = op_assemble(dim, n1, n2, n3, h1, h2, h3, omega, 1, bc, src1, src2, src3, kappa_sq, gamma, grad1, grad2,
                       grad3, lap_tau, on_device);
      B = op_axpby(mk(1.0 - beta, 0.0), *H2, mk(beta, 0.0), *H1);
      delete H1;
      H1 = nullptr;
      hier = hier_build(B, levels, 10, 0.1);
      delete B;
      B = nullptr;
      HADR_CUDA(cudaEventRecord(e1, c.stream));
      HADR_CUDA(cudaEventSynchronize(e1));
      float ms = 0.f;
      HADR_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      if (t_setup) *t_setup = ms * 1e-3;
      DevVec dq(qhat, N, on_device, true), da(a_out, N, on_device, false);
      Report r;
      fgmres(*H2, hier, dq.p, nullptr, da.p, restart, maxiter, tol, r);
      da.copy_out(a_out);
      c.sync();
      rep->iterations = r.iterations;
      rep->converged = r.converged;
      rep->note = r.note;
      rep->bnorm = r.bnorm;
      rep->final_relres = r.final_relres;
      rep->wall_time = r.wall_time;
      rep->device_time = r.device_time;
      rep->ortho_max = r.ortho_max;
      const int nh = (int)r.history.size();
      rep->history_len = nh;
      if (history)
        for (int i = 0; i < nh && i < history_cap; ++i) history[i] = r.history[i];
    } catch (...) {
      delete H1;
      delete B;
      hier_release(hier);
      delete H2;
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
      throw;
    }
    hier_release(hier);
    delete H2;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  });
}

void hadr_op_destroy(hadr_op h) {
  if (!h) return;
  if (h->own) delete h->op;
  delete h;
}

int hadr_transfer(int n1, int n2, int n3, int direction, const double* in, double* out, int on_device) {
  return guarded([&] {
    if ((n1 - 1) % 2 || (n2 - 1) % 2 || (n3 > 1 && (n3 - 1) % 2))
      throw ValueError("cannot coarsen: interval count is odd");
    Ctx& c = Ctx::get();
    const long Nf = (long)n1 * n2 * n3;
    const long Nc = (long)((n1 - 1) / 2 + 1) * ((n2 - 1) / 2 + 1) * ((n3 - 1) / 2 + 1);
    if (direction == 0) {
      DevVec di(in, Nf, on_device, true), dout(out, Nc, on_device, false);
      launch_restrict(c.lc, n1, n2, n3, di.p, dout.p, gate_always());
      HADR_CUDA(cudaGetLastError());
      dout.copy_out(out);
    } else {
      DevVec di(in, Nc, on_device, true), dout(out, Nf, on_device, false);
      HADR_CUDA(cudaMemsetAsync(dout.p, 0, Nf * sizeof(cplx), c.stream));
      launch_prolong_add(c.lc, n1, n2, n3, di.p, dout.p, gate_always());
      HADR_CUDA(cudaGetLastError());
      dout.copy_out(out);
    }
    c.sync();
  });
}

static hadr_hier wrap_hier(Hier* h) {
  hadr_hier_s* s = new hadr_hier_s();
  s->h = h;
  for (auto& L : h->lv) s->level_handles.push_back(hadr_op_s{L.A, false});
  return s;
}

int hadr_hier_create(hadr_op fine, int max_levels, int coarse_steps, double coarse_tol, hadr_hier* out) {
  return guarded([&] { *out = wrap_hier(hier_build(fine->op, max_levels, coarse_steps, coarse_tol)); });
}

int hadr_hier_from_ops(int n_levels, const hadr_op* ops, int coarse_steps, double coarse_tol, hadr_hier* out) {
  return guarded([&] {
    std::vector<Op*> v;
    for (int i = 0; i < n_levels; ++i) v.push_back(ops[i]->op);
    *out = wrap_hier(hier_from_ops(n_levels, v.data(), coarse_steps, coarse_tol));
  });
}

int hadr_hier_info(hadr_hier h, int* n_levels, int* shapes) {
  return guarded([&] {
    *n_levels = (int)h->h->lv.size();
    if (shapes)
      for (size_t i = 0; i < h->h->lv.size(); ++i) {
        shapes[3 * i] = h->h->lv[i].n1;
        shapes[3 * i + 1] = h->h->lv[i].n2;
        shapes[3 * i + 2] = h->h->lv[i].n3;
      }
  });
}

int hadr_hier_level_op(hadr_hier h, int level, hadr_op* out) {
  return guarded([&] {
    if (level < 1 || level > (int)h->level_handles.size()) throw ValueError("level out of range");
    *out = &h->level_handles[level - 1];
  });
}

int hadr_kcycle(hadr_hier hh, int level, const double* b, const double* x, double* x_out, int* visits,
                int on_device) {
  return guarded([&] {
    Hier* h = hh->h;
    const int nl = (int)h->lv.size();
    if (level < 1 || level > nl) throw ValueError("level outside 1.." + std::to_string(nl));
    if (level == nl) throw ValueError("k_cycle at the coarsest level has no coarse grid");
    const long n = h->lv[level - 1].N;
    DevVec db(b, n, on_device, true), dxo(x_out, n, on_device, false);
    DevVec dx(x, n, on_device, true);
    h->kcycle_direct(level - 1, db.p, x ? dx.p : nullptr, dxo.p, visits);
    dxo.copy_out(x_out);
    Ctx::get().sync();
  });
}

int hadr_precond_apply(hadr_hier hh, const double* r, double* z, int on_device) {
  return guarded([&] {
    Hier* h = hh->h;
    const long n = h->lv[0].N;
    DevVec dr(r, n, on_device, true), dz(z, n, on_device, false);
    h->apply(dr.p, dz.p);
    HADR_CUDA(cudaGetLastError());
    dz.copy_out(z);
    Ctx::get().sync();
    if (!on_device) {  // staged buffers die with this call: drop their graph
      auto it = h->graphs.find(std::make_pair((const void*)dr.p, (void*)dz.p));
      if (it != h->graphs.end()) {
        cudaGraphExecDestroy(it->second);
        h->graphs.erase(it);
      }
    }
  });
}

long long hadr_launch_count(void) { return g_launch_count; }

int hadr_ce_bench(hadr_hier hh, int level, int reps, double* avg_ms) {
  return guarded([&] {
    Ctx& c = Ctx::get();
    Hier* h = hh->h;
    const int li = level - 1;
    const int nl = (int)h->lv.size();
    if (li < 1 || li >= nl - 1) throw ValueError("the engine's inner-FGMRES entry needs 2 <= level < n_levels");
    if (!h->use_ce(li)) throw ValueError("this level does not run in the cluster engine");
    auto once = [&]() { launch_cluster_engine(c.stream, h->ce_desc, 1, li, nullptr, nullptr, nullptr, CE_CTAS,
                                              h->ce_tile(li)); };
    for (int i = 0; i < 3; ++i) once();
    cudaEvent_t e0, e1;
    HADR_CUDA(cudaEventCreate(&e0));
    HADR_CUDA(cudaEventCreate(&e1));
    HADR_CUDA(cudaEventRecord(e0, c.stream));
    for (int i = 0; i < reps; ++i) once();
    HADR_CUDA(cudaEventRecord(e1, c.stream));
    HADR_CUDA(cudaEventSynchronize(e1));
    HADR_CUDA(cudaGetLastError());
    float ms = 0.f;
    HADR_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    *avg_ms = ms / reps;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  });
}

int hadr_op_bench(hadr_op h, const double* x, double* y, int reps, int variant, double* avg_ms) {
  return guarded([&] {
    Ctx& c = Ctx::get();
    Op* op = h->op;
    if (g_pair_compress && !op->pc_tried) op->pair_compress();  // as the hierarchy's fine level
    if (!op->pcode && g_class_compress > (op->n3 > 1 ? 0 : 1) && !op->cc_tried && op->nofs > 13)
      op->class_compress();  // as the hierarchy's coarse graph-path levels
    const cplx* xd = (const cplx*)x;
    cplx* yd = (cplx*)y;
    cplx* vtmp = dalloc<cplx>(op->N);
    cplx* utmp = dalloc<cplx>(op->N);  // dot partner V0: its own stream, as in the relaxation
    cplx* ztmp = variant == 3 ? dalloc<cplx>(op->N) : nullptr;
    HADR_CUDA(cudaMemsetAsync(utmp, 0, op->N * sizeof(cplx), c.stream));
    double* sc = c.dscal + 56;
    const double one = 1.0;
    HADR_CUDA(cudaMemcpyAsync(sc, &one, sizeof(double), cudaMemcpyHostToDevice, c.stream));
    auto once = [&]() {
      StencilArgs a{};
      a.A = op->dev();
      a.x = xd;
      a.y = yd;
      a.gate = gate_always();
      a.rs = c.rs;
      if (variant == 0) {  // y = A x
        a.epi = epi_none();
        launch_stencil(c.lc, IN_PLAIN, OUT_APPLY, RED_NONE, a);
      } else if (variant == 2) {  // y = A x, <u, y> (the split relaxation's stencil)
        a.u = utmp;
        a.epi = epi_store(c.dscal);
        launch_stencil(c.lc, IN_PLAIN, OUT_APPLY, RED_DOT, a);
      } else if (variant == 3) {  // split relaxation step: V = s x, z = D^-1 V, then y = A z, <u, y>
        launch_scale_jac(c.lc, op->N, xd, sc, op->inv_diag(), vtmp, ztmp, gate_always());
        a.x = ztmp;
        a.u = utmp;
        a.epi = epi_store(c.dscal);
        launch_stencil(c.lc, IN_PLAIN, OUT_APPLY, RED_DOT, a);
      } else {             // relaxation Arnoldi input: y = A (D^-1 (s x)), V = s x, <V0, y>
        a.scale = sc;
        a.dinv = op->inv_diag();
        a.vout = vtmp;
        a.u = utmp;
        a.epi = epi_store(c.dscal);
        launch_stencil(c.lc, IN_SCALE | IN_JAC | IN_WRITEV, OUT_APPLY, RED_DOT, a);
      }
    };
    for (int i = 0; i < 3; ++i) once();
    cudaEvent_t e0, e1;
    HADR_CUDA(cudaEventCreate(&e0));
    HADR_CUDA(cudaEventCreate(&e1));
    HADR_CUDA(cudaEventRecord(e0, c.stream));
    for (int i = 0; i < reps; ++i) once();
    HADR_CUDA(cudaEventRecord(e1, c.stream));
    HADR_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    HADR_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    *avg_ms = ms / reps;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    dfree(vtmp);
    dfree(utmp);
    if (ztmp) dfree(ztmp);
  });
}

int hadr_ce_profile(unsigned long long* out48, int reset) {
  return guarded([&] {
    Ctx::get().sync();
    if (ce_profile_read(out48, reset)) throw std::runtime_error("ce_profile_read failed");
  });
}

int hadr_set_option(const char* name, double value) {
  return guarded([&] {
    std::string n(name ? name : "");
    if (n == "ce_profile") {
      g_ce_prof_on = value != 0.0;
    } else if (n == "ce_smem_coef") {
      g_ce_smem_coef = value != 0.0;
      for (;;) {
        Hier* h = hier_pool_pop();
        if (!h) break;
        delete h;
      }
    } else if (n == "mid_ppt" || n == "mid_max_n" || n == "mid_min_n") {
      if (n == "mid_ppt") g_mid_ppt = (int)value;
      if (n == "mid_min_n") g_mid_min_n = (long)value;
      if (n == "mid_max_n") g_mid_max_n = (long)value;
      for (;;) {
        Hier* h = hier_pool_pop();
        if (!h) break;
        delete h;
      }
    } else if (n == "defer_mgs") {
      g_defer_mgs = value != 0.0;
      for (;;) {
        Hier* h = hier_pool_pop();
        if (!h) break;
        delete h;
      }
    } else if (n == "ce_cgs2") {
      g_ce_cgs2 = value != 0.0;
      for (;;) {  // captured graphs carry the engine's launch flags
        Hier* h = hier_pool_pop();
        if (!h) break;
        delete h;
      }
    } else if (n == "kcycle_c64") {
      g_kcycle_c64 = value != 0.0;
    } else if (n == "ce_smem_relax") {
      g_ce_smem_relax = value != 0.0;
      for (;;) {
        Hier* h = hier_pool_pop();
        if (!h) break;
        delete h;
      }
    } else if (n == "cl_max_n") {
      g_cl_max_n = (long)value;
      for (;;) {
        Hier* h = hier_pool_pop();
        if (!h) break;
        delete h;
      }
    } else if (n == "stencil_tile") {
      g_stencil_tile = (int)value;
      for (;;) {
        Hier* h = hier_pool_pop();
        if (!h) break;
        delete h;
      }
    } else if (n == "small_max_work") {
      g_small_max_work = (long)value;
      for (;;) {
        Hier* h = hier_pool_pop();
        if (!h) break;
        delete h;
      }
    } else if (n == "stencil_march" || n == "march_min_n" || n == "march_min_n2d") {
      if (n == "stencil_march")
        g_stencil_march = (int)value;
      else if (n == "march_min_n")
        g_march_min_n = (long)value;
      else
        g_march_min_n2d = (long)value;
      for (;;) {
        Hier* h = hier_pool_pop();
        if (!h) break;
        delete h;
      }
    } else if (n == "relax_split") {
      g_relax_split = (long)value;
      for (;;) {
        Hier* h = hier_pool_pop();
        if (!h) break;
        delete h;
      }
    } else if (n == "class_compress") {
      g_class_compress = (int)value;
      for (;;) {
        Hier* h = hier_pool_pop();
        if (!h) break;
        delete h;
      }
    } else if (n == "pair_compress") {
      g_pair_compress = value != 0.0;
      for (;;) {
        Hier* h = hier_pool_pop();
        if (!h) break;
        delete h;
      }
    } else if (n == "pdl") {
      g_pdl = value != 0.0;
      for (;;) {  // captured graphs carry the old launch attributes
        Hier* h = hier_pool_pop();
        if (!h) break;
        delete h;
      }
    } else if (n == "dist_min_planes") {
      g_dist_min_planes = (int)value;
    } else if (n == "dist_min_work") {
      g_dist_min_work = value;
    } else if (n == "dist_levels") {
      g_dist_levels = (int)value;
    } else if (n == "ce_max_n") {
      g_ce_max_n = (long)value;
      // recycled hierarchies hold graphs captured under the old setting
      for (;;) {
        Hier* h = hier_pool_pop();
        if (!h) break;
        delete h;
      }
    } else {
      throw ValueError("unknown option " + n);
    }
  });
}

int hadr_dist_nccl_id(char* out) {
  return guarded([&] { dist_nccl_unique_id(out); });
}

int hadr_dist_init_nccl(int rank, int size, const char* unique_id) {
  return guarded([&] { dist_init_nccl(rank, size, unique_id); });
}

int hadr_dist_init_host(int rank, int size, hadr_host_allgather ag, hadr_host_sendrecv sr, hadr_host_bcast bc) {
  return guarded([&] { dist_init_host(rank, size, ag, sr, bc); });
}

int hadr_dist_finalize(void) {
  return guarded([&] { dist_finalize(); });
}

int hadr_dist_info(int* rank, int* size, int* kind) {
  Comm* cm = dist_comm();
  if (rank) *rank = cm ? cm->rank : 0;
  if (size) *size = cm ? cm->size : 1;
  if (kind) *kind = cm ? cm->kind : 0;
  return 0;
}

int hadr_dist_plan(int n1, int n2, int n3, int max_levels, int* bounds, int* n_dist_levels, int* n_levels) {
  return guarded([&] {
    const SlabPlan p = slab_plan(n1, n2, n3, max_levels);
    for (size_t i = 0; i < p.bounds.size(); ++i) bounds[i] = p.bounds[i];
    *n_dist_levels = p.ndist;
    *n_levels = p.nlev;
  });
}

int hadr_slab_plan(int n1, int n2, int n3, int max_levels, int size, int* bounds, int* n_dist_levels, int* n_levels) {
  return guarded([&] {
    const SlabPlan p = slab_plan_for(n1, n2, n3, max_levels, size);
    for (size_t i = 0; i < p.bounds.size(); ++i) bounds[i] = p.bounds[i];
    *n_dist_levels = p.ndist;
    *n_levels = p.nlev;
  });
}

int hadr_march_plan(int n1own, int n2, int n3, int jac, int* out10) {
  return guarded([&] {
    if (!march_plan(n1own, n2, n3, jac, out10)) throw ValueError("the marching kernel declines this shape");
  });
}

int hadr_slab_bounds(int n1, int size, int align, int* bounds) {
  return guarded([&] {
    const std::vector<int> b = slab_bounds(n1, size, align);
    if (b.empty()) throw ValueError("cannot split the axis into slabs");
    for (size_t i = 0; i < b.size(); ++i) bounds[i] = b[i];
  });
}

int hadr_fast_march(int dim, const int* n, const double* h, const double* tau0, const double* g01,
                    const double* g02, const double* g03, const double* kappa, const int* src, int order,
                    double* tau1, long long* n_accepted) {
  return guarded([&] {
    const double* g0[3] = {g01, g02, g03};
    try {
      *n_accepted = (long long)hadr::fast_march(dim, n, h, tau0, g0, kappa, src, order, tau1);
    } catch (const std::invalid_argument& e) {
      throw ValueError(e.what());
    }
  });
}

int hadr_relative_error(long long n, const double* u, const double* u_ref, double floor, double* err,
                        double* floor_used, long long* count, const long long* idx, int nidx, double* vals,
                        int on_device) {
  return guarded([&] {
    if (n <= 0) throw ValueError("relative_error: empty field");
    if (nidx < 0 || (nidx > 0 && (!idx || !vals))) throw ValueError("relative_error: bad order-statistic request");
    Ctx& c = Ctx::get();
    DevVec du(u, n, on_device, true), dr(u_ref, n, on_device, true);
    double* derr = nullptr;
    if (err) derr = on_device ? err : dalloc<double>(n);
    accuracy_stats(n, du.p, dr.p, floor, derr, floor_used, count, idx, nidx, vals);
    if (err && !on_device) {
      HADR_CUDA(cudaMemcpyAsync(err, derr, n * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
      c.sync();
      dfree(derr);
    }
  });
}

double hadr_stream_timer(int start) {
  static cudaEvent_t ev[2] = {nullptr, nullptr};
  try {
    Ctx& c = Ctx::get();
    if (!ev[0]) {
      HADR_CUDA(cudaEventCreate(&ev[0]));
      HADR_CUDA(cudaEventCreate(&ev[1]));
    }
    if (start) {
      HADR_CUDA(cudaEventRecord(ev[0], c.stream));
      return 0.0;
    }
    HADR_CUDA(cudaEventRecord(ev[1], c.stream));
    HADR_CUDA(cudaEventSynchronize(ev[1]));
    float ms = 0.f;
    HADR_CUDA(cudaEventElapsedTime(&ms, ev[0], ev[1]));
    return ms;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1.0;
  }
}

void hadr_hier_destroy(hadr_hier h) {
  if (!h) return;
  hier_release(h->h);
  delete h;
}

int hadr_pool_trim(void) {
  return guarded([&] {
    for (;;) {  // drop recycled hierarchies, then cached blocks
      Hier* h = hier_pool_pop();
      if (!h) break;
      delete h;
    }
    pool_trim();
  });
}

int hadr_gmres_relax(hadr_op A, const double* b, const double* x, int steps, double* x_out, int on_device) {
  return guarded([&] {
    Op* op = A->op;
    DevVec db(b, op->N, on_device, true), dx(x, op->N, on_device, true), dxo(x_out, op->N, on_device, false);
    gmres_relax(*op, db.p, dx.p, dxo.p, steps);
    dxo.copy_out(x_out);
    Ctx::get().sync();
  });
}

int hadr_fgmres(hadr_op A, hadr_hier M, const double* b, const double* x0, int restart, int maxiter, double tol,
                double* x_out, hadr_report* rep, double* history, int history_cap, int on_device) {
  return hadr_fgmres_ex(A, M, b, x0, restart, maxiter, tol, 0, x_out, rep, history, history_cap, on_device);
}

int hadr_fgmres_ex(hadr_op A, hadr_hier M, const double* b, const double* x0, int restart, int maxiter, double tol,
                   int flags, double* x_out, hadr_report* rep, double* history, int history_cap, int on_device) {
  return guarded([&] {
    Op* op = A->op;
    DevVec db(b, op->N, on_device, true), dx0(x0, op->N, on_device, true), dx(x_out, op->N, on_device, false);
    Report r;
    fgmres(*op, M ? M->h : nullptr, db.p, x0 ? dx0.p : nullptr, dx.p, restart, maxiter, tol, r, flags);
    dx.copy_out(x_out);
    Ctx::get().sync();
    rep->iterations = r.iterations;
    rep->converged = r.converged;
    rep->note = r.note;
    rep->bnorm = r.bnorm;
    rep->final_relres = r.final_relres;
    rep->wall_time = r.wall_time;
    rep->device_time = r.device_time;
    rep->ortho_max = r.ortho_max;
    const int nh = (int)r.history.size();
    rep->history_len = nh;
    if (history)
      for (int i = 0; i < nh && i < history_cap; ++i) history[i] = r.history[i];
  });
}

}  // extern "C"
