// Host engine of the amplitude solve.  Mirrors helmadr/multigrid.py and
// helmadr/krylov.py control flow; the device does every vector operation and
// every data-dependent branch of the preconditioner, the host only drives the
// outer FGMRES (one small read-back per outer iteration).
#include "engine.h"
#include "dist.h"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>

namespace hadr {

long g_ce_max_n = 32768;
// The engine's 16 SMs (and the single-cluster vector kernels) pay per coefficient streamed: the 2D
// limit of 32768 points x 21 offsets is 688k coefficients per stencil.  3D upwind levels carry up to
// 81 offsets per row — the 33^2 x 17 level streams 1.5 M coefficients (24 MB) per stencil — and run
// faster on plain grids over all SMs (B200: config-5 recipe 551.6 -> 484.5 ms per solve, config 4
// 2032 -> 2003 ms), while the 27-offset shifted-Laplacian level of the same size (0.5 M) is faster
// in the engine (standard_sl 1251 vs 1125 Mdof*it/s).  A level is engine / cluster sized when
// N <= ce_max_n (cl_max_n) and N x offsets <= small_max_work.
long g_small_max_work = 32768L * 21;  // option "small_max_work" 
int g_kcycle_c64 = 0;

// ---------------------------------------------------------------------------
// caching allocator
// ---------------------------------------------------------------------------
static std::map<void*, size_t>& live_blocks() {
  static std::map<void*, size_t> m;
  return m;
}
static std::multimap<size_t, void*>& free_blocks() {
  static std::multimap<size_t, void*> m;
  return m;
}

void* pool_alloc(size_t bytes) {
  bytes = (bytes + 511) & ~size_t(511);
  auto& fb = free_blocks();
  auto it = fb.find(bytes);
  void* p = nullptr;
  if (it != fb.end()) {
    p = it->second;
    fb.erase(it);
  } else {
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e != cudaSuccess) {  // out of memory: drop the cache and retry once
      cudaGetLastError();
      pool_trim();
      HADR_CUDA(cudaMalloc(&p, bytes));
    }
  }
  live_blocks()[p] = bytes;
  return p;
}

void pool_free(void* p) {
  auto& lb = live_blocks();
  auto it = lb.find(p);
  if (it == lb.end()) {  // interior pointer (slab vectors point past their lower halo)
    it = lb.upper_bound(p);
    if (it == lb.begin()) return;
    --it;
    if ((char*)p >= (char*)it->first + it->second) return;
  }
  free_blocks().emplace(it->second, it->first);
  lb.erase(it);
}

size_t pool_trim() {
  size_t n = 0;
  for (auto& kv : free_blocks()) {
    cudaFree(kv.second);
    n += kv.first;
  }
  free_blocks().clear();
  return n;
}

// ---------------------------------------------------------------------------
// context
// ---------------------------------------------------------------------------
Ctx& Ctx::get() {
  static Ctx* c = nullptr;
  if (!c) {
    Ctx* n = new Ctx();
    HADR_CUDA(cudaGetDevice(&n->device));
    HADR_CUDA(cudaDeviceGetAttribute(&n->nsm, cudaDevAttrMultiProcessorCount, n->device));
    HADR_CUDA(cudaStreamCreateWithFlags(&n->stream, cudaStreamNonBlocking));
    n->rs.partials = dalloc<double>(4 * 8192);
    n->rs2.partials = dalloc<double>(4 * 8192);
    n->rs2.ticket = nullptr;
    n->rs.ticket = dalloc<unsigned>(4);
    HADR_CUDA(cudaMemset(n->rs.ticket, 0, 4 * sizeof(unsigned)));
    n->dscal = dalloc<double>(64);
    HADR_CUDA(cudaMallocHost(&n->hscal, 64 * sizeof(double)));
    n->lc.stream = n->stream;
    n->lc.max_blocks = n->nsm * 8;  // 8 resident 256-thread CTAs per SM
    c = n;
  }
  return *c;
}

// ---------------------------------------------------------------------------
// operators
// ---------------------------------------------------------------------------
Op::~Op() {
  dfree(coef);
  dfree(coef32);
  dfree(dinv);
  dfree(pcode);
  dfree(pcoef);
  dfree(pcoef32);
  dfree(ccode);
  dfree(ccoef);
  dfree(ccoef32);
  dfree(ctab);
  dfree(cnsl);
}

void Op::make_c64() {
  if (!coef32) coef32 = dalloc<float2>((size_t)alloc_len()) + base_off();
  launch_to_c64(Ctx::get().stream, alloc_len(), coef - base_off(), coef32 - base_off());
  if (pcode) {
    if (!pcoef32) pcoef32 = dalloc<float2>((size_t)nslot * nloc());
    launch_to_c64(Ctx::get().stream, (long)nslot * nloc(), pcoef, pcoef32);
  }
  if (ccode) {
    if (!ccoef32) ccoef32 = dalloc<float2>((size_t)nsl * nloc());
    launch_to_c64(Ctx::get().stream, (long)nsl * nloc(), ccoef, ccoef32);
  }
}

int g_class_compress = 2;
long g_relax_split = 8192;  // (1 << 20 until session 5: the 139k- and 18.5k-point 3D levels gain too: config-5 recipe -2.7%)

bool Op::class_compress() {
  cc_tried = true;
  auto drop = [&] {
    dfree(ccode);
    dfree(ccoef);
    dfree(ccoef32);
    dfree(ctab);
    dfree(cnsl);
    ccode = nullptr;
    ccoef = nullptr;
    ccoef32 = nullptr;
    ctab = nullptr;
    cnsl = nullptr;
    nsl = 0;
    return false;
  };
  const int dim = n3 > 1 ? 3 : 2;
  for (int o = 0; o < nofs; ++o) {
    const int a[3] = {d1[o], d2[o], d3[o]};
    int far = 0;
    for (int ax = 0; ax < 3; ++ax) {
      if (a[ax] < -2 || a[ax] > 2) return drop();
      far += (a[ax] == 2 || a[ax] == -2);
    }
    if (far > 1) return drop();
  }
  // classes: per axis '-' (only the -2 side), '+' or both; ordered by size so the
  // classifier's first fit is the smallest class that covers the row
  int ncls = 1;
  for (int ax = 0; ax < dim; ++ax) ncls *= 3;
  struct Cls {
    std::vector<int> offs;
    int mixed;
  };
  std::vector<Cls> cl;
  for (int c = 0; c < ncls; ++c) {
    int st[3] = {0, 0, 0}, cc = c, mixed = 0;
    for (int ax = 0; ax < dim; ++ax) {
      st[ax] = cc % 3;
      cc /= 3;
      mixed |= st[ax] == 2;
    }
    Cls k{{}, mixed};
    for (int o = 0; o < nofs; ++o) {
      const int a[3] = {d1[o], d2[o], d3[o]};
      bool in = true;
      for (int ax = 0; ax < dim; ++ax)
        if (a[ax] == 2 || a[ax] == -2) in = in && (st[ax] == 2 || (a[ax] > 0) == (st[ax] == 1));
      if (in) k.offs.push_back(o);
    }
    cl.push_back(k);
  }
  std::stable_sort(cl.begin(), cl.end(), [](const Cls& x, const Cls& y) { return x.offs.size() < y.offs.size(); });
  std::vector<unsigned long long> live(2 * ncls, 0ull);
  std::vector<int> hn(ncls), hm(ncls);
  for (int c = 0; c < ncls; ++c) {
    for (int o : cl[c].offs) live[2 * c + (o >> 6)] |= 1ull << (o & 63);
    hn[c] = (int)cl[c].offs.size();
    hm[c] = cl[c].mixed;
  }
  if (hn[0] * 5 > nofs * 4) return drop();  // even the smallest class saves < 20% of the planes
  Ctx& cx = Ctx::get();
  const long n = nloc();
  const bool refresh = ccode != nullptr;
  if (!ccode) ccode = dalloc<uint16_t>(n);
  if (!cnsl) cnsl = dalloc<int>(ncls);
  unsigned long long* dlive = dalloc<unsigned long long>(2 * ncls);
  int* dmix = dalloc<int>(ncls);
  HADR_CUDA(cudaMemcpyAsync(dlive, live.data(), live.size() * 8, cudaMemcpyHostToDevice, cx.stream));
  HADR_CUDA(cudaMemcpyAsync(cnsl, hn.data(), ncls * sizeof(int), cudaMemcpyHostToDevice, cx.stream));
  HADR_CUDA(cudaMemcpyAsync(dmix, hm.data(), ncls * sizeof(int), cudaMemcpyHostToDevice, cx.stream));
  unsigned long long* st = (unsigned long long*)(cx.dscal + 48);
  HADR_CUDA(cudaMemsetAsync(st, 0, 3 * sizeof(unsigned long long), cx.stream));
  StencilDev A = dev();
  launch_class_classify(cx.stream, A, ncls, dlive, cnsl, dmix, ccode, st);
  HADR_CUDA(cudaGetLastError());
  unsigned long long hs[3] = {0, 0, 0};
  HADR_CUDA(cudaMemcpyAsync(hs, st, sizeof(hs), cudaMemcpyDeviceToHost, cx.stream));
  cx.sync();
  dfree(dlive);
  dfree(dmix);
  mixed_rows = (long)hs[2];
  const int used = (int)hs[1];
  // worth it only if the rows read clearly fewer planes than the union on average
  unsigned long long bad = (hs[0] * 100 > (unsigned long long)n * nofs * 85) ? 1ull : 0ull;
  if (refresh && used != nsl) bad = 1;  // the captured graphs hold the old layout
  if (slab()) dist_comm()->allreduce_or_u64(&bad, 1, cx.stream);  // every rank takes the same path
  if (bad) return drop();
  if (!ccoef) ccoef = dalloc<cplx>((size_t)used * n);
  if (!ctab) ctab = dalloc<int4>((size_t)ncls * used);
  nsl = used;
  std::vector<int> otab((size_t)ncls * used, 0);
  std::vector<int4> ht((size_t)ncls * used, make_int4(0, 0, 0, 0));
  for (int c = 0; c < ncls; ++c)
    for (int q = 0; q < std::min(hn[c], used); ++q) {
      const int o = cl[c].offs[q];
      otab[(size_t)c * used + q] = o;
      ht[(size_t)c * used + q] = make_int4((int)(((long)d1[o] * n2 + d2[o]) * n3 + d3[o]), d1[o], d2[o], d3[o]);
    }
  int* dot = dalloc<int>(otab.size());
  HADR_CUDA(cudaMemcpyAsync(dot, otab.data(), otab.size() * sizeof(int), cudaMemcpyHostToDevice, cx.stream));
  HADR_CUDA(cudaMemcpyAsync(ctab, ht.data(), ht.size() * sizeof(int4), cudaMemcpyHostToDevice, cx.stream));
  launch_class_fill(cx.stream, A, ccode, cnsl, dot, used, ccoef, n);
  HADR_CUDA(cudaGetLastError());
  cx.sync();
  dfree(dot);
  if (coef32) {
    if (!ccoef32) ccoef32 = dalloc<float2>((size_t)nsl * n);
    launch_to_c64(cx.stream, (long)nsl * n, ccoef, ccoef32);
  }
  return true;
}

int g_pair_compress = 1;

bool Op::pair_compress() {
  pc_tried = true;
  auto drop = [&] {
    dfree(pcode);
    dfree(pcoef);
    dfree(pcoef32);
    pcode = nullptr;
    pcoef = nullptr;
    pcoef32 = nullptr;
    nslot = 0;
    return false;
  };
  // exactly the plus-radius-2 union in sorted order: centre, +-1 and +-2 along each axis
  const int dim = n3 > 1 ? 3 : 2;
  if (nofs != (dim == 2 ? 9 : 13)) return drop();
  {
    int k = 0;
    bool ok = true;
    for (int a1 = -2; a1 <= 2; ++a1)
      for (int a2 = -2; a2 <= 2; ++a2)
        for (int a3 = (dim == 3 ? -2 : 0); a3 <= (dim == 3 ? 2 : 0); ++a3) {
          if ((a1 != 0) + (a2 != 0) + (a3 != 0) > 1) continue;
          ok = ok && k < nofs && d1[k] == a1 && d2[k] == a2 && d3[k] == a3;
          ++k;
        }
    if (!ok || k != nofs) return drop();
  }
  int pos_a[HADR_MAX_OFS], pos_b[HADR_MAX_OFS], bit[HADR_MAX_OFS];
  const int ns = pair_layout(nofs, pos_a, pos_b, bit);
  if (ns == 0) return drop();
  const long n = nloc();
  if (pcode && nslot != ns) drop();
  if (!pcode) {
    pcode = dalloc<uint8_t>(n);
    pcoef = dalloc<cplx>((size_t)ns * n);
  }
  nslot = ns;
  Ctx& c = Ctx::get();
  int* flag = (int*)c.dscal + 33;
  HADR_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), c.stream));
  StencilDev A = dev();
  launch_pair_compress(c.stream, A, ns, pos_a, pos_b, bit, pcoef, n, pcode, flag);
  HADR_CUDA(cudaGetLastError());
  int conflict = 0;
  HADR_CUDA(cudaMemcpyAsync(&conflict, flag, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  c.sync();
  if (slab()) {  // every rank must take the same kernel path (identical graphs, no divergence)
    unsigned long long f = (unsigned long long)conflict;
    dist_comm()->allreduce_or_u64(&f, 1, c.stream);
    conflict = f != 0;
  }
  if (conflict) return drop();
  if (coef32) {  // mixed precision: complex64 copy of the compressed planes as well
    if (!pcoef32) pcoef32 = dalloc<float2>((size_t)nslot * n);
    launch_to_c64(c.stream, (long)nslot * n, pcoef, pcoef32);
  }
  return true;
}

StencilDev Op::dev() const {
  StencilDev s{};
  s.n1 = n1;
  s.n2 = n2;
  s.n3 = n3;
  s.nofs = nofs;
  s.p0 = p0;
  s.n1own = own();
  s.pstride = stride();
  for (int o = 0; o < nofs; ++o) {
    s.d1[o] = d1[o];
    s.d2[o] = d2[o];
    s.d3[o] = d3[o];
  }
  s.halo = 0;
  for (int o = 0; o < nofs; ++o)
    s.halo = std::max(s.halo, std::abs((d1[o] * n2 + d2[o]) * n3 + d3[o]));
  s.std2d = 0;
  if (n3 == 1 && (nofs == 21 || nofs == 9 || nofs == 5)) {
    bool same = true;
    for (int o = 0; o < nofs; ++o) {
      const int a = nofs == 21 ? Std2D::d1<21>(o) : nofs == 9 ? Std2D::d1<9>(o) : Std2D::d1<5>(o);
      const int b = nofs == 21 ? Std2D::d2<21>(o) : nofs == 9 ? Std2D::d2<9>(o) : Std2D::d2<5>(o);
      same = same && d1[o] == a && d2[o] == b && d3[o] == 0;
    }
    if (same) s.std2d = nofs;
  }
  s.coef = coef;
  s.coef32 = coef32;
  s.pcode = pcode;
  s.pcoef = pcoef;
  s.pcoef32 = pcoef32;
  s.pstr = nloc();
  s.ccode = ccode;
  s.ccoef = ccoef;
  s.ccoef32 = ccoef32;
  s.ctab = ctab;
  s.cnsl = cnsl;
  s.cstr = nloc();
  s.nsl = nsl;
  return s;
}

int Op::center() const {
  for (int o = 0; o < nofs; ++o)
    if (d1[o] == 0 && d2[o] == 0 && d3[o] == 0) return o;
  return -1;
}

// dinv over the owned points; slab operators keep kHalo halo planes (filled by exchange)
static void compute_inv_diag(const Op& A, cplx* dinv) {
  Ctx& c = Ctx::get();
  const int ce = A.center();
  int* flag = (int*)c.dscal + 32;
  HADR_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), c.stream));
  launch_inv_diag(c.stream, A.nloc(), ce >= 0 ? A.coef + (long)ce * A.stride() : nullptr, dinv, flag);
  unsigned long long hflag = 0;
  HADR_CUDA(cudaMemcpyAsync(&hflag, flag, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  c.sync();
  if (A.slab()) {
    Comm* cm = dist_comm();
    cm->halo(dinv, A.n23() * sizeof(cplx), A.own(), kHalo, c.stream);
    cm->allreduce_or_u64(&hflag, 1, c.stream);
  }
  if (hflag || ce < 0) throw ValueError("hierarchy operator has zero diagonal entries");
}

const cplx* Op::inv_diag() {
  if (dinv) return dinv;
  const long h = slab() ? (long)kHalo * n23() : 0;
  cplx* d = dalloc<cplx>(nloc() + 2 * h) + h;
  try {
    compute_inv_diag(*this, d);
  } catch (...) {
    dfree(d);
    throw;
  }
  dinv = d;
  return dinv;
}

void Op::refresh_inv_diag() {
  if (!dinv) {
    inv_diag();
    return;
  }
  compute_inv_diag(*this, dinv);
}

static void copy_geometry(Op* op, const Op& A) {
  op->n1 = A.n1;
  op->n2 = A.n2;
  op->n3 = A.n3;
  op->N = A.N;
  op->p0 = A.p0;
  op->nown = A.nown;
  op->hal = A.hal;
  op->pstride = A.pstride;
}
static void alloc_coef(Op* op) {  // after geometry + nofs
  op->coef = dalloc<cplx>((size_t)op->alloc_len()) + op->base_off();
}

Op* op_copy(const Op& A) {
  Ctx& c = Ctx::get();
  Op* op = new Op();
  copy_geometry(op, A);
  op->nofs = A.nofs;
  for (int o = 0; o < A.nofs; ++o) {
    op->d1[o] = A.d1[o];
    op->d2[o] = A.d2[o];
    op->d3[o] = A.d3[o];
  }
  alloc_coef(op);
  HADR_CUDA(cudaMemcpyAsync(op->coef - op->base_off(), A.coef - A.base_off(), (size_t)A.alloc_len() * sizeof(cplx),
                            cudaMemcpyDeviceToDevice, c.stream));
  return op;
}

static inline bool mask_has(const Mask125& m, int q) { return (m.w[q >> 6] >> (q & 63)) & 1ull; }
static inline void mask_set(Mask125& m, int q) { m.w[q >> 6] |= 1ull << (q & 63); }
static inline bool mask_eq(const Mask125& a, const Mask125& b) { return a.w[0] == b.w[0] && a.w[1] == b.w[1]; }

// slots ascending == lexicographic (d1, d2, d3) == ascending CSR column for in-grid entries
static void set_offsets_from_mask(Op* op, const Mask125& mask, int* slot_of /*125*/) {
  op->nofs = 0;
  for (int q = 0; q < 125; ++q) {
    slot_of[q] = -1;
    if (mask_has(mask, q)) {
      slot_of[q] = op->nofs;
      op->d1[op->nofs] = (int8_t)(q / 25 - 2);
      op->d2[op->nofs] = (int8_t)((q / 5) % 5 - 2);
      op->d3[op->nofs] = (int8_t)(q % 5 - 2);
      op->nofs++;
    }
  }
}

static Mask125 layout_mask(const Op& A) {
  Mask125 m{{0ull, 0ull}};
  for (int o = 0; o < A.nofs; ++o) mask_set(m, slot125(A.d1[o], A.d2[o], A.d3[o]));
  return m;
}

Op* op_from_csr(int n1, int n2, int n3, long nnz, const int64_t* indptr, const int32_t* indices, const cplx* data) {
  Ctx& c = Ctx::get();
  const long N = (long)n1 * n2 * n3;
  int64_t* dptr = dalloc<int64_t>(N + 1);
  int32_t* dind = dalloc<int32_t>(nnz);
  cplx* ddat = dalloc<cplx>(nnz);
  unsigned long long* dmask = dalloc<unsigned long long>(3);
  int* dslot = dalloc<int>(125);
  Op* op = new Op();
  op->n1 = n1;
  op->n2 = n2;
  op->n3 = n3;
  op->N = N;
  try {
    HADR_CUDA(cudaMemcpyAsync(dptr, indptr, (N + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, c.stream));
    HADR_CUDA(cudaMemcpyAsync(dind, indices, nnz * sizeof(int32_t), cudaMemcpyHostToDevice, c.stream));
    HADR_CUDA(cudaMemcpyAsync(ddat, data, nnz * sizeof(cplx), cudaMemcpyHostToDevice, c.stream));
    HADR_CUDA(cudaMemsetAsync(dmask, 0, 3 * sizeof(unsigned long long), c.stream));
    launch_csr_mask(c.stream, n1, n2, n3, dptr, dind, dmask);
    unsigned long long hm[3];
    HADR_CUDA(cudaMemcpyAsync(hm, dmask, sizeof(hm), cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    if (hm[2]) throw ValueError("operator reaches beyond the 5x5x5 stencil box; not a structured grid stencil");
    Mask125 m{{hm[0], hm[1]}};
    if (!m.w[0] && !m.w[1]) mask_set(m, slot125(0, 0, 0));  // all-zero matrix: keep a centre plane
    int slot[125];
    set_offsets_from_mask(op, m, slot);
    HADR_CUDA(cudaMemcpyAsync(dslot, slot, sizeof(slot), cudaMemcpyHostToDevice, c.stream));
    op->coef = dalloc<cplx>((size_t)op->nofs * N);
    HADR_CUDA(cudaMemsetAsync(op->coef, 0, (size_t)op->nofs * N * sizeof(cplx), c.stream));
    launch_csr_scatter(c.stream, n1, n2, n3, dptr, dind, ddat, dslot, op->coef);
    HADR_CUDA(cudaGetLastError());
    c.sync();
  } catch (...) {
    dfree(dptr), dfree(dind), dfree(ddat), dfree(dmask), dfree(dslot);
    delete op;
    throw;
  }
  dfree(dptr), dfree(dind), dfree(ddat), dfree(dmask), dfree(dslot);
  return op;
}

Op* op_from_planes(int n1, int n2, int n3, int nofs, const int* offsets, const cplx* coef_host) {
  if (nofs < 1 || nofs > HADR_MAX_OFS) throw ValueError("n_offsets out of range");
  Ctx& c = Ctx::get();
  Op* op = new Op();
  op->n1 = n1;
  op->n2 = n2;
  op->n3 = n3;
  op->N = (long)n1 * n2 * n3;
  op->nofs = nofs;
  for (int o = 0; o < nofs; ++o) {
    const int a = offsets[3 * o], b = offsets[3 * o + 1], cc = offsets[3 * o + 2];
    if (std::abs(a) > 2 || std::abs(b) > 2 || std::abs(cc) > 2 || (n3 == 1 && cc != 0)) {
      delete op;
      throw ValueError("offsets must lie in the 5x5x5 box (d3 = 0 in 2D)");
    }
    op->d1[o] = (int8_t)a;
    op->d2[o] = (int8_t)b;
    op->d3[o] = (int8_t)cc;
    if (o > 0 && slot125(a, b, cc) <= slot125(op->d1[o - 1], op->d2[o - 1], op->d3[o - 1])) {
      delete op;
      throw ValueError("offsets must be strictly ascending in (d1, d2, d3)");
    }
  }
  op->coef = dalloc<cplx>((size_t)nofs * op->N);
  HADR_CUDA(cudaMemcpyAsync(op->coef, coef_host, (size_t)nofs * op->N * sizeof(cplx), cudaMemcpyHostToDevice,
                            c.stream));
  c.sync();
  return op;
}

// alpha*A + beta*B on the union pattern: (alpha*A).data, (beta*B).data, CSR + CSR (helmadr/drivers.py:156)
Op* op_axpby(cplx alpha, const Op& A, cplx beta, const Op& B) {
  if (A.n1 != B.n1 || A.n2 != B.n2 || A.n3 != B.n3) throw ValueError("dimension mismatch");
  if (A.p0 != B.p0 || A.nown != B.nown || A.hal != B.hal || A.stride() != B.stride())
    throw ValueError("slab layout mismatch");
  Ctx& c = Ctx::get();
  Mask125 m = layout_mask(A);
  const Mask125 mb = layout_mask(B);
  m.w[0] |= mb.w[0];
  m.w[1] |= mb.w[1];
  Op* op = new Op();
  copy_geometry(op, A);
  int slot[125];
  set_offsets_from_mask(op, m, slot);
  int ma[HADR_MAX_OFS], mbs[HADR_MAX_OFS];
  for (int o = 0; o < A.nofs; ++o) ma[o] = slot[slot125(A.d1[o], A.d2[o], A.d3[o])];
  for (int o = 0; o < B.nofs; ++o) mbs[o] = slot[slot125(B.d1[o], B.d2[o], B.d3[o])];
  int* dm = dalloc<int>(2 * HADR_MAX_OFS);
  HADR_CUDA(cudaMemcpyAsync(dm, ma, sizeof(ma), cudaMemcpyHostToDevice, c.stream));
  HADR_CUDA(cudaMemcpyAsync(dm + HADR_MAX_OFS, mbs, sizeof(mbs), cudaMemcpyHostToDevice, c.stream));
  alloc_coef(op);
  cplx* ob = op->coef - op->base_off();
  HADR_CUDA(cudaMemsetAsync(ob, 0, (size_t)op->alloc_len() * sizeof(cplx), c.stream));
  launch_remap_planes(c.stream, A.stride(), A.coef - A.base_off(), A.nofs, dm, ob, alpha, 1);
  launch_remap_planes(c.stream, B.stride(), B.coef - B.base_off(), B.nofs, dm + HADR_MAX_OFS, ob, beta, 1);
  HADR_CUDA(cudaGetLastError());
  c.sync();
  dfree(dm);
  return op;
}

static Op* op_clone_with_center(const Op& A) {
  if (A.slab()) throw ValueError("operation not available on slab operators");
  Ctx& c = Ctx::get();
  Mask125 m = layout_mask(A);
  mask_set(m, slot125(0, 0, 0));
  Op* op = new Op();
  copy_geometry(op, A);
  int slot[125];
  set_offsets_from_mask(op, m, slot);
  int ma[HADR_MAX_OFS];
  for (int o = 0; o < A.nofs; ++o) ma[o] = slot[slot125(A.d1[o], A.d2[o], A.d3[o])];
  int* dm = dalloc<int>(HADR_MAX_OFS);
  HADR_CUDA(cudaMemcpyAsync(dm, ma, sizeof(ma), cudaMemcpyHostToDevice, c.stream));
  op->coef = dalloc<cplx>((size_t)op->nofs * op->N);
  HADR_CUDA(cudaMemsetAsync(op->coef, 0, (size_t)op->nofs * op->N * sizeof(cplx), c.stream));
  launch_remap_planes(c.stream, A.N, A.coef, A.nofs, dm, op->coef, mk(1.0, 0.0), 0);
  c.sync();
  dfree(dm);
  return op;
}

Op* op_add_diag_real(const Op& A, cplx sc, const double* field_host) {
  Ctx& c = Ctx::get();
  Op* op = op_clone_with_center(A);
  double* df = dalloc<double>(A.N);
  HADR_CUDA(cudaMemcpyAsync(df, field_host, A.N * sizeof(double), cudaMemcpyHostToDevice, c.stream));
  launch_add_diag_real(c.stream, A.N, op->coef + (long)op->center() * op->N, sc, df);
  HADR_CUDA(cudaGetLastError());
  c.sync();
  dfree(df);
  return op;
}

Op* op_similarity(const Op& A, const cplx* left_host, const cplx* right_host) {
  if (A.slab()) throw ValueError("operation not available on slab operators");
  Ctx& c = Ctx::get();
  Op* op = new Op();
  copy_geometry(op, A);
  op->nofs = A.nofs;
  for (int o = 0; o < A.nofs; ++o) {
    op->d1[o] = A.d1[o];
    op->d2[o] = A.d2[o];
    op->d3[o] = A.d3[o];
  }
  cplx* dl = dalloc<cplx>(A.N);
  cplx* dr = dalloc<cplx>(A.N);
  HADR_CUDA(cudaMemcpyAsync(dl, left_host, A.N * sizeof(cplx), cudaMemcpyHostToDevice, c.stream));
  HADR_CUDA(cudaMemcpyAsync(dr, right_host, A.N * sizeof(cplx), cudaMemcpyHostToDevice, c.stream));
  op->coef = dalloc<cplx>((size_t)A.nofs * A.N);
  launch_similarity(c.stream, A.dev(), op->coef, dl, dr);
  HADR_CUDA(cudaGetLastError());
  c.sync();
  dfree(dl);
  dfree(dr);
  return op;
}

static inline int coarse_dim(int n) { return (n - 1) / 2 + 1; }

static Mask125 galerkin_mask(const Op& A) {
  Ctx& c = Ctx::get();
  unsigned long long* dmask = (unsigned long long*)(c.dscal + 40);
  HADR_CUDA(cudaMemsetAsync(dmask, 0, 2 * sizeof(unsigned long long), c.stream));
  launch_galerkin(c.stream, A.dev(), coarse_dim(A.n1), coarse_dim(A.n2), coarse_dim(A.n3), dmask, nullptr, nullptr);
  Mask125 m{{0ull, 0ull}};
  HADR_CUDA(cudaMemcpyAsync(m.w, dmask, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, c.stream));
  c.sync();
  mask_set(m, slot125(0, 0, 0));  // the diagonal is always kept
  return m;
}

// C's offsets define the planes.  check_mask: the same pass also ORs the non-zero
// pattern; returns false when it is not C's layout (the caller rebuilds).
static bool galerkin_write(const Op& A, Op& C, bool check_mask = false) {
  Ctx& c = Ctx::get();
  int* dslot = dalloc<int>(125);
  int slot[125];
  for (int q = 0; q < 125; ++q) slot[q] = -1;
  for (int o = 0; o < C.nofs; ++o) slot[slot125(C.d1[o], C.d2[o], C.d3[o])] = o;
  HADR_CUDA(cudaMemcpyAsync(dslot, slot, sizeof(slot), cudaMemcpyHostToDevice, c.stream));
  unsigned long long* dmask = check_mask ? (unsigned long long*)(c.dscal + 40) : nullptr;
  if (dmask) HADR_CUDA(cudaMemsetAsync(dmask, 0, 2 * sizeof(unsigned long long), c.stream));
  launch_galerkin(c.stream, A.dev(), C.n1, C.n2, C.n3, dmask, dslot, C.coef);
  HADR_CUDA(cudaGetLastError());
  Mask125 m{{0ull, 0ull}};
  if (dmask) HADR_CUDA(cudaMemcpyAsync(m.w, dmask, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, c.stream));
  c.sync();
  dfree(dslot);
  if (!check_mask) return true;
  mask_set(m, slot125(0, 0, 0));
  return mask_eq(m, layout_mask(C));
}

Op* op_galerkin(const Op& A) {
  if ((A.n1 - 1) % 2 || (A.n2 - 1) % 2 || (A.n3 > 1 && (A.n3 - 1) % 2))
    throw ValueError("cannot coarsen: interval count is odd");
  const Mask125 m = galerkin_mask(A);
  Op* op = new Op();
  op->n1 = coarse_dim(A.n1);
  op->n2 = coarse_dim(A.n2);
  op->n3 = coarse_dim(A.n3);
  op->N = (long)op->n1 * op->n2 * op->n3;
  int slot[125];
  set_offsets_from_mask(op, m, slot);
  op->coef = dalloc<cplx>((size_t)op->nofs * op->N);
  galerkin_write(A, *op);
  return op;
}

// Assembly of the rows of global axis-0 planes [r0, r0 + nr) into an operator whose
// geometry (slab or whole grid) is given; fields are global arrays (host or device).
static Op* assemble_rows(int dim, int n1, int n2, int n3, double h1, double h2, double h3, double omega, int scheme,
                         const int* bc, int src1, int src2, int src3, const double* ksq, const double* gam,
                         const double* g1, const double* g2, const double* g3, const double* lap,
                         bool fields_on_device, int p0, int nown, int hal) {
  if (dim != 2 && dim != 3) throw ValueError("dim must be 2 or 3");
  if (n1 < 5 || n2 < 5 || (dim == 3 && n3 < 5)) throw ValueError("grid needs at least 5 nodes per dimension");
  if (scheme < 0 || scheme > 3) throw ValueError("scheme must be central/upwind1/upwind2/helmholtz");
  if (dim == 2) n3 = 1;
  Ctx& c = Ctx::get();
  const long N = (long)n1 * n2 * n3;
  const long n23 = (long)n2 * n3;
  const bool slab = nown > 0;
  const int own = slab ? nown : n1;
  const int r0 = std::max(p0 - hal, 0), r1 = std::min(p0 + own + hal, n1);
  const int nr = r1 - r0;
  const long NR = (long)nr * n23;
  const double* src[6] = {ksq, gam, g1, g2, g3, lap};
  const bool need[6] = {true, true, scheme != 3, scheme != 3, scheme != 3 && dim == 3, scheme != 3};
  const double* fld[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  double* df = nullptr;
  if (fields_on_device) {
    for (int i = 0; i < 6; ++i) fld[i] = need[i] ? src[i] + (long)r0 * n23 : nullptr;
  } else {
    df = dalloc<double>(6 * NR);
    for (int i = 0; i < 6; ++i)
      if (need[i]) {
        HADR_CUDA(cudaMemcpyAsync(df + i * NR, src[i] + (long)r0 * n23, NR * sizeof(double), cudaMemcpyHostToDevice,
                                  c.stream));
        fld[i] = df + i * NR;
      }
  }
  const int NP = dim == 2 ? 9 : 13;
  const long pst = slab ? (long)(own + 2 * hal) * n23 : N;  // plane stride
  const long boff = slab ? (long)hal * n23 : 0;
  cplx* cp = dalloc<cplx>(NP * pst);
  HADR_CUDA(cudaMemsetAsync(cp, 0, NP * pst * sizeof(cplx), c.stream));
  unsigned* dmask = dalloc<unsigned>(1);
  HADR_CUDA(cudaMemsetAsync(dmask, 0, sizeof(unsigned), c.stream));
  launch_assemble(c.stream, dim, n1, n2, n3, h1, h2, h3, omega, scheme, bc, src1, src2, src3, fld[0], fld[1], fld[2],
                  fld[3], fld[4], fld[5], cp + boff + (long)(r0 - p0) * n23, dmask, r0, nr, pst);
  unsigned hm = 0;
  HADR_CUDA(cudaMemcpyAsync(&hm, dmask, sizeof(unsigned), cudaMemcpyDeviceToHost, c.stream));
  c.sync();
  if (slab) {  // every rank must agree on the offset planes
    unsigned long long w = hm;
    dist_comm()->allreduce_or_u64(&w, 1, c.stream);
    hm = (unsigned)w;
  }
  static const int d9[9][3] = {{-2, 0, 0}, {-1, 0, 0}, {0, -2, 0}, {0, -1, 0}, {0, 0, 0},
                               {0, 1, 0},  {0, 2, 0},  {1, 0, 0},  {2, 0, 0}};
  static const int d13[13][3] = {{-2, 0, 0}, {-1, 0, 0}, {0, -2, 0}, {0, -1, 0}, {0, 0, -2}, {0, 0, -1}, {0, 0, 0},
                                 {0, 0, 1},  {0, 0, 2},  {0, 1, 0},  {0, 2, 0},  {1, 0, 0},  {2, 0, 0}};
  hm |= 1u << (dim == 2 ? 4 : 6);  // keep the centre plane
  Op* op = new Op();
  op->n1 = n1;
  op->n2 = n2;
  op->n3 = n3;
  op->N = N;
  if (slab) {
    op->p0 = p0;
    op->nown = nown;
    op->hal = hal;
    op->pstride = pst;
  }
  int used[13], nu = 0;
  for (int q = 0; q < NP; ++q)
    if (hm & (1u << q)) {
      const int* d = dim == 2 ? d9[q] : d13[q];
      op->d1[nu] = (int8_t)d[0];
      op->d2[nu] = (int8_t)d[1];
      op->d3[nu] = (int8_t)d[2];
      used[nu++] = q;
    }
  op->nofs = nu;
  alloc_coef(op);
  for (int o = 0; o < nu; ++o)
    HADR_CUDA(cudaMemcpyAsync(op->coef - boff + (long)o * pst, cp + (long)used[o] * pst, pst * sizeof(cplx),
                              cudaMemcpyDeviceToDevice, c.stream));
  HADR_CUDA(cudaGetLastError());
  c.sync();
  dfree(df);
  dfree(cp);
  dfree(dmask);
  return op;
}

Op* op_assemble(int dim, int n1, int n2, int n3, double h1, double h2, double h3, double omega, int scheme,
                const int* bc, int src1, int src2, int src3, const double* ksq, const double* gam, const double* g1,
                const double* g2, const double* g3, const double* lap, bool fields_on_device) {
  return assemble_rows(dim, n1, n2, n3, h1, h2, h3, omega, scheme, bc, src1, src2, src3, ksq, gam, g1, g2, g3, lap,
                       fields_on_device, 0, 0, 0);
}

Op* op_assemble_slab(int dim, int n1, int n2, int n3, double h1, double h2, double h3, double omega, int scheme,
                     const int* bc, int src1, int src2, int src3, const double* ksq, const double* gam,
                     const double* g1, const double* g2, const double* g3, const double* lap, bool fields_on_device,
                     int p0, int nown) {
  if (!dist_comm()) throw ValueError("no distributed context");
  return assemble_rows(dim, n1, n2, n3, h1, h2, h3, omega, scheme, bc, src1, src2, src3, ksq, gam, g1, g2, g3, lap,
                       fields_on_device, p0, nown, 1);
}

// Slab Galerkin (multi-GPU): this rank forms coarse rows [cb[r], cb[r+1]) from its fine slab,
// whose lower halo row is exchanged first.  gather = 1: the rows of every rank are
// broadcast so each rank holds the full (replicated) coarse operator; gather = 0: a slab
// operator with one halo row each side.
static Op* op_galerkin_slab(Op& A, const std::vector<int>& cb, bool gather) {
  Comm* cm = dist_comm();
  Ctx& c = Ctx::get();
  if (!A.slab() || A.hal < 1) throw ValueError("galerkin_slab: fine operator is not a slab operator");
  const int r = cm->rank, R = cm->size;
  const int q0 = cb[r], nq = cb[r + 1] - cb[r];
  for (int o = 0; o < A.nofs; ++o)
    cm->halo(A.coef + (long)o * A.stride(), A.n23() * sizeof(cplx), A.own(), 1, c.stream);
  const int n1c = coarse_dim(A.n1), n2c = coarse_dim(A.n2), n3c = coarse_dim(A.n3);
  const long n23c = (long)n2c * n3c, Nc = (long)n1c * n23c;
  unsigned long long* dmask = (unsigned long long*)(c.dscal + 40);
  HADR_CUDA(cudaMemsetAsync(dmask, 0, 2 * sizeof(unsigned long long), c.stream));
  launch_galerkin(c.stream, A.dev(), n1c, n2c, n3c, dmask, nullptr, nullptr, q0, nq, 0);
  Mask125 m{{0ull, 0ull}};
  HADR_CUDA(cudaMemcpyAsync(m.w, dmask, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, c.stream));
  c.sync();
  cm->allreduce_or_u64(m.w, 2, c.stream);
  mask_set(m, slot125(0, 0, 0));
  Op* op = new Op();
  op->n1 = n1c;
  op->n2 = n2c;
  op->n3 = n3c;
  op->N = Nc;
  int slot[125];
  set_offsets_from_mask(op, m, slot);
  if (!gather) {
    op->p0 = q0;
    op->nown = nq;
    op->hal = 1;
    op->pstride = (long)(nq + 2) * n23c;
  }
  alloc_coef(op);
  HADR_CUDA(cudaMemsetAsync(op->coef - op->base_off(), 0, op->alloc_len() * sizeof(cplx), c.stream));
  int* dslot = dalloc<int>(125);
  HADR_CUDA(cudaMemcpyAsync(dslot, slot, sizeof(slot), cudaMemcpyHostToDevice, c.stream));
  if (!gather) {
    launch_galerkin(c.stream, A.dev(), n1c, n2c, n3c, nullptr, dslot, op->coef, q0, nq, op->stride());
  } else {
    // rank-major staging (each rank's rows of all planes contiguous) -> R broadcasts -> plane layout
    cplx* tmp = dalloc<cplx>((size_t)op->nofs * Nc);
    launch_galerkin(c.stream, A.dev(), n1c, n2c, n3c, nullptr, dslot, tmp + (long)op->nofs * q0 * n23c, q0, nq,
                    (long)nq * n23c);
    cm->group_start();
    for (int rr = 0; rr < R; ++rr)
      cm->bcast(tmp + (long)op->nofs * cb[rr] * n23c, (size_t)op->nofs * (cb[rr + 1] - cb[rr]) * n23c * sizeof(cplx),
                rr, c.stream);
    cm->group_end();
    for (int rr = 0; rr < R; ++rr) {
      const size_t w = (size_t)(cb[rr + 1] - cb[rr]) * n23c * sizeof(cplx);
      if (!w) continue;
      HADR_CUDA(cudaMemcpy2DAsync(op->coef + (long)cb[rr] * n23c, Nc * sizeof(cplx),
                                  tmp + (long)op->nofs * cb[rr] * n23c, w, w, op->nofs, cudaMemcpyDeviceToDevice,
                                  c.stream));
    }
    c.sync();
    dfree(tmp);
  }
  HADR_CUDA(cudaGetLastError());
  c.sync();
  dfree(dslot);
  return op;
}

void op_apply(const Op& A, const cplx* x, cplx* y) {
  Ctx& c = Ctx::get();
  StencilArgs a{};
  a.A = A.dev();
  a.x = x;
  a.y = y;
  a.gate = gate_always();
  a.rs = c.rs;
  a.epi = epi_none();
  launch_stencil(c.lc, IN_PLAIN, OUT_APPLY, RED_NONE, a);
}

// ---------------------------------------------------------------------------
// hierarchy
// ---------------------------------------------------------------------------
std::vector<Shape3> coarsenable_levels(int n1, int n2, int n3, int max_levels) {
  // helmadr/multigrid.py:98-110 per axis; an axis of size 1 (2D: n3 = 1) is not coarsened
  std::vector<Shape3> s{{n1, n2, n3}};
  while ((int)s.size() < max_levels) {
    const Shape3 m = s.back();
    const int dims = m.n3 > 1 ? 3 : 2;
    const int mm[3] = {m.n1, m.n2, m.n3};
    int cc[3] = {m.n1, m.n2, m.n3};
    bool ok = true;
    for (int a = 0; a < dims; ++a) {
      if ((mm[a] - 1) % 2) ok = false;
      cc[a] = (mm[a] - 1) / 2 + 1;
      if (cc[a] < 3) ok = false;
    }
    if (!ok) break;
    s.push_back({cc[0], cc[1], cc[2]});
  }
  return s;
}

Hier::~Hier() {
  for (auto& kv : graphs) cudaGraphExecDestroy(kv.second);
  for (auto& L : lv) {
    if (L.own) delete L.A;
    dfree(L.r);
    for (auto* v : L.V) dfree(v);
    dfree(L.w[0]);
    dfree(L.w[1]);
    dfree(L.z);
    dfree(L.rctl);
    dfree(L.fb), dfree(L.fx), dfree(L.fV0), dfree(L.fu), dfree(L.fZ0), dfree(L.fZ1), dfree(L.fw), dfree(L.fr);
    dfree(L.fctl);
  }
  dfree(kact);
  dfree(visits);
  dfree(ce_desc);
}

int g_ce_smem_relax = 1;
int g_defer_mgs = 1;  // option "defer_mgs": fold the MGS dots' finalize kernels into the next axpy

// the level's relaxation fits the engine's shared memory (ce_relax_sm)
static bool level_smr(const Level& L) {
  return g_ce_smem_relax && !L.dist &&
         ce_relax_sm_bytes(L.N, L.A->dev().halo, L.s, CE_CTAS) <= CE_SMEM_BUDGET;
}
int g_ce_smem_coef = 1;  // option "ce_smem_coef": stage a fitting level's coefficient rows in shared memory
// ... and its coefficient rows fit beside it (the standard 2D complex128 stencils, whose
// fast loop reads them: the coarsest 65^2 level of config 2 — 20 stencils per engine launch)
static bool level_smc(const Level& L) {
  const StencilDev A = L.A->dev();
  return g_ce_smem_coef && level_smr(L) && A.std2d && !A.coef32 &&
         ce_relax_smc_bytes(L.N, A.halo, L.s, A.nofs, CE_CTAS) <= CE_SMEM_BUDGET;
}

size_t Hier::ce_tile(int li) const {
  size_t m = 0;  // the engine touches levels li .. coarsest
  for (int i = li; i < (int)lv.size(); ++i) {
    const int h = lv[i].A->dev().halo;
    m = std::max(m, ce_tile_bytes(lv[i].N, h, CE_CTAS));
    if (lv[i].smr) m = std::max(m, ce_relax_sm_bytes(lv[i].N, h, lv[i].s, CE_CTAS));
    if (lv[i].smc) m = std::max(m, ce_relax_smc_bytes(lv[i].N, h, lv[i].s, lv[i].A->nofs, CE_CTAS));
  }
  return m;
}

bool Hier::use_ce(int li) const {
  return ce_desc != nullptr && g_ce_max_n > 0 && li < (int)lv.size() && !lv[li].dist && lv[li].N <= g_ce_max_n && lv[li].N * lv[li].A->nofs <= g_small_max_work &&
         (int)lv.size() <= CE_MAXLEV && ce_tile(li) <= 200 * 1024;
}

const LaunchCfg& Hier::lcf(const Level& L) const { return L.dist ? dlc : L.lc; }

void Hier::xchg(const Level& L, const cplx* v) const {
  if (L.dist) dist_comm()->halo((void*)v, (size_t)L.n2 * L.n3 * sizeof(cplx), L.nown, kHalo, Ctx::get().stream);
}

cplx* Hier::valloc(const Level& L) const {
  if (!L.dist) return dalloc<cplx>(L.N);
  const long h = (long)kHalo * L.n2 * L.n3;
  cplx* p = dalloc<cplx>(L.N + 2 * h);
  HADR_CUDA(cudaMemset(p, 0, (L.N + 2 * h) * sizeof(cplx)));
  return p + h;
}

void Hier::alloc_workspace() {
  const int nl = (int)lv.size();
  for (int i = 0; i < nl; ++i) {
    Level& L = lv[i];
    L.n1 = L.A->n1;
    L.n2 = L.A->n2;
    L.n3 = L.A->n3;
    L.N = L.A->nloc();
    L.dist = L.A->slab();
    L.p0 = L.A->p0;
    L.nown = L.A->own();
    L.dinv = L.A->inv_diag();
    L.s = (i == nl - 1) ? coarse_steps : (i + 2);  // relax_steps(l) = l + 1 (helmadr/multigrid.py:87-88)
    if (L.s > RMAX) throw ValueError("relaxation length exceeds the device limit (16)");
    L.s = (int)std::min<long>(L.s, L.A->N);
    L.smr = level_smr(L);  // the engine descriptor and ce_tile() agree for the hierarchy's lifetime
    L.lc = Ctx::get().lc;
    if (L.n3 == 1 && L.N > g_mid_min_n && L.N <= g_mid_max_n) L.lc.ppt = g_mid_ppt;
    if (L.N * L.A->nofs > g_small_max_work) L.lc.cl_max_n = 0;  // plain grids only
    L.smc = level_smc(L);
    for (int j = 0; j <= L.s; ++j) L.V[j] = valloc(L);
    L.w[0] = valloc(L);
    L.w[1] = valloc(L);
    L.r = valloc(L);
    // (not where the marching kernel runs: it applies D^-1 (s w) to its shared-memory input tiles)
    if (g_relax_split > 0 && L.n3 > 1 && L.N >= g_relax_split && !march_takes(L.A->dev())) L.z = valloc(L);
    L.rctl = dalloc<RelaxCtl>(1);
    HADR_CUDA(cudaMemset(L.rctl, 0, sizeof(RelaxCtl)));
    if (i >= 1) {
      L.fb = valloc(L);
      L.fx = valloc(L);
      L.fV0 = valloc(L);
      L.fu = valloc(L);
      L.fZ0 = valloc(L);
      L.fZ1 = valloc(L);
      L.fw = valloc(L);
      L.fr = valloc(L);
      L.fctl = dalloc<FgCtl>(1);
      HADR_CUDA(cudaMemset(L.fctl, 0, sizeof(FgCtl)));
      // the inner FGMRES(2) tolerance is fixed per hierarchy: set once (fg_init resets the rest)
      HADR_CUDA(cudaMemcpy(&L.fctl->tol, &coarse_tol, sizeof(double), cudaMemcpyHostToDevice));
    }
  }
  kact = dalloc<int>(nl + 1);
  visits = dalloc<int>(nl + 1);
  HADR_CUDA(cudaMemset(kact, 0, (nl + 1) * sizeof(int)));
  HADR_CUDA(cudaMemset(visits, 0, (nl + 1) * sizeof(int)));
  if (c64)  // mixed precision: the K-cycle applies complex64-stored operators
    for (auto& L : lv) L.A->make_c64();
  if (nl <= CE_MAXLEV) {
    CEDesc h{};
    h.nlev = nl;
    h.coarse_steps = lv[nl - 1].s;  // min(coarse_steps, N) as the graph path (helmadr/krylov.py steps = min(steps, n))
    h.coarse_tol = coarse_tol;
    for (int i = 0; i < nl; ++i) {
      const Level& L = lv[i];
      CELevel& d = h.lv[i];
      d.A = L.A->dev();
      d.dinv = L.dinv;
      d.N = L.N;
      d.s = L.s;
      d.smr = L.smr ? 1 : 0;
      d.smc = L.smc ? 1 : 0;
      d.r = L.r;
      for (int j = 0; j <= RMAX; ++j) d.V[j] = L.V[j];
      d.w[0] = L.w[0];
      d.w[1] = L.w[1];
      d.fb = L.fb, d.fx = L.fx, d.fV0 = L.fV0, d.fu = L.fu, d.fZ0 = L.fZ0, d.fZ1 = L.fZ1, d.fw = L.fw, d.fr = L.fr;
    }
    ce_desc = dalloc<CEDesc>(1);
    HADR_CUDA(cudaMemcpy(ce_desc, &h, sizeof(CEDesc), cudaMemcpyHostToDevice));
  }
}

static std::vector<Hier*>& hier_pool() {
  static std::vector<Hier*> p;
  return p;
}

Hier* hier_pool_pop() {
  auto& pool = hier_pool();
  if (pool.empty()) return nullptr;
  Hier* h = pool.back();
  pool.pop_back();
  return h;
}

std::vector<long long> hier_option_signature() {
  return {g_ce_smem_relax, g_ce_smem_coef, g_ce_max_n, g_cl_max_n, g_stencil_tile, g_relax_split, g_class_compress, g_pair_compress,
          g_pdl, g_ce_prof_on, g_kcycle_c64, g_ce_cgs2, g_defer_mgs, g_mid_ppt, g_mid_min_n, g_mid_max_n,
          g_stencil_march, g_march_min_n, g_march_min_n2d, g_small_max_work};
}

void hier_release(Hier* h) {
  if (!h) return;
  auto& pool = hier_pool();
  // a hierarchy released after an option change (e.g. freed late by the Python GC) carries
  // descriptors and graphs of the old options: never recycle it
  if (h->poolable && pool.size() < 4 && h->opt_sig == hier_option_signature()) {
    pool.push_back(h);
    return;
  }
  delete h;
}

// Refresh a recycled hierarchy in place: same shapes and offset layouts, so the
// captured K-cycle graphs (which reference its buffers) stay valid.
static bool hier_refresh(Hier* h, const Op& fine) {
  Ctx& c = Ctx::get();
  Op& L0 = *h->lv[0].A;
  if (L0.n1 != fine.n1 || L0.n2 != fine.n2 || L0.n3 != fine.n3 || !mask_eq(layout_mask(L0), layout_mask(fine)))
    return false;
  HADR_CUDA(cudaMemcpyAsync(L0.coef, fine.coef, (size_t)fine.nofs * fine.N * sizeof(cplx), cudaMemcpyDeviceToDevice,
                            c.stream));
  if (L0.pcode && !L0.pair_compress()) return false;  // kernel path captured in the graphs changed
  for (size_t l = 1; l < h->lv.size(); ++l) {
    Op& F = *h->lv[l - 1].A;
    Op& C = *h->lv[l].A;
    if (!galerkin_write(F, C, true)) return false;  // one pass: values + pattern check
    if (C.ccode && !C.class_compress()) return false;  // kernel path captured in the graphs changed
  }
  for (auto& L : h->lv) {
    L.A->refresh_inv_diag();
    if (h->c64) L.A->make_c64();
  }
  return true;
}

Hier* hier_build(Op* fine, int max_levels, int coarse_steps, double coarse_tol) {
  auto shapes = coarsenable_levels(fine->n1, fine->n2, fine->n3, max_levels);
  if (shapes.size() < 2)
    throw ValueError("grid cannot support two multigrid levels ((n_d - 1) must be even with at least 3 coarse nodes)");
  auto& pool = hier_pool();
  for (size_t i = 0; i < pool.size(); ++i) {
    Hier* h = pool[i];
    if (h->lv.size() != shapes.size() || h->coarse_steps != coarse_steps || h->coarse_tol != coarse_tol ||
        h->c64 != (g_kcycle_c64 != 0) || h->opt_sig != hier_option_signature())
      continue;
    bool same = true;
    for (size_t l = 0; l < shapes.size(); ++l)
      same = same && h->lv[l].n1 == shapes[l].n1 && h->lv[l].n2 == shapes[l].n2 && h->lv[l].n3 == shapes[l].n3;
    if (!same) continue;
    pool.erase(pool.begin() + i);
    if (hier_refresh(h, *fine)) return h;
    delete h;  // layout changed: rebuild from scratch
    break;
  }
  Hier* h = new Hier();
  h->coarse_steps = coarse_steps;
  h->coarse_tol = coarse_tol;
  h->poolable = true;
  h->c64 = g_kcycle_c64 != 0;
  try {
    Level L0;
    L0.A = op_copy(*fine);  // own a copy: the graphs then never depend on the caller's buffers
    L0.own = true;
    h->lv.push_back(L0);
    for (size_t i = 1; i < shapes.size(); ++i) {
      Level L;
      L.A = op_galerkin(*h->lv.back().A);
      L.own = true;
      h->lv.push_back(L);
    }
    if (g_pair_compress && h->lv[0].A->nloc() > g_cl_max_n) h->lv[0].A->pair_compress();
    for (size_t l = 1; l < h->lv.size(); ++l) {  // graph-path levels; in 3D the cluster-engine levels too
      Op& C = *h->lv[l].A;
      if (g_class_compress > (C.n3 > 1 ? 0 : 1) && (C.nloc() > g_cl_max_n || C.n3 > 1)) C.class_compress();
    }
    h->alloc_workspace();
  } catch (...) {
    delete h;
    throw;
  }
  return h;
}

Hier* hier_from_ops(int nlev, Op** ops, int coarse_steps, double coarse_tol) {
  if (nlev < 2) throw ValueError("need at least two levels");
  Hier* h = new Hier();
  h->coarse_steps = coarse_steps;
  h->coarse_tol = coarse_tol;
  try {
    for (int i = 0; i < nlev; ++i) {
      Level L;
      L.A = ops[i];
      if (i > 0 && (ops[i]->n1 != (ops[i - 1]->n1 - 1) / 2 + 1 || ops[i]->n2 != (ops[i - 1]->n2 - 1) / 2 + 1 ||
                    ops[i]->n3 != (ops[i - 1]->n3 - 1) / 2 + 1))
        throw ValueError("level shapes must halve: (n-1)/2+1");
      h->lv.push_back(L);
    }
    h->alloc_workspace();
  } catch (...) {
    delete h;
    throw;
  }
  return h;
}

// ---------------------------------------------------------------------------
// multi-GPU slab hierarchy: levels 0 .. ndist-1 are split in
// axis-0 slabs, the coarse rest is agglomerated (replicated on every rank)
// ---------------------------------------------------------------------------
static std::vector<int> level_bounds(const std::vector<int>& fine, int l, int n1l) {
  std::vector<int> b(fine.size());
  for (size_t r = 0; r + 1 < fine.size(); ++r) b[r] = fine[r] >> l;
  b.back() = n1l;
  return b;
}

// Which levels to split (cost model in DESIGN.md §7): a coarse level stays
// distributed while every slab keeps >= dist_min_planes planes and splitting it saves more
// per reduction-separated step than the collective it adds.  A step at level l moves about
// N_l S_l x 16 B (S_l: coefficient planes per point, nominal 54 for 3D / 15 for 2D coarse
// Galerkin operators); splitting saves (1 - 1/R) of that at ~6.5 TB/s, an all-gather or halo
// exchange over NVLink costs ~20 us, so split while N_l S_l >= dist_min_work R / (R - 1)
// with dist_min_work = 8e6 (= 20 us x 6.5 TB/s / 16 B).  Config 4 (513^2 x 257): levels
// 513^2x257, 257^2x129 and 129^2x65 split at 2-8 ranks, 65^2x33 down replicated.
SlabPlan slab_plan_for(int n1, int n2, int n3, int max_levels, int R) {
  auto shapes = coarsenable_levels(n1, n2, n3, max_levels);
  const int nl = (int)shapes.size();
  if (nl < 2)
    throw ValueError("grid cannot support two multigrid levels ((n_d - 1) must be even with at least 3 coarse nodes)");
  if (R < 1) throw ValueError("slab plan needs at least one rank");
  for (int nd = nl - 1; nd >= 1; --nd) {
    if (g_dist_levels > 0 && nd != std::min(g_dist_levels, nl - 1)) continue;
    std::vector<int> b = slab_bounds(n1, R, 1 << nd);
    if (b.empty()) continue;
    bool ok = true;
    for (int l = 0; l < nd && ok; ++l) {
      const std::vector<int> bl = level_bounds(b, l, shapes[l].n1);
      const int need = l == 0 ? kHalo : std::max(kHalo, g_dist_levels > 0 ? kHalo : g_dist_min_planes);
      for (int r = 0; r < R; ++r) ok = ok && bl[r + 1] - bl[r] >= need;
      const double pts = (double)shapes[l].n1 * shapes[l].n2 * shapes[l].n3;
      const double planes = shapes[l].n3 > 1 ? 54.0 : 15.0;
      if (l > 0 && g_dist_levels <= 0 && R > 1 && pts * planes < g_dist_min_work * R / (R - 1.0)) ok = false;
    }
    if (ok) return SlabPlan{b, nd, nl};
  }
  throw ValueError("grid too small for the requested number of slab ranks");
}

SlabPlan slab_plan(int n1, int n2, int n3, int max_levels) {
  Comm* cm = dist_comm();
  if (!cm) throw ValueError("no distributed context (hadr_dist_init_*)");
  return slab_plan_for(n1, n2, n3, max_levels, cm->size);
}

Hier* hier_build_dist(Op* fine, const SlabPlan& plan, int coarse_steps, double coarse_tol) {
  Comm* cm = dist_comm();
  if (!cm) throw ValueError("no distributed context (hadr_dist_init_*)");
  const int rk = cm->rank;
  if (!fine->slab() || fine->p0 != plan.bounds[rk] || fine->own() != plan.bounds[rk + 1] - plan.bounds[rk])
    throw ValueError("fine operator does not match the slab plan");
  auto shapes = coarsenable_levels(fine->n1, fine->n2, fine->n3, plan.nlev);
  Hier* h = new Hier();
  h->coarse_steps = coarse_steps;
  h->coarse_tol = coarse_tol;
  h->c64 = g_kcycle_c64 != 0;
  h->ndist = plan.ndist;
  h->dlc = Ctx::get().lc;
  h->dlc.dist = &cm->red;
  try {
    Level L0;
    L0.A = op_copy(*fine);
    L0.own = true;
    L0.bounds = level_bounds(plan.bounds, 0, shapes[0].n1);
    h->lv.push_back(L0);
    for (int l = 1; l < plan.nlev; ++l) {
      Op& F = *h->lv.back().A;
      Level L;
      if (l <= plan.ndist) {
        const std::vector<int> cb = level_bounds(plan.bounds, l, shapes[l].n1);
        L.A = op_galerkin_slab(F, cb, l == plan.ndist);
        if (l < plan.ndist) L.bounds = cb;
      } else {
        L.A = op_galerkin(F);
      }
      L.own = true;
      h->lv.push_back(L);
    }
    if (g_pair_compress) h->lv[0].A->pair_compress();
    for (size_t l = 1; l < h->lv.size(); ++l) {  // slab levels and the replicated graph-path levels
      Op& C = *h->lv[l].A;
      if (g_class_compress > (C.n3 > 1 ? 0 : 1) && (C.slab() || C.nloc() > g_cl_max_n)) C.class_compress();
    }
    h->alloc_workspace();
  } catch (...) {
    delete h;
    throw;
  }
  return h;
}

__global__ void k_count(int* visits, int idx, Gate g) {
  if (gate_open(g)) visits[idx] += 1;
}

void Hier::emit_relax(Level& L, const cplx* b, const cplx* x, cplx* xo, int s, Gate g) {
  // helmadr/krylov.py:91-119 ; r = b - A x (skipped for x == 0: r = b exactly)
  Ctx& c = Ctx::get();
  const LaunchCfg& lc0 = lcf(L);
  const StencilDev A = L.A->dev();
  const cplx* r = b;
  if (x) {
    xchg(L, x);
    StencilArgs a{};
    a.A = A;
    a.x = x;
    a.b = b;
    a.y = L.w[1];
    a.gate = g;
    a.rs = c.rs;
    a.epi = epi(EPI_RELAX_BETA, L.rctl, 0, s);  // the epilogue also initialises the control block
    launch_stencil(lc0, IN_PLAIN, OUT_RESID, RED_NORM, a);
    r = L.w[1];
  } else {
    launch_scale(lc0, L.N, b, nullptr, nullptr, RED_NORM, g, c.rs, epi(EPI_RELAX_BETA, L.rctl, 0, s));
  }
  RelaxCtl* rc = L.rctl;
  for (int j = 0; j < s; ++j) {
    Gate gj = gate_var(g.active, &rc->cur, 1u << j);
    cplx* w = L.w[j % 2];
    StencilArgs a{};
    a.A = A;
    a.x = (j == 0) ? r : L.w[(j - 1) % 2];
    a.scale = (j == 0) ? &rc->inv_beta : &rc->inv_hn;
    a.dinv = L.dinv;
    a.vout = L.V[j];
    a.y = w;
    a.u = L.V[0];
    a.gate = gj;
    a.rs = c.rs;
    a.epi = epi(EPI_RELAX_H, rc, 0, j);
    if (L.z) {
      // large 3D level: V[j] = s w and z = D^-1 V[j] once per point, then a plain stencil on z
      // (the fused form re-derives D^-1 (s w) for each of a point's 10-54 neighbours)
      launch_scale_jac(lc0, L.N, a.x, a.scale, L.dinv, L.V[j], L.z, gj);
      a.x = L.z;
      xchg(L, L.z);
    }
    // MGS chain: each dot's 1-block finalize is folded into the next axpy (Pend), the
    // partials alternating between the two scratch buffers
    Pend pend{};
    const bool defer = g_defer_mgs && !L.dist;
    g_defer_out = defer ? &pend : nullptr;
    if (!L.z) {
      xchg(L, a.x);
      launch_stencil(lc0, IN_SCALE | IN_JAC | IN_WRITEV, OUT_APPLY, j == 0 ? RED_DOT_CENTER : RED_DOT, a);
    } else {
      launch_stencil(lc0, IN_PLAIN, OUT_APPLY, RED_DOT, a);
    }
    int buf = 0;  // the producer wrote c.rs
    for (int i = 0; i < j; ++i) {
      Pend in = pend;
      pend = Pend{};
      launch_axpy_red(lc0, L.N, w, &rc->H[i * RMAX + j], L.V[i], RED_DOT, L.V[i + 1], gj, buf ? c.rs : c.rs2,
                      epi(EPI_RELAX_H, rc, i + 1, j), in);
      buf ^= 1;
    }
    g_defer_out = nullptr;
    launch_axpy_red(lc0, L.N, w, &rc->H[j * RMAX + j], L.V[j], RED_NORM, nullptr, gj, buf ? c.rs : c.rs2,
                    epi(EPI_RELAX_STEP, rc, 0, j), pend);
  }
  LinComb lc{};
  for (int j = 0; j < s; ++j) lc.v[j] = L.V[j];
  lc.y = rc->y;
  lc.kptr = &rc->k;
  lc.base = x;
  lc.dinv = L.dinv;
  lc.out = xo;
  launch_lincomb(lc0, L.N, lc, g);
}

void Hier::emit_kcycle(int li, const cplx* b, const cplx* x0, cplx* xo, Gate g, bool count) {
  // helmadr/multigrid.py:132-171
  Ctx& c = Ctx::get();
  const int nl = (int)lv.size();
  if (li < 0 || li >= nl - 1) throw ValueError("level outside 1..n_levels-1");
  if (!x0 && !count && use_ce(li)) {  // the whole cycle fits one cluster
    launch_cluster_engine(c.stream, ce_desc, 0, li, b, xo, g.active, CE_CTAS, ce_tile(li));
    return;
  }
  Level& L = lv[li];
  Level& C = lv[li + 1];
  const LaunchCfg& lc0 = lcf(L);
  if (count) k_count<<<1, 1, 0, c.stream>>>(visits, li, g);
  emit_relax(L, b, x0, xo, L.s, g);
  StencilArgs a{};
  a.A = L.A->dev();
  a.x = xo;
  a.b = b;
  a.y = L.r;
  a.gate = g;
  a.rs = c.rs;
  a.epi = epi_none();
  xchg(L, xo);
  launch_stencil(lc0, IN_PLAIN, OUT_RESID, RED_NONE, a);
  if (!L.dist) {
    launch_restrict(lc0, L.n1, L.n2, L.n3, L.r, C.fb, g);
  } else {
    // slab restriction: coarse rows [cb[r], cb[r+1]) need the fine row below the slab
    Comm* cm = dist_comm();
    const int rk = cm->rank;
    const long n23c = (long)C.n2 * C.n3;
    std::vector<int> cb(cm->size + 1);
    for (int q = 0; q < cm->size; ++q) cb[q] = L.bounds[q] / 2;
    cb[cm->size] = C.n1;
    xchg(L, L.r);
    launch_restrict(lc0, L.n1, L.n2, L.n3, L.r, C.dist ? C.fb : C.fb + (long)cb[rk] * n23c, g, L.p0, cb[rk],
                    cb[rk + 1] - cb[rk]);
    if (!C.dist) {  // agglomerate: every rank gets the whole coarse right-hand side
      cm->group_start();
      for (int q = 0; q < cm->size; ++q)
        cm->bcast(C.fb + (long)cb[q] * n23c, (size_t)(cb[q + 1] - cb[q]) * n23c * sizeof(cplx), q, c.stream);
      cm->group_end();
    }
  }
  if (li + 1 == nl - 1) {
    if (count) k_count<<<1, 1, 0, c.stream>>>(visits, li + 1, g);
    if (!count && use_ce(li + 1))
      launch_cluster_engine(c.stream, ce_desc, 2, li + 1, nullptr, nullptr, g.active, CE_CTAS, ce_tile(li + 1));
    else
      emit_relax(C, C.fb, nullptr, C.fx, C.s, g);
  } else if (!count && use_ce(li + 1)) {
    launch_cluster_engine(c.stream, ce_desc, 1, li + 1, nullptr, nullptr, g.active, CE_CTAS, ce_tile(li + 1));
  } else {
    emit_inner(li + 1, g, count);
  }
  if (!L.dist) {
    launch_prolong_add(lc0, L.n1, L.n2, L.n3, C.fx, xo, g);
  } else {
    xchg(C, C.fx);  // slab coarse level: the row above the coarse slab
    launch_prolong_add(lc0, L.n1, L.n2, L.n3, C.fx, xo, g, L.p0, L.nown, C.dist ? C.p0 : 0);
  }
  emit_relax(L, b, xo, xo, L.s, g);
}

void Hier::emit_inner(int ci, Gate g, bool count) {
  // FGMRES(restart=2, maxiter=2, tol=coarse_tol) on level ci, preconditioned by
  // k_cycle(ci) (helmadr/multigrid.py:159-167, helmadr/krylov.py:122-242)
  Ctx& c = Ctx::get();
  Level& C = lv[ci];
  FgCtl* f = C.fctl;
  const StencilDev A = C.A->dev();
  const long n = C.N;
  const LaunchCfg& lcc = lcf(C);
  int* act = kact + ci;
  const unsigned bA = 1u << FG_A, bC = 1u << FG_CONT, bB = 1u << FG_BRK, bR = 1u << FG_RST;
  launch_scale(lcc, n, C.fb, nullptr, nullptr, RED_NORM, g, c.rs, epi(EPI_FG_INIT, f));
  const Gate gA = gate_var(g.active, &f->path, bA);
  launch_scale(lcc, n, C.fb, &f->inv_r, C.fV0, 0, gA, c.rs, epi_none());
  // ---- iteration 1 ----
  launch_set_gate(c.stream, act, gA);
  emit_kcycle(ci, C.fV0, nullptr, C.fZ0, gate_on(act), count);
  {
    StencilArgs a{};
    a.A = A;
    a.x = C.fZ0;
    a.y = C.fw;
    a.u = C.fV0;
    a.gate = gA;
    a.rs = c.rs;
    a.epi = epi(EPI_FG_S, f, 0, 0);
    xchg(C, a.x);
    launch_stencil(lcc, IN_PLAIN, OUT_APPLY, RED_NORM | RED_DOT, a);
    launch_axpy_red(lcc, n, C.fw, &f->H[0], C.fV0, RED_NORM, nullptr, gA, c.rs, epi(EPI_FG_N, f, 0, 0, 1));
    const Gate gAr = gate_var2(g.active, &f->path, bA, &f->reo, 2u);
    launch_dot(lcc, n, C.fV0, C.fw, gAr, c.rs, epi(EPI_FG_CORR, f, 0, 0));
    launch_axpy_red(lcc, n, C.fw, &f->corr[0], C.fV0, RED_NORM, nullptr, gAr, c.rs, epi(EPI_FG_N2, f, 0, 0, 1));
  }
  // ---- early exit after iteration 1: x = Z0 y0, r = b - A x, restart decision ----
  {
    const Gate gB = gate_var(g.active, &f->path, bB);
    launch_fg_finalize(lcc, n, f, C.fZ0, C.fZ1, C.fx, gB, 1);
    StencilArgs a{};
    a.A = A;
    a.x = C.fx;
    a.b = C.fb;
    a.y = C.fr;
    a.gate = gB;
    a.rs = c.rs;
    a.epi = epi(EPI_FG_RES, f);
    xchg(C, a.x);
    launch_stencil(lcc, IN_PLAIN, OUT_RESID, RED_NORM, a);
  }
  // ---- iteration 2: u = V1 (continue) or u = r/||r|| (restart cycle) ----
  launch_scale(lcc, n, C.fw, &f->inv_w, C.fu, 0, gate_var(g.active, &f->path, bC), c.rs, epi_none());
  launch_scale(lcc, n, C.fr, &f->inv_r, C.fu, 0, gate_var(g.active, &f->path, bR), c.rs, epi_none());
  const Gate gCR = gate_var(g.active, &f->path, bC | bR);
  launch_set_gate(c.stream, act, gCR);
  emit_kcycle(ci, C.fu, nullptr, C.fZ1, gate_on(act), count);
  {  // continue: j = 1 against basis (V0, u)
    const Gate gC = gate_var(g.active, &f->path, bC);
    StencilArgs a{};
    a.A = A;
    a.x = C.fZ1;
    a.y = C.fw;
    a.u = C.fV0;
    a.gate = gC;
    a.rs = c.rs;
    a.epi = epi(EPI_FG_S, f, 0, 1);
    xchg(C, a.x);
    launch_stencil(lcc, IN_PLAIN, OUT_APPLY, RED_NORM | RED_DOT, a);
    launch_axpy_red(lcc, n, C.fw, &f->H[0 * MMAX + 1], C.fV0, RED_DOT, C.fu, gC, c.rs, epi(EPI_FG_H, f, 1, 1));
    launch_axpy_red(lcc, n, C.fw, &f->H[1 * MMAX + 1], C.fu, RED_NORM, nullptr, gC, c.rs,
                    epi(EPI_FG_N, f, 0, 1, 1));
    const Gate gCr = gate_var2(g.active, &f->path, bC, &f->reo, 2u);
    launch_dot(lcc, n, C.fV0, C.fw, gCr, c.rs, epi(EPI_FG_CORR, f, 0, 1));
    launch_axpy_red(lcc, n, C.fw, &f->corr[0], C.fV0, RED_DOT, C.fu, gCr, c.rs, epi(EPI_FG_CORR, f, 1, 1));
    launch_axpy_red(lcc, n, C.fw, &f->corr[1], C.fu, RED_NORM, nullptr, gCr, c.rs, epi(EPI_FG_N2, f, 0, 1, 1));
  }
  {  // restart cycle: j = 0 against basis (u)
    const Gate gR = gate_var(g.active, &f->path, bR);
    StencilArgs a{};
    a.A = A;
    a.x = C.fZ1;
    a.y = C.fw;
    a.u = C.fu;
    a.gate = gR;
    a.rs = c.rs;
    a.epi = epi(EPI_FG_S, f, 0, 0);
    xchg(C, a.x);
    launch_stencil(lcc, IN_PLAIN, OUT_APPLY, RED_NORM | RED_DOT, a);
    launch_axpy_red(lcc, n, C.fw, &f->H[0], C.fu, RED_NORM, nullptr, gR, c.rs, epi(EPI_FG_N, f, 0, 0, 1));
    const Gate gRr = gate_var2(g.active, &f->path, bR, &f->reo, 2u);
    launch_dot(lcc, n, C.fu, C.fw, gRr, c.rs, epi(EPI_FG_CORR, f, 0, 0));
    launch_axpy_red(lcc, n, C.fw, &f->corr[0], C.fu, RED_NORM, nullptr, gRr, c.rs, epi(EPI_FG_N2, f, 0, 0, 1));
  }
  launch_fg_finalize(lcc, n, f, C.fZ0, C.fZ1, C.fx, gate_var(g.active, &f->path, (1u << FG_FIN) | (1u << FG_ZERO)),
                     0);
}

void Hier::apply(const cplx* v, cplx* z) {
  Ctx& c = Ctx::get();
  if (ndist > 0 && !dist_comm()->graphable()) {  // host-callback exchanges: emit directly
    launch_set_gate(c.stream, kact, gate_always());
    emit_kcycle(0, v, nullptr, z, gate_on(kact), false);
    HADR_CUDA(cudaGetLastError());
    return;
  }
  auto key = std::make_pair((const void*)v, (void*)z);
  auto it = graphs.find(key);
  if (it == graphs.end()) {
    cudaGraph_t graph;
    const long long before = g_launch_count;
    HADR_CUDA(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
    try {
      launch_set_gate(c.stream, kact, gate_always());
      emit_kcycle(0, v, nullptr, z, gate_on(kact), false);
    } catch (...) {
      cudaStreamEndCapture(c.stream, &graph);
      g_launch_count = before;
      throw;
    }
    HADR_CUDA(cudaStreamEndCapture(c.stream, &graph));
    graph_kernels[key] = g_launch_count - before;  // captured, not launched
    g_launch_count = before;
    cudaGraphExec_t exec;
    HADR_CUDA(cudaGraphInstantiate(&exec, graph, 0));
    HADR_CUDA(cudaGraphDestroy(graph));
    it = graphs.emplace(key, exec).first;
  }
  HADR_CUDA(cudaGraphLaunch(it->second, c.stream));
  g_launch_count += graph_kernels[key];
}

void Hier::kcycle_direct(int li, const cplx* b, const cplx* x0, cplx* xo, int* visits_host) {
  Ctx& c = Ctx::get();
  const int nl = (int)lv.size();
  HADR_CUDA(cudaMemsetAsync(visits, 0, (nl + 1) * sizeof(int), c.stream));
  launch_set_gate(c.stream, kact + li, gate_always());
  emit_kcycle(li, b, x0, xo, gate_on(kact + li), visits_host != nullptr);
  HADR_CUDA(cudaGetLastError());
  if (visits_host) HADR_CUDA(cudaMemcpyAsync(visits_host, visits, nl * sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  c.sync();
}

// ---------------------------------------------------------------------------
// public gmres_relax (helmadr/krylov.py:82-88)
// ---------------------------------------------------------------------------
void gmres_relax(Op& A, const cplx* b, const cplx* x, cplx* xo, int steps) {
  Ctx& c = Ctx::get();
  if (steps > RMAX) throw ValueError("gmres_relax: steps exceeds the device limit (16)");
  Hier h;  // scratch holder for one level's relaxation workspace
  Level L;
  L.A = &A;
  L.n1 = A.n1;
  L.n2 = A.n2;
  L.n3 = A.n3;
  L.N = A.N;
  L.dinv = A.inv_diag();
  L.s = (int)std::min<long>(std::max(steps, 0), A.N);
  L.lc = c.lc;
  for (int j = 0; j <= L.s; ++j) L.V[j] = dalloc<cplx>(L.N);
  L.w[0] = dalloc<cplx>(L.N);
  L.w[1] = dalloc<cplx>(L.N);
  L.rctl = dalloc<RelaxCtl>(1);
  HADR_CUDA(cudaMemsetAsync(L.rctl, 0, sizeof(RelaxCtl), c.stream));
  h.lv.push_back(L);
  h.emit_relax(h.lv[0], b, x, xo, L.s, gate_always());
  HADR_CUDA(cudaGetLastError());
  c.sync();
  h.lv[0].A = nullptr;  // borrowed
}

// ---------------------------------------------------------------------------
// outer FGMRES (helmadr/krylov.py:122-242); Givens / history / stopping on the
// host exactly as the reference, vector work on the device
// ---------------------------------------------------------------------------
static inline cplx hmul(cplx a, cplx b) { return mk(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
static inline cplx hadd(cplx a, cplx b) { return mk(a.x + b.x, a.y + b.y); }
static inline cplx hsub(cplx a, cplx b) { return mk(a.x - b.x, a.y - b.y); }
static inline cplx hconj(cplx a) { return mk(a.x, -a.y); }
static inline cplx hneg(cplx a) { return mk(-a.x, -a.y); }
static inline double habs(cplx a) { return std::hypot(a.x, a.y); }

struct OuterWS {
  long N = 0;
  int m = 0;
  long h = 0;
  std::vector<cplx*> V, Z;
  cplx *w = nullptr, *r = nullptr, *t = nullptr;  // t: V[:k]^T y of the non-flexible update
  double* gram = nullptr;                          // <v_i, v_j> pairs (collect_diagnostics)
  FgCtl* f = nullptr;
  FgCtl* hf = nullptr;  // pinned
  double* inv = nullptr;  // device scalar(s)
  ~OuterWS() {
    for (auto p : V) dfree(p);
    for (auto p : Z) dfree(p);
    dfree(w), dfree(r), dfree(t), dfree(gram), dfree(f), dfree(inv);
    if (hf) cudaFreeHost(hf);
  }
};

static cplx* halo_vec(long N, long h) {  // h halo entries each side (slab vectors)
  if (!h) return dalloc<cplx>(N);
  cplx* p = dalloc<cplx>(N + 2 * h);
  HADR_CUDA(cudaMemset(p, 0, (N + 2 * h) * sizeof(cplx)));
  return p + h;
}

static OuterWS* outer_ws(long N, int m, long h) {
  static OuterWS* ws = nullptr;
  if (ws && ws->N == N && ws->m >= m && ws->h == h) return ws;
  delete ws;
  ws = new OuterWS();
  ws->N = N;
  ws->m = m;
  ws->h = h;
  for (int j = 0; j <= m; ++j) ws->V.push_back(halo_vec(N, h));
  for (int j = 0; j < m; ++j) ws->Z.push_back(halo_vec(N, h));
  ws->w = halo_vec(N, h);
  ws->r = halo_vec(N, h);
  ws->t = halo_vec(N, h);
  ws->gram = dalloc<double>(2 * MMAX * MMAX);
  ws->f = dalloc<FgCtl>(1);
  HADR_CUDA(cudaMemset(ws->f, 0, sizeof(FgCtl)));
  HADR_CUDA(cudaMallocHost(&ws->hf, sizeof(FgCtl)));
  ws->inv = dalloc<double>(4);
  return ws;
}

void fgmres(Op& A, Hier* M, const cplx* b, const cplx* x0, cplx* x, int restart, int maxiter, double tol,
            Report& rep, int flags) {
  if (restart < 1) throw ValueError("restart must be >= 1");
  if (tol <= 0) throw ValueError("tol must be positive");
  if (restart > MMAX) throw ValueError("restart exceeds the device limit (16)");
  if (M && (M->lv[0].N != A.nloc() || M->lv[0].dist != A.slab())) throw ValueError("preconditioner dimension mismatch");
  Ctx& c = Ctx::get();
  auto t0 = std::chrono::steady_clock::now();
  // slab operator (multi-GPU): vectors are this rank's owned points, with kHalo halo planes
  // around every stencil input (x included: the caller allocates it with halos)
  const long N = A.nloc();
  LaunchCfg lcd = c.lc;
  if (A.slab()) lcd.dist = &dist_comm()->red;
  auto xchg = [&](const cplx* v) {
    if (A.slab()) dist_comm()->halo((void*)v, A.n23() * sizeof(cplx), A.own(), kHalo, c.stream);
  };
  OuterWS* ws = outer_ws(N, restart, A.slab() ? (long)kHalo * A.n23() : 0);
  if (g_pair_compress && !A.pc_tried && N > g_cl_max_n) A.pair_compress();
  const StencilDev Ad = A.dev();
  auto norm2 = [&](const cplx* v) -> double {
    launch_scale(lcd, N, v, nullptr, nullptr, RED_NORM, gate_always(), c.rs, epi_store(c.dscal));
    HADR_CUDA(cudaMemcpyAsync(c.hscal, c.dscal, sizeof(double), cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    return std::sqrt(c.hscal[0]);
  };
  auto resid_norm = [&](const cplx* xx, cplx* rr) -> double {  // rr = b - A xx, ||rr||
    StencilArgs a{};
    a.A = Ad;
    a.x = xx;
    a.b = b;
    a.y = rr;
    a.gate = gate_always();
    a.rs = c.rs;
    a.epi = epi_store(c.dscal);
    xchg(xx);
    launch_stencil(lcd, IN_PLAIN, OUT_RESID, RED_NORM, a);
    HADR_CUDA(cudaMemcpyAsync(c.hscal, c.dscal, sizeof(double), cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    return std::sqrt(c.hscal[0]);
  };
  rep = Report();
  cudaEvent_t ev0, ev1;
  HADR_CUDA(cudaEventCreate(&ev0));
  HADR_CUDA(cudaEventCreate(&ev1));
  HADR_CUDA(cudaEventRecord(ev0, c.stream));
  auto finish_timing = [&]() {
    HADR_CUDA(cudaEventRecord(ev1, c.stream));
    HADR_CUDA(cudaEventSynchronize(ev1));
    float ms = 0.f;
    HADR_CUDA(cudaEventElapsedTime(&ms, ev0, ev1));
    rep.device_time = ms * 1e-3;
    cudaEventDestroy(ev0);
    cudaEventDestroy(ev1);
    rep.wall_time = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  };
  const double bnorm = norm2(b);
  rep.bnorm = bnorm;
  if (bnorm == 0.0) {
    HADR_CUDA(cudaMemsetAsync(x, 0, N * sizeof(cplx), c.stream));
    c.sync();
    rep.history = {0.0};
    rep.converged = 1;
    finish_timing();
    return;
  }
  double rnorm;
  if (x0) {
    if (x0 != x) HADR_CUDA(cudaMemcpyAsync(x, x0, N * sizeof(cplx), cudaMemcpyDeviceToDevice, c.stream));
    rnorm = resid_norm(x, ws->r);
  } else {
    HADR_CUDA(cudaMemsetAsync(x, 0, N * sizeof(cplx), c.stream));
    HADR_CUDA(cudaMemcpyAsync(ws->r, b, N * sizeof(cplx), cudaMemcpyDeviceToDevice, c.stream));
    rnorm = bnorm;  // r = b - A*0 = b
  }
  rep.history.push_back(rnorm);
  const double target = tol * bnorm;
  int it = 0;
  int note = 0;
  std::vector<cplx> H, cs, sn, g;
  FgCtl* f = ws->f;
  FgCtl* hf = ws->hf;
  while (it < maxiter && rnorm > target) {
    const int m = std::min(restart, maxiter - it);
    H.assign((m + 1) * m, mk(0, 0));
    cs.assign(m, mk(0, 0));
    sn.assign(m, mk(0, 0));
    g.assign(m + 1, mk(0, 0));
    g[0] = mk(rnorm, 0);
    auto Hm = [&](int i, int j) -> cplx& { return H[i * m + j]; };
    // V[0] = r / rnorm
    c.hscal[1] = 1.0 / rnorm;  // r / rnorm == r * (1/rnorm) in numpy (Smith division by a real)
    HADR_CUDA(cudaMemcpyAsync(ws->inv, &c.hscal[1], sizeof(double), cudaMemcpyHostToDevice, c.stream));
    launch_scale(lcd, N, ws->r, ws->inv, ws->V[0], 0, gate_always(), c.rs, epi_none());
    int k = 0;
    bool broke = false;
    for (int j = 0; j < m; ++j) {
      const cplx* z = ws->V[j];
      if (M) {
        M->apply(ws->V[j], ws->Z[j]);
        z = ws->Z[j];
      }
      // w = A z ; w0 = ||w|| ; H[0,j] = <V0, w>
      StencilArgs a{};
      a.A = Ad;
      a.x = z;
      a.y = ws->w;
      a.u = ws->V[0];
      a.gate = gate_always();
      a.rs = c.rs;
      a.epi = epi(EPI_FG_S, f, 0, j);
      xchg(z);
      launch_stencil(lcd, IN_PLAIN, OUT_APPLY, RED_NORM | RED_DOT, a);
      for (int i = 0; i < j; ++i)
        launch_axpy_red(lcd, N, ws->w, &f->H[i * MMAX + j], ws->V[i], RED_DOT, ws->V[i + 1], gate_always(), c.rs,
                        epi(EPI_FG_H, f, i + 1, j));
      launch_axpy_red(lcd, N, ws->w, &f->H[j * MMAX + j], ws->V[j], RED_NORM, nullptr, gate_always(), c.rs,
                      epi(EPI_FG_N, f, 0, j, 0));
      const Gate gr = gate_var(nullptr, &f->reo, 2u);
      launch_dot(lcd, N, ws->V[0], ws->w, gr, c.rs, epi(EPI_FG_CORR, f, 0, j));
      for (int i = 0; i < j; ++i)
        launch_axpy_red(lcd, N, ws->w, &f->corr[i], ws->V[i], RED_DOT, ws->V[i + 1], gr, c.rs,
                        epi(EPI_FG_CORR, f, i + 1, j));
      launch_axpy_red(lcd, N, ws->w, &f->corr[j], ws->V[j], RED_NORM, nullptr, gr, c.rs, epi(EPI_FG_N2, f, 0, j, 0));
      HADR_CUDA(cudaGetLastError());
      HADR_CUDA(cudaMemcpyAsync(hf, f, sizeof(FgCtl), cudaMemcpyDeviceToHost, c.stream));
      c.sync();
      for (int i = 0; i <= j; ++i) Hm(i, j) = hf->H[i * MMAX + j];
      const double wnorm = hf->wn;
      Hm(j + 1, j) = mk(wnorm, 0);
      if (!std::isfinite(wnorm)) {
        note = 1;
        broke = true;
        k = j;
        break;
      }
      const bool lucky = wnorm <= kBreakdownEps * std::max(bnorm, 1e-300);
      if (!lucky) {
        c.hscal[2] = 1.0 / wnorm;
        HADR_CUDA(cudaMemcpyAsync(ws->inv + 1, &c.hscal[2], sizeof(double), cudaMemcpyHostToDevice, c.stream));
        launch_scale(lcd, N, ws->w, ws->inv + 1, ws->V[j + 1], 0, gate_always(), c.rs, epi_none());
      }
      for (int i = 0; i < j; ++i) {
        cplx t = hadd(hmul(cs[i], Hm(i, j)), hmul(sn[i], Hm(i + 1, j)));
        Hm(i + 1, j) = hadd(hmul(hneg(hconj(sn[i])), Hm(i, j)), hmul(hconj(cs[i]), Hm(i + 1, j)));
        Hm(i, j) = t;
      }
      const double aa = habs(Hm(j, j)), bb = habs(Hm(j + 1, j));
      const double den = std::sqrt(aa * aa + bb * bb);
      if (den == 0.0) {
        cs[j] = mk(1, 0);
        sn[j] = mk(0, 0);
      } else {
        cs[j] = cdiv_np(hconj(Hm(j, j)), mk(den, 0));
        sn[j] = cdiv_np(hconj(Hm(j + 1, j)), mk(den, 0));
      }
      Hm(j, j) = hadd(hmul(cs[j], Hm(j, j)), hmul(sn[j], Hm(j + 1, j)));
      Hm(j + 1, j) = mk(0, 0);
      g[j + 1] = hmul(hneg(hconj(sn[j])), g[j]);
      g[j] = hmul(cs[j], g[j]);
      it += 1;
      k = j + 1;
      rep.history.push_back(habs(g[j + 1]));
      if (lucky || rep.history.back() <= target) break;
    }
    if ((flags & FG_DIAGNOSTICS) && k > 0) {  // G = V[:k] V[:k]^H off the diagonal (helmadr/krylov.py:214-217)
      int np_ = 0;
      for (int i = 0; i < k; ++i)
        for (int jj = i + 1; jj < k; ++jj, ++np_)
          launch_dot(lcd, N, ws->V[i], ws->V[jj], gate_always(), c.rs, epi_store(ws->gram + 2 * np_));
      if (np_) {
        std::vector<double> gh(2 * np_);
        HADR_CUDA(cudaMemcpyAsync(gh.data(), ws->gram, gh.size() * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
        c.sync();
        for (int q = 0; q < np_; ++q) rep.ortho_max = std::max(rep.ortho_max, std::hypot(gh[2 * q], gh[2 * q + 1]));
      }
    }
    if (k > 0) {
      std::vector<cplx> y(g.begin(), g.begin() + k);
      if (k == 1) {
        y[0] = cdiv_np(g[0], Hm(0, 0));
      } else {
        for (int jj = k - 1; jj >= 0; --jj) {
          y[jj] = cdiv_np(y[jj], Hm(jj, jj));
          for (int i = 0; i < jj; ++i) y[i] = hsub(y[i], hmul(y[jj], Hm(i, jj)));
        }
      }
      const bool flexible = !(flags & FG_NONFLEXIBLE) || !M;
      LinComb lcb{};
      for (int i = 0; i < k; ++i) {
        lcb.v[i] = flexible && M ? ws->Z[i] : ws->V[i];
        lcb.yv[i] = y[i];
      }
      lcb.kfix = k;
      if (flexible) {  // x + Z[:k]^T y
        lcb.base = x;
        lcb.out = x;
        launch_lincomb(lcd, N, lcb, gate_always());
      } else {  // x + M(V[:k]^T y)   (helmadr/krylov.py:222-223)
        lcb.base = nullptr;
        lcb.out = ws->t;
        launch_lincomb(lcd, N, lcb, gate_always());
        M->apply(ws->t, ws->w);
        LinComb add{};
        add.v[0] = ws->w;
        add.yv[0] = mk(1.0, 0.0);
        add.kfix = 1;
        add.base = x;
        add.out = x;
        launch_lincomb(lcd, N, add, gate_always());
      }
    }
    rnorm = resid_norm(x, ws->r);
    if (broke) break;
  }
  rep.iterations = it;
  rep.note = note;
  rep.final_relres = rnorm / bnorm;
  rep.converged = (rnorm <= target * (1.0 + 1e-12)) && !note;
  finish_timing();
}

}  // namespace hadr
