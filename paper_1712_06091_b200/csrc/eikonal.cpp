// Factored-eikonal fast marching on the host (setup; the travel time is an input
// of the amplitude solve, north_star).  A restatement of the reference's
// heap-ordered marcher (helmadr/_fmm.py:22-331, driven by
// helmadr/eikonal.py:72-99): the unknown is t1 in tau = tau0 * t1, one-sided
// upwind differences per axis give a scalar quadratic per node, the larger root
// is the causal one; ties in the heap break on the node index.  Compiled
// without floating-point contraction, so the 2D march reproduces the
// reference's arithmetic (tests pin it against the reference's own output).
//
// 3D (the reference has no 3D marcher): the same local
// solver with a third axis — the all-axes update first, then the one-axis
// updates and the same fallbacks (a decision, documented in DESIGN.md).
#include <cmath>
#include <cstdint>
#include <limits>
#include <stdexcept>
#include <vector>

namespace hadr {
namespace {

constexpr double INF = std::numeric_limits<double>::infinity();
enum : uint8_t { FAR = 0, NARROW = 1, ACCEPTED = 2 };

struct Heap {
  std::vector<double> keys;
  std::vector<int64_t> idxs;
  int64_t size = 0;
  explicit Heap(int64_t cap) : keys(cap), idxs(cap) {}
  // helmadr/_fmm.py:24-40
  void push(double key, int64_t idx) {
    int64_t i = size;
    while (i > 0) {
      const int64_t p = (i - 1) >> 1;
      const double kp = keys[p];
      const int64_t ip = idxs[p];
      if (kp > key || (kp == key && ip > idx)) {
        keys[i] = kp;
        idxs[i] = ip;
        i = p;
      } else {
        break;
      }
    }
    keys[i] = key;
    idxs[i] = idx;
    ++size;
  }
  // helmadr/_fmm.py:43-67
  void pop(double& key, int64_t& idx) {
    key = keys[0];
    idx = idxs[0];
    --size;
    const double lk = keys[size];
    const int64_t li = idxs[size];
    int64_t i = 0;
    for (;;) {
      int64_t c = 2 * i + 1;
      if (c >= size) break;
      if (c + 1 < size && (keys[c + 1] < keys[c] || (keys[c + 1] == keys[c] && idxs[c + 1] < idxs[c]))) c += 1;
      if (keys[c] < lk || (keys[c] == lk && idxs[c] < li)) {
        keys[i] = keys[c];
        idxs[i] = idxs[c];
        i = c;
      } else {
        break;
      }
    }
    keys[i] = lk;
    idxs[i] = li;
  }
};

// larger real root of A t^2 + B t + C = 0, stable form (helmadr/_fmm.py:70-88)
bool larger_root(double A, double B, double C, double& r) {
  if (A == 0.0) {
    if (B == 0.0) return false;
    r = -C / B;
    return true;
  }
  const double disc = B * B - 4.0 * A * C;
  if (disc < 0.0) return false;
  const double sq = std::sqrt(disc);
  const double qq = B >= 0.0 ? -0.5 * (B + sq) : -0.5 * (B - sq);
  double r1 = qq / A;
  if (qq != 0.0) {
    const double r2 = C / qq;
    if (r2 > r1) r1 = r2;
  }
  r = r1;
  return true;
}

struct AxisData {
  bool have = false, have2 = false;
  double a1 = 0, b1 = 0, a2 = 0, b2 = 0, nbt = 0, h = 0;
};

// upwind one-sided difference data of one axis (helmadr/_fmm.py:91-125)
AxisData axis_data(int64_t k, int i, int size, int64_t stride, double h, const double* tau1, const double* tau,
                   const uint8_t* state, int order) {
  AxisData d;
  d.h = h;
  double tm = INF, tp = INF;
  if (i > 0 && state[k - stride] == ACCEPTED) tm = tau[k - stride];
  if (i < size - 1 && state[k + stride] == ACCEPTED) tp = tau[k + stride];
  if (tm == INF && tp == INF) return d;
  int s;
  if (tm <= tp) {
    s = -1;
    d.nbt = tm;
  } else {
    s = 1;
    d.nbt = tp;
  }
  const int64_t nb1 = k + s * stride;
  d.a1 = (double)(-s) / h;
  d.b1 = (double)s * tau1[nb1] / h;
  if (order == 2) {
    const int j2 = i + 2 * s;
    if (0 <= j2 && j2 < size) {
      const int64_t nb2 = k + 2 * s * stride;
      // the in-line second value must not exceed the first
      if (state[nb2] == ACCEPTED && tau[nb2] <= tau[nb1] + 1e-12 * (1.0 + tau[nb1])) {
        d.have2 = true;
        d.a2 = (double)(-s) * 3.0 / (2.0 * h);
        d.b2 = (double)s * (4.0 * tau1[nb1] - tau1[nb2]) / (2.0 * h);
      }
    }
  }
  d.have = true;
  return d;
}

inline bool causal(double cand, double nbt) { return cand >= nbt - 1e-12 * (1.0 + nbt); }

struct Grid {
  int dim;
  int n[3];
  double h[3];
  int64_t stride[3];
  const double* tau0;
  const double* g0[3];
  const double* kappa;
};

// candidate t1 at node k from the accepted neighbours; -1 if none (helmadr/_fmm.py:133-230)
double node_candidate(const Grid& G, int64_t k, const double* tau1, const double* tau, const uint8_t* state,
                      int order) {
  const double t0 = G.tau0[k];
  const double ksq = G.kappa[k] * G.kappa[k];
  int idx[3];
  {
    int64_t r = k;
    for (int a = G.dim - 1; a >= 0; --a) {
      idx[a] = (int)(r % G.n[a]);
      r /= G.n[a];
    }
  }
  AxisData ax[3];
  bool any = false, all = true;
  for (int a = 0; a < G.dim; ++a) {
    ax[a] = axis_data(k, idx[a], G.n[a], G.stride[a], G.h[a], tau1, tau, state, order);
    any = any || ax[a].have;
    all = all && ax[a].have;
  }
  if (!any) return -1.0;
  double g0[3];
  for (int a = 0; a < G.dim; ++a) g0[a] = G.g0[a][k];

  // full update over every axis with the per-axis selected orders
  if (all) {
    double p[3], q[3];
    for (int a = 0; a < G.dim; ++a) {
      if (ax[a].have2) {
        p[a] = t0 * ax[a].a2 + g0[a];
        q[a] = t0 * ax[a].b2;
      } else {
        p[a] = t0 * ax[a].a1 + g0[a];
        q[a] = t0 * ax[a].b1;
      }
    }
    double A = p[0] * p[0] + p[1] * p[1];
    double Bi = p[0] * q[0] + p[1] * q[1];
    double Cq = q[0] * q[0] + q[1] * q[1];
    double nmax = ax[0].nbt >= ax[1].nbt ? ax[0].nbt : ax[1].nbt;
    if (G.dim == 3) {
      A = A + p[2] * p[2];
      Bi = Bi + p[2] * q[2];
      Cq = Cq + q[2] * q[2];
      nmax = nmax >= ax[2].nbt ? nmax : ax[2].nbt;
    }
    double t;
    if (larger_root(A, 2.0 * Bi, Cq - ksq, t) && t > 0.0) {
      const double cand = t0 * t;
      if (causal(cand, nmax)) return t;
    }
  }

  double best = INF, best_t1 = -1.0;
  if (G.dim == 3) {  // 3D extension: two-axis updates before the one-axis ones
    for (int a = 0; a < 3; ++a)
      for (int b = a + 1; b < 3; ++b) {
        if (!ax[a].have || !ax[b].have) continue;
        const int ab[2] = {a, b};
        double p[2], q[2];
        for (int m = 0; m < 2; ++m) {
          const AxisData& d = ax[ab[m]];
          p[m] = t0 * (d.have2 ? d.a2 : d.a1) + g0[ab[m]];
          q[m] = t0 * (d.have2 ? d.b2 : d.b1);
        }
        double t;
        if (larger_root(p[0] * p[0] + p[1] * p[1], 2.0 * (p[0] * q[0] + p[1] * q[1]), q[0] * q[0] + q[1] * q[1] - ksq,
                        t) &&
            t > 0.0 && causal(t0 * t, ax[a].nbt >= ax[b].nbt ? ax[a].nbt : ax[b].nbt) && t0 * t < best) {
          best = t0 * t;
          best_t1 = t;
        }
      }
    if (best_t1 > 0.0) return best_t1;
  }

  // one-axis updates: second order if admissible, else first order
  for (int a = 0; a < G.dim; ++a) {
    const AxisData& d = ax[a];
    if (!d.have) continue;
    bool done = false;
    double t;
    if (d.have2) {
      const double p = t0 * d.a2 + g0[a];
      const double q = t0 * d.b2;
      if (larger_root(p * p, 2.0 * p * q, q * q - ksq, t) && t > 0.0 && causal(t0 * t, d.nbt)) {
        if (t0 * t < best) {
          best = t0 * t;
          best_t1 = t;
        }
        done = true;
      }
    }
    if (!done) {
      const double p = t0 * d.a1 + g0[a];
      const double q = t0 * d.b1;
      if (larger_root(p * p, 2.0 * p * q, q * q - ksq, t) && t > 0.0 && causal(t0 * t, d.nbt)) {
        if (t0 * t < best) {
          best = t0 * t;
          best_t1 = t;
        }
      }
    }
  }
  if (best_t1 > 0.0) return best_t1;

  // no admissible root: the one-axis first-order root, else tau_nb + h*kappa
  for (int a = 0; a < G.dim; ++a) {
    const AxisData& d = ax[a];
    if (!d.have) continue;
    const double p = t0 * d.a1 + g0[a];
    const double q = t0 * d.b1;
    double t;
    if (!(larger_root(p * p, 2.0 * p * q, q * q - ksq, t) && t > 0.0)) t = (d.nbt + d.h * G.kappa[k]) / t0;
    if (best_t1 < 0.0 || t0 * t < best) {
      best = t0 * t;
      best_t1 = t;
    }
  }
  return best_t1;
}

}  // namespace

// Returns the number of accepted nodes (== N on success), or -(accepted) when the heap
// capacity (6N + 16, as the reference) is exceeded.
int64_t fast_march(int dim, const int* n, const double* h, const double* tau0, const double* const* g0,
                   const double* kappa, const int* src, int order, double* tau1_out) {
  if (dim != 2 && dim != 3) throw std::invalid_argument("dim must be 2 or 3");
  if (order != 1 && order != 2) throw std::invalid_argument("order must be 1 or 2");
  Grid G{};
  G.dim = dim;
  int64_t N = 1;
  for (int a = 0; a < dim; ++a) {
    G.n[a] = n[a];
    G.h[a] = h[a];
    G.g0[a] = g0[a];
    N *= n[a];
    if (src[a] < 0 || src[a] >= n[a]) throw std::invalid_argument("source outside the grid");
  }
  {
    int64_t s = 1;
    for (int a = dim - 1; a >= 0; --a) {
      G.stride[a] = s;
      s *= n[a];
    }
  }
  G.tau0 = tau0;
  G.kappa = kappa;
  double* tau1 = tau1_out;
  std::vector<double> tau(N, INF);
  std::vector<uint8_t> state(N, FAR);
  for (int64_t k = 0; k < N; ++k) tau1[k] = INF;
  Heap heap(6 * N + 16);

  // seed the source and its in-grid box neighbourhood at t1 = kappa(x0) (helmadr/_fmm.py:233-261)
  int64_t ks = 0;
  for (int a = 0; a < dim; ++a) ks += (int64_t)src[a] * G.stride[a];
  const double kap0 = kappa[ks];
  std::vector<int64_t> seeds;
  const int span3 = dim == 3 ? 1 : 0;
  for (int d1 = -1; d1 <= 1; ++d1)
    for (int d2 = -1; d2 <= 1; ++d2)
      for (int d3 = -span3; d3 <= span3; ++d3) {
        const int dd[3] = {d1, d2, d3};
        bool in = true;
        int64_t kk = 0;
        for (int a = 0; a < dim; ++a) {
          const int j = src[a] + dd[a];
          in = in && j >= 0 && j < n[a];
          kk += (int64_t)j * G.stride[a];
        }
        if (!in) continue;
        tau1[kk] = kap0;
        tau[kk] = tau0[kk] * kap0;
        state[kk] = ACCEPTED;
        seeds.push_back(kk);
      }
  const int nseed = (int)seeds.size();
  for (int a = 0; a < nseed; ++a) {  // selection sort by (tau, index)
    int m = a;
    for (int b = a + 1; b < nseed; ++b)
      if (tau[seeds[b]] < tau[seeds[m]] || (tau[seeds[b]] == tau[seeds[m]] && seeds[b] < seeds[m])) m = b;
    std::swap(seeds[a], seeds[m]);
  }
  int64_t naccept = nseed;

  // accept node kk: relax its face neighbours (helmadr/_fmm.py:264-290)
  auto relax = [&](int64_t kk) -> bool {
    int idx[3];
    int64_t r = kk;
    for (int a = dim - 1; a >= 0; --a) {
      idx[a] = (int)(r % n[a]);
      r /= n[a];
    }
    for (int a = 0; a < dim; ++a)
      for (int sgn = -1; sgn <= 1; sgn += 2) {
        const int j = idx[a] + sgn;
        if (j < 0 || j >= n[a]) continue;
        const int64_t nb = kk + sgn * G.stride[a];
        if (state[nb] == ACCEPTED) continue;
        const double t = node_candidate(G, nb, tau1, tau.data(), state.data(), order);
        if (t > 0.0 && tau0[nb] * t < tau[nb]) {
          tau1[nb] = t;
          tau[nb] = tau0[nb] * t;
          state[nb] = NARROW;
          if (heap.size >= (int64_t)heap.keys.size()) return false;
          heap.push(tau[nb], nb);
        }
      }
    return true;
  };

  for (int s = 0; s < nseed; ++s)
    if (!relax(seeds[s])) return -naccept;
  while (heap.size > 0) {  // helmadr/_fmm.py:293-331
    double key;
    int64_t idx;
    heap.pop(key, idx);
    if (state[idx] == ACCEPTED) continue;
    if (key > tau[idx]) continue;  // stale entry
    state[idx] = ACCEPTED;
    ++naccept;
    if (!relax(idx)) return -naccept;
  }
  return naccept;
}

}  // namespace hadr
