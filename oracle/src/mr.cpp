// ORACLE — test infrastructure only (see oracle.hpp).
// Multiresolution tree (reading O.6 with grading radius 2,
// DESIGN.md R-G2), FV diffusion operator on the leaves (reading O.5,
// DESIGN.md R-F), Rock4 integration (reading O.4), the
// reaction substep over leaves and the Strang step.
//
// Data structure: a hash map key -> node over ALL tree nodes, deliberately
// unlike the GPU's dense level arrays and the paper's blocks.  All passes are
// plain loops.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <thread>

#include "oracle.hpp"

namespace orc {

namespace {
constexpr int kGradeRadius = 2;  // DESIGN.md R-G2

int pow3(int d) { return d == 2 ? 9 : 27; }

void key_coords(int dim, uint64_t key, int* level, int32_t* k) {
  *level = key_level(key);
  demorton(dim, *level, key_morton(key), k);
}

void child_coords(int dim, const int32_t* k, int delta, int32_t* c) {
  // Morton child order: the appended digit group is (b_x, b_y[, b_z]), x most significant.
  for (int a = 0; a < dim; ++a) c[a] = 2 * k[a] + ((delta >> (dim - 1 - a)) & 1);
}

int32_t mirror(int32_t i, int level) {
  const int32_t n = int32_t(1) << level;
  if (i < 0) return 0;          // even mirror u_{-1} := u_0 (reading S10)
  if (i >= n) return n - 1;
  return i;
}

bool inside(int dim, int level, const int32_t* k) {
  const int32_t n = int32_t(1) << level;
  for (int a = 0; a < dim; ++a)
    if (k[a] < 0 || k[a] >= n) return false;
  return true;
}

// P2 (Eq. inter_1d; tensor product P:619-621): separable, x then y
// then z; r = u0 + s * 0.125 * (u_minus - u_plus), s = +1 for child bit 0.
double step1d(double um, double u0, double up, int bit) {
  double dlt = um - up;
  double t = 0.125 * dlt;
  if (bit) t = -t;
  return u0 + t;
}

double predict_vals(int dim, const double* v, const int* cb) {
  if (dim == 2) {
    double r[3];
    for (int oy = 0; oy < 3; ++oy) r[oy] = step1d(v[oy * 3 + 0], v[oy * 3 + 1], v[oy * 3 + 2], cb[0]);
    return step1d(r[0], r[1], r[2], cb[1]);
  }
  double q[3];
  for (int oz = 0; oz < 3; ++oz) {
    double r[3];
    for (int oy = 0; oy < 3; ++oy) {
      const double* w = v + (oz * 3 + oy) * 3;
      r[oy] = step1d(w[0], w[1], w[2], cb[0]);
    }
    q[oz] = step1d(r[0], r[1], r[2], cb[1]);
  }
  return step1d(q[0], q[1], q[2], cb[2]);
}

// 3^d neighbourhood of (level, k), mirrored at the domain boundary; index ((oz*3+oy)*3+ox).
int stencil_keys(int dim, int level, const int32_t* k, uint64_t* out) {
  int n = 0;
  const int nz = dim == 3 ? 3 : 1;
  for (int oz = 0; oz < nz; ++oz)
    for (int oy = 0; oy < 3; ++oy)
      for (int ox = 0; ox < 3; ++ox) {
        int32_t c[3];
        const int o[3] = {ox - 1, oy - 1, oz - 1};
        for (int a = 0; a < dim; ++a) c[a] = mirror(k[a] + o[a], level);
        out[n++] = make_key(dim, level, c);
      }
  return n;
}

// Predict node (level j, k) from its parent's neighbourhood using stored node values.
bool predict_node(const Grid& g, int j, const int32_t* k, int comp_count, double* out) {
  int32_t p[3];
  int cb[3] = {0, 0, 0};
  for (int a = 0; a < g.dim; ++a) { p[a] = k[a] >> 1; cb[a] = k[a] & 1; }
  uint64_t sk[27];
  const int ns = stencil_keys(g.dim, j - 1, p, sk);
  std::vector<const Node*> sn(ns);
  for (int s = 0; s < ns; ++s) {
    auto it = g.nodes.find(sk[s]);
    if (it == g.nodes.end()) return false;
    sn[s] = &it->second;
  }
  double v[27];
  for (int i = 0; i < comp_count; ++i) {
    for (int s = 0; s < ns; ++s) v[s] = sn[s]->u[i];
    out[i] = predict_vals(g.dim, v, cb);
  }
  return true;
}

// P1: parent = (((c0 + c1) + c2) + ...) * 2^-d, children in Morton order.
void project_node(Grid& g, uint64_t key) {
  int j;
  int32_t k[3];
  key_coords(g.dim, key, &j, k);
  Node& P = g.nodes.at(key);
  const int nc = 1 << g.dim;
  std::vector<const Node*> ch(nc);
  for (int d = 0; d < nc; ++d) {
    int32_t c[3];
    child_coords(g.dim, k, d, c);
    ch[d] = &g.nodes.at(make_key(g.dim, j + 1, c));
  }
  const double scale = std::ldexp(1.0, -g.dim);
  for (int i = 0; i < g.m; ++i) {
    double s = ch[0]->u[i];
    for (int d = 1; d < nc; ++d) s = s + ch[d]->u[i];
    P.u[i] = s * scale;
  }
}

std::vector<uint64_t> sorted_keys(const Grid& g, bool want_leaf) {
  std::vector<uint64_t> ks;
  for (auto& kv : g.nodes)
    if (kv.second.leaf == want_leaf) ks.push_back(kv.first);
  std::sort(ks.begin(), ks.end());
  return ks;
}

// Projection of leaf values onto every internal node, finest level first.
void project_all(Grid& g) {
  std::vector<uint64_t> ik = sorted_keys(g, false);
  std::sort(ik.begin(), ik.end(), [](uint64_t a, uint64_t b) {
    if (key_level(a) != key_level(b)) return key_level(a) > key_level(b);
    return a < b;
  });
  for (uint64_t key : ik) project_node(g, key);
}

// P3/P4: details and significance Q(n) = max_i (d_i/s_i)^2 for every node with
// level >= max(1, lmin); s_i = max(1, max over leaves |u_i|) (reading C6).
int compute_significance(Grid& g) {
  std::vector<double> smax(g.m, 1.0);
  for (auto& kv : g.nodes)
    if (kv.second.leaf)
      for (int i = 0; i < g.m; ++i) smax[i] = std::max(smax[i], std::fabs(kv.second.u[i]));
  std::vector<double> uh(g.m);
  for (auto& kv : g.nodes) {
    int j;
    int32_t k[3];
    key_coords(g.dim, kv.first, &j, k);
    kv.second.Q = 0.0;
    if (j < std::max(1, g.lmin)) continue;
    if (!predict_node(g, j, k, g.m, uh.data())) return -5;
    double Q = 0.0;
    for (int i = 0; i < g.m; ++i) {
      double dd = kv.second.u[i] - uh[i];
      double t = dd / smax[i];
      Q = std::max(Q, t * t);
    }
    kv.second.Q = Q;
  }
  return 0;
}

double threshold_sq(const Grid& g, int j) {  // E_j = eps^2 2^{d (j - J)}
  return std::ldexp(g.eps * g.eps, g.dim * (j - g.lmax));
}

// P7: coarsening to a fixed point; all collapsible nodes collapse simultaneously.
void coarsen_fixed_point(Grid& g) {
  const int nc = 1 << g.dim;
  while (true) {
    std::vector<uint64_t> collapse;
    for (auto& kv : g.nodes) {
      const Node& P = kv.second;
      if (P.leaf) continue;
      int j;
      int32_t k[3];
      key_coords(g.dim, kv.first, &j, k);
      if (j < g.lmin) continue;
      const double E = threshold_sq(g, j + 1);
      bool ok = true;
      for (int d = 0; d < nc && ok; ++d) {
        int32_t c[3];
        child_coords(g.dim, k, d, c);
        auto it = g.nodes.find(make_key(g.dim, j + 1, c));
        if (it == g.nodes.end()) { ok = false; break; }
        const Node& C = it->second;
        if (!C.leaf || C.is_new || !(C.Q < E)) ok = false;
      }
      if (!ok) continue;
      // no internal node at level j+1 within distance kGradeRadius of any child
      int32_t lo[3], hi[3];
      for (int a = 0; a < g.dim; ++a) { lo[a] = 2 * k[a] - kGradeRadius; hi[a] = 2 * k[a] + 1 + kGradeRadius; }
      int32_t q[3] = {0, 0, 0};
      const int32_t zlo = g.dim == 3 ? lo[2] : 0, zhi = g.dim == 3 ? hi[2] : 0;
      for (q[2] = zlo; q[2] <= zhi && ok; ++q[2])
        for (q[1] = lo[1]; q[1] <= hi[1] && ok; ++q[1])
          for (q[0] = lo[0]; q[0] <= hi[0] && ok; ++q[0]) {
            if (!inside(g.dim, j + 1, q)) continue;
            auto it = g.nodes.find(make_key(g.dim, j + 1, q));
            if (it != g.nodes.end() && !it->second.leaf) ok = false;
          }
      if (ok) collapse.push_back(kv.first);
    }
    if (collapse.empty()) break;
    for (uint64_t key : collapse) {
      int j;
      int32_t k[3];
      key_coords(g.dim, key, &j, k);
      for (int d = 0; d < nc; ++d) {
        int32_t c[3];
        child_coords(g.dim, k, d, c);
        g.nodes.erase(make_key(g.dim, j + 1, c));
      }
      g.nodes.at(key).leaf = true;  // value = its projection (already stored)
    }
  }
}

void refine_leaf(Grid& g, uint64_t key) {
  int j;
  int32_t k[3];
  key_coords(g.dim, key, &j, k);
  Node& L = g.nodes.at(key);
  L.leaf = false;
  for (int d = 0; d < (1 << g.dim); ++d) {
    int32_t c[3];
    child_coords(g.dim, k, d, c);
    Node n;
    n.leaf = true;
    n.is_new = true;
    n.u.assign(g.m, 0.0);
    g.nodes.emplace(make_key(g.dim, j + 1, c), std::move(n));
  }
}

// P5/P6 grading repair: for every internal node, every level-j position within
// distance kGradeRadius inside Omega must be present; refine the covering leaf.
void grade_fixed_point(Grid& g) {
  while (true) {
    std::vector<uint64_t> to_refine;
    for (auto& kv : g.nodes) {
      if (kv.second.leaf) continue;
      int j;
      int32_t k[3];
      key_coords(g.dim, kv.first, &j, k);
      int32_t q[3] = {0, 0, 0};
      const int R = kGradeRadius;
      const int32_t zlo = g.dim == 3 ? k[2] - R : 0, zhi = g.dim == 3 ? k[2] + R : 0;
      for (q[2] = zlo; q[2] <= zhi; ++q[2])
        for (q[1] = k[1] - R; q[1] <= k[1] + R; ++q[1])
          for (q[0] = k[0] - R; q[0] <= k[0] + R; ++q[0]) {
            if (!inside(g.dim, j, q)) continue;
            if (g.nodes.count(make_key(g.dim, j, q))) continue;
            int32_t a[3] = {q[0], q[1], q[2]};
            int la = j;
            while (true) {
              for (int x = 0; x < g.dim; ++x) a[x] >>= 1;
              --la;
              auto it = g.nodes.find(make_key(g.dim, la, a));
              if (it != g.nodes.end()) { to_refine.push_back(it->first); break; }
            }
          }
    }
    if (to_refine.empty()) break;
    std::sort(to_refine.begin(), to_refine.end());
    to_refine.erase(std::unique(to_refine.begin(), to_refine.end()), to_refine.end());
    for (uint64_t key : to_refine)
      if (g.nodes.at(key).leaf) refine_leaf(g, key);
  }
}

std::vector<Rock4Coeffs> g_table;
}  // namespace

// Test hooks exposing the oracle's own threshold and prediction (pinned in tests/test_oracle_mr.py).
double mr_threshold_sq(int dim, int lmax, double eps, int j) {
  Grid g;
  g.dim = dim; g.lmax = lmax; g.eps = eps;
  return threshold_sq(g, j);
}
double mr_predict_vals(int dim, const double* v, const int* cb) { return predict_vals(dim, v, cb); }

// ============================================================== build / adapt
int grid_build(Grid& g, int dim, int lmin, int lmax, double eps, int m, const double* u) {
  if ((dim != 2 && dim != 3) || lmin < 0 || lmin > lmax || lmax > level_cap(dim) || m < 1 || eps < 0)
    return -1;
  g = Grid();
  g.dim = dim; g.lmin = lmin; g.lmax = lmax; g.eps = eps; g.m = m;
  const int64_t n1 = int64_t(1) << lmax;
  const int64_t N = dim == 2 ? n1 * n1 : n1 * n1 * n1;
  for (int64_t idx = 0; idx < N; ++idx) {  // row-major, x fastest
    int32_t k[3] = {int32_t(idx % n1), int32_t((idx / n1) % n1), int32_t(idx / (n1 * n1))};
    Node nd;
    nd.leaf = true;
    nd.u.resize(m);
    for (int i = 0; i < m; ++i) nd.u[i] = u[i * N + idx];
    g.nodes.emplace(make_key(dim, lmax, k), std::move(nd));
  }
  for (int j = lmax - 1; j >= 0; --j) {
    const int64_t nj = int64_t(1) << j;
    const int64_t Nj = dim == 2 ? nj * nj : nj * nj * nj;
    for (int64_t idx = 0; idx < Nj; ++idx) {
      int32_t k[3] = {int32_t(idx % nj), int32_t((idx / nj) % nj), int32_t(idx / (nj * nj))};
      Node nd;
      nd.leaf = false;
      nd.u.assign(m, 0.0);
      uint64_t key = make_key(dim, j, k);
      g.nodes.emplace(key, std::move(nd));
      project_node(g, key);
    }
  }
  if (int rc = compute_significance(g)) return rc;
  coarsen_fixed_point(g);
  grid_compile(g);
  return grid_check_graded(g);
}

int grid_from_leaves(Grid& g, int dim, int lmin, int lmax, double eps, int m, int64_t n,
                     const uint64_t* keys, const double* u) {
  if ((dim != 2 && dim != 3) || lmin < 0 || lmin > lmax || lmax > level_cap(dim) || m < 1) return -1;
  g = Grid();
  g.dim = dim; g.lmin = lmin; g.lmax = lmax; g.eps = eps; g.m = m;
  for (int64_t r = 0; r < n; ++r) {
    Node nd;
    nd.leaf = true;
    nd.u.resize(m);
    for (int i = 0; i < m; ++i) nd.u[i] = u[i * n + r];
    if (!g.nodes.emplace(keys[r], std::move(nd)).second) return -5;
  }
  for (int64_t r = 0; r < n; ++r) {
    int j;
    int32_t k[3];
    key_coords(dim, keys[r], &j, k);
    while (j > 0) {
      for (int a = 0; a < dim; ++a) k[a] >>= 1;
      --j;
      uint64_t pk = make_key(dim, j, k);
      auto it = g.nodes.find(pk);
      if (it != g.nodes.end()) {
        if (it->second.leaf) return -5;  // a leaf with a descendant leaf
        break;
      }
      Node nd;
      nd.leaf = false;
      nd.u.assign(m, 0.0);
      g.nodes.emplace(pk, std::move(nd));
    }
  }
  // every internal node must have all children (leaves partition Omega)
  for (auto& kv : g.nodes) {
    if (kv.second.leaf) continue;
    int j;
    int32_t k[3];
    key_coords(dim, kv.first, &j, k);
    for (int d = 0; d < (1 << dim); ++d) {
      int32_t c[3];
      child_coords(dim, k, d, c);
      if (!g.nodes.count(make_key(dim, j + 1, c))) return -5;
    }
  }
  project_all(g);
  grid_compile(g);
  return 0;
}

int grid_adapt(Grid& g) {
  // H6.1 projection, H6.2 details + significance (pre-adaptation values)
  project_all(g);
  if (int rc = compute_significance(g)) return rc;
  for (auto& kv : g.nodes) kv.second.is_new = false;
  // H6.3 refinement R0 = {leaf n : level < J, D(n) > eps_level} (strict), then grading
  std::vector<uint64_t> r0;
  for (auto& kv : g.nodes) {
    if (!kv.second.leaf) continue;
    int j = key_level(kv.first);
    if (j < g.lmax && kv.second.Q > threshold_sq(g, j)) r0.push_back(kv.first);
  }
  for (uint64_t key : r0) refine_leaf(g, key);
  grade_fixed_point(g);
  // H6.4 new-node values by prediction, increasing level order
  for (int j = 1; j <= g.lmax; ++j) {
    std::vector<uint64_t> nk;
    for (auto& kv : g.nodes)
      if (kv.second.is_new && key_level(kv.first) == j) nk.push_back(kv.first);
    std::sort(nk.begin(), nk.end());
    std::vector<std::vector<double>> vals(nk.size(), std::vector<double>(g.m));
    for (size_t r = 0; r < nk.size(); ++r) {
      int32_t k[3];
      int jj;
      key_coords(g.dim, nk[r], &jj, k);
      if (!predict_node(g, j, k, g.m, vals[r].data())) return -5;
    }
    for (size_t r = 0; r < nk.size(); ++r) g.nodes.at(nk[r]).u = vals[r];
  }
  // H6.5 coarsening fixed point (nodes created in this call excluded)
  coarsen_fixed_point(g);
  for (auto& kv : g.nodes) kv.second.is_new = false;
  grid_compile(g);
  return grid_check_graded(g);
}

int grid_check_graded(const Grid& g) {
  for (auto& kv : g.nodes) {
    int j;
    int32_t k[3];
    key_coords(g.dim, kv.first, &j, k);
    if (kv.second.leaf) {
      if (j < g.lmin) return -5;
      continue;
    }
    for (int d = 0; d < (1 << g.dim); ++d) {
      int32_t c[3];
      child_coords(g.dim, k, d, c);
      if (!g.nodes.count(make_key(g.dim, j + 1, c))) return -5;
    }
    int32_t q[3] = {0, 0, 0};
    const int R = kGradeRadius;
    const int32_t zlo = g.dim == 3 ? k[2] - R : 0, zhi = g.dim == 3 ? k[2] + R : 0;
    for (q[2] = zlo; q[2] <= zhi; ++q[2])
      for (q[1] = k[1] - R; q[1] <= k[1] + R; ++q[1])
        for (q[0] = k[0] - R; q[0] <= k[0] + R; ++q[0])
          if (inside(g.dim, j, q) && !g.nodes.count(make_key(g.dim, j, q))) return -5;
  }
  return 0;
}

// ============================================================== FV operator (O.5)
void grid_compile(Grid& g) {
  g.leaf_keys = sorted_keys(g, true);
  g.int_keys.clear();
  for (auto& kv : g.nodes)
    if (!kv.second.leaf && key_level(kv.first) >= g.lmin) g.int_keys.push_back(kv.first);
  std::sort(g.int_keys.begin(), g.int_keys.end());
  const int64_t nl = int64_t(g.leaf_keys.size()), ni = int64_t(g.int_keys.size());
  std::unordered_map<uint64_t, int64_t> vidx;
  vidx.reserve(size_t(nl + ni) * 2);
  for (int64_t r = 0; r < nl; ++r) vidx[g.leaf_keys[r]] = r;
  for (int64_t r = 0; r < ni; ++r) vidx[g.int_keys[r]] = nl + r;
  const int nc = 1 << g.dim;
  // projection program: internal nodes, decreasing level
  std::vector<int64_t> order(ni);
  for (int64_t r = 0; r < ni; ++r) order[r] = r;
  std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
    return key_level(g.int_keys[a]) > key_level(g.int_keys[b]);
  });
  g.proj_order.assign(ni, 0);
  g.proj_children.assign(ni * nc, 0);
  for (int64_t r = 0; r < ni; ++r) {
    const uint64_t key = g.int_keys[order[r]];
    g.proj_order[r] = nl + order[r];
    int j;
    int32_t k[3];
    key_coords(g.dim, key, &j, k);
    for (int d = 0; d < nc; ++d) {
      int32_t c[3];
      child_coords(g.dim, k, d, c);
      g.proj_children[r * nc + d] = vidx.at(make_key(g.dim, j + 1, c));
    }
  }
  // rows
  g.row_start.assign(nl + 1, 0);
  g.terms.clear();
  g.sten_pool.clear();
  const double gw = 1.0 + (g.dim == 2 ? 1.5625 : 1.953125);  // 1 + (5/4)^d
  double rho = 0.0;
  auto push_sten = [&](int level, const int32_t* kk) -> int64_t {
    uint64_t sk[27];
    const int ns = stencil_keys(g.dim, level, kk, sk);
    const int64_t off = int64_t(g.sten_pool.size());
    for (int s = 0; s < ns; ++s) g.sten_pool.push_back(vidx.at(sk[s]));  // present by grading
    return off;
  };
  for (int64_t r = 0; r < nl; ++r) {
    g.row_start[r] = int64_t(g.terms.size());
    int j;
    int32_t k[3];
    key_coords(g.dim, g.leaf_keys[r], &j, k);
    const double cj = std::ldexp(1.0, 2 * j);  // 1/h_j^2
    double rowsum = 0.0;
    int64_t c_sten = -1;
    for (int a = 0; a < g.dim; ++a)
      for (int dir = -1; dir <= 1; dir += 2) {
        int32_t nb[3] = {k[0], k[1], k[2]};
        nb[a] += dir;
        if (!inside(g.dim, j, nb)) continue;  // F3: homogeneous Neumann, zero flux
        auto it = g.nodes.find(make_key(g.dim, j, nb));
        if (it != g.nodes.end() && it->second.leaf) {  // F2
          Term t{0, vidx.at(it->first), -1, {0, 0, 0}, cj};
          g.terms.push_back(t);
          rowsum += 2.0 * cj;
        } else if (g.op_mode == OP_TWO_POINT) {
          // reading R-T: flux (u_N - u_C) |face| / |x_N - x_C| across the face, the distance between
          // the centres of a level-j and a level-(j+1) cell being 1.5 h_{j+1} along the normal; divided
          // by |C|.  Toward a coarser leaf L: |face| = h_j^{d-1}, distance 1.5 h_j -> coef cj / 1.5.
          // Toward finer leaves F: |face| = h_{j+1}^{d-1} each, distance 1.5 h_{j+1}, |C| = 2^d h_{j+1}^d
          // -> coef 4^{j+1} / (1.5 2^d) per F.  Conservative: |C| coef_CF = |F| coef_FC.
          if (it != g.nodes.end()) {
            const double cff = std::ldexp(1.0, 2 * (j + 1) - g.dim) / 1.5;
            for (int d = 0; d < nc; ++d) {
              int32_t f[3];
              child_coords(g.dim, nb, d, f);
              if (f[a] != (dir > 0 ? 2 * nb[a] : 2 * nb[a] + 1)) continue;
              Term t{0, vidx.at(make_key(g.dim, j + 1, f)), -1, {0, 0, 0}, cff};
              g.terms.push_back(t);
              rowsum += 2.0 * cff;
            }
          } else {
            int32_t L[3];
            for (int x = 0; x < g.dim; ++x) L[x] = nb[x] >> 1;
            const double ccj = cj / 1.5;
            Term t{0, vidx.at(make_key(g.dim, j - 1, L)), -1, {0, 0, 0}, ccj};
            g.terms.push_back(t);
            rowsum += 2.0 * ccj;
          }
        } else if (it != g.nodes.end()) {  // F5: neighbour refined
          if (c_sten < 0) c_sten = push_sten(j, k);
          const double cf = std::ldexp(1.0, 2 * (j + 1) - g.dim);
          for (int d = 0; d < nc; ++d) {
            int32_t f[3];
            child_coords(g.dim, nb, d, f);
            if (f[a] != (dir > 0 ? 2 * nb[a] : 2 * nb[a] + 1)) continue;
            int32_t cc[3] = {f[0], f[1], f[2]};
            cc[a] -= dir;  // the child of C adjacent to F
            Term t{2, vidx.at(make_key(g.dim, j + 1, f)), c_sten, {cc[0] & 1, cc[1] & 1, cc[2] & 1}, cf};
            g.terms.push_back(t);
            rowsum += gw * cf;
          }
        } else {  // F4: neighbour covered by the coarser leaf L = parent(nb)
          int32_t L[3];
          for (int x = 0; x < g.dim; ++x) L[x] = nb[x] >> 1;
          const int64_t off = push_sten(j - 1, L);
          Term t{1, -1, off, {nb[0] & 1, nb[1] & 1, nb[2] & 1}, cj};
          g.terms.push_back(t);
          rowsum += gw * cj;
        }
      }
    rho = std::max(rho, rowsum);
  }
  g.row_start[nl] = int64_t(g.terms.size());
  g.rho1 = rho;
}

void grid_apply(const Grid& g, const double* x, double* y, std::vector<double>& V) {
  const int64_t nl = int64_t(g.leaf_keys.size()), ni = int64_t(g.int_keys.size());
  const int nc = 1 << g.dim;
  V.resize(nl + ni);
  for (int64_t r = 0; r < nl; ++r) V[r] = x[r];
  const double scale = std::ldexp(1.0, -g.dim);
  for (int64_t r = 0; r < ni; ++r) {  // F6: internal value = projection of the current vector
    const int64_t* ch = &g.proj_children[r * nc];
    double s = V[ch[0]];
    for (int d = 1; d < nc; ++d) s = s + V[ch[d]];
    V[g.proj_order[r]] = s * scale;
  }
  const int ns = pow3(g.dim);
  double v[27];
  for (int64_t r = 0; r < nl; ++r) {
    double acc = 0.0;
    for (int64_t t = g.row_start[r]; t < g.row_start[r + 1]; ++t) {
      const Term& T = g.terms[t];
      if (T.type == 0) {
        acc += (V[T.idx] - V[r]) * T.coef;
      } else {
        for (int s = 0; s < ns; ++s) v[s] = V[g.sten_pool[T.sten + s]];
        const double gh = predict_vals(g.dim, v, T.cbits);
        if (T.type == 1) acc += (gh - V[r]) * T.coef;
        else acc += (V[T.idx] - gh) * T.coef;
      }
    }
    y[r] = acc;
  }
}

// ============================================================== Rock4 (O.4)
bool rock4_load(const char* path) {
  std::ifstream f(path);
  if (!f) return false;
  g_table.clear();
  std::string line;
  std::vector<std::string> lines;
  while (std::getline(f, line))
    if (!line.empty() && line[0] != '#') lines.push_back(line);
  size_t i = 0;
  while (i < lines.size()) {
    std::istringstream hs(lines[i]);
    Rock4Coeffs c;
    hs >> c.s >> c.ell >> c.sigma[0] >> c.sigma[1] >> c.sigma[2] >> c.sigma[3];
    if (!hs || c.s < 5 || i + 1 + size_t(c.s - 4) > lines.size()) break;  // truncated table
    for (int k = 0; k < c.s - 4; ++k) {
      std::istringstream rs(lines[i + 1 + k]);
      double a, b, d;
      rs >> a >> b >> d;
      c.mu.push_back(a); c.nu.push_back(b); c.kappa.push_back(d);
    }
    i += 1 + (c.s - 4);
    g_table.push_back(c);
  }
  return !g_table.empty() && g_table[0].s == 5;
}

const Rock4Coeffs* rock4_get(int s) {
  if (s < 5 || s - 5 >= int(g_table.size())) return nullptr;
  return &g_table[s - 5];
}

int rock4_smax() { return g_table.empty() ? 0 : g_table.back().s; }

namespace {
// y = (h eps) A x
void hA(const Grid& g, double he, const double* x, double* y, std::vector<double>& V, int64_t* mv) {
  grid_apply(g, x, y, V);
  const int64_t n = int64_t(g.leaf_keys.size());
  for (int64_t r = 0; r < n; ++r) y[r] = he * y[r];
  ++*mv;
}

// One Rock4 step of size h with s stages (K3) and its error vector (K4).
void rock4_step(const Grid& g, const double* x, double he, const Rock4Coeffs& C, double* xn,
                double* e, std::vector<double>& V, int64_t* mv) {
  const int64_t n = int64_t(g.leaf_keys.size());
  std::vector<double> gp(x, x + n), gc(x, x + n), gn(n), Ag(n), v(n), Av(n);
  // recurrence stages (H3.2): g_{k+1} = mu_k hA g_k + nu_k g_k + kappa_k g_{k-1}
  for (int k = 0; k < C.s - 4; ++k) {
    hA(g, he, gc.data(), Ag.data(), V, mv);
    for (int64_t r = 0; r < n; ++r) gn[r] = C.mu[k] * Ag[r] + C.nu[k] * gc[r] + C.kappa[k] * gp[r];
    gp.swap(gc);
    gc.swap(gn);
  }
  // finishing by Horner (H3.3): x_{n+1} = w(hA) y, w = 1 + s1 z + s2 z^2 + s3 z^3 + s4 z^4
  const double* y = gc.data();
  for (int64_t r = 0; r < n; ++r) v[r] = C.sigma[3] * y[r];
  for (int q = 2; q >= 0; --q) {
    hA(g, he, v.data(), Av.data(), V, mv);
    for (int64_t r = 0; r < n; ++r) v[r] = C.sigma[q] * y[r] + Av[r];
  }
  hA(g, he, v.data(), Av.data(), V, mv);
  for (int64_t r = 0; r < n; ++r) xn[r] = y[r] + Av[r];
  // K4: e = sigma4 (hA)^4 y
  std::vector<double> w(y, y + n);
  for (int q = 0; q < 4; ++q) {
    hA(g, he, w.data(), Av.data(), V, mv);
    w.swap(Av);
  }
  for (int64_t r = 0; r < n; ++r) e[r] = C.sigma[3] * w[r];
}
}  // namespace

int rock4_forced_step(const Grid& g, const double* x, double eps_i, double h, int s, double* out,
                      double* err_vec) {
  const Rock4Coeffs* C = rock4_get(s);
  if (!C) return -1;
  std::vector<double> V, e(g.leaf_keys.size());
  int64_t mv = 0;
  rock4_step(g, x, h * eps_i, *C, out, err_vec ? err_vec : e.data(), V, &mv);
  return 0;
}

int rock4_integrate(const Grid& g, double* x, double eps_i, double T, double rtol, double atol,
                    int s_max, Rock4Stats* st, double* hprop) {
  const int64_t n = int64_t(g.leaf_keys.size());
  const int smax = std::min(s_max, rock4_smax());
  const Rock4Coeffs* Cmax = rock4_get(smax);
  if (!Cmax || T <= 0.0) return -1;
  const double rho = eps_i * g.rho1;
  std::vector<double> xn(n), e(n), V;
  Rock4Stats s;
  double t = 0.0, h = T;
  if (hprop && *hprop > 0.0 && *hprop < T) h = *hprop;  // R-K5b: the previous substep's proposal
  double hwant = h;
  bool reject_prev = false;
  while (true) {
    bool last = false;
    if (h * rho > Cmax->ell) h = Cmax->ell / rho;
    hwant = h;
    if (t + h >= T) { h = T - t; last = true; }
    int sc = 5;  // K3: s = min{s >= 5 : ell_s >= h rho}
    while (sc < smax && rock4_get(sc)->ell < h * rho) ++sc;
    const Rock4Coeffs& C = *rock4_get(sc);
    rock4_step(g, x, h * eps_i, C, xn.data(), e.data(), V, &s.matvecs);
    double acc = 0.0;  // K4: err = RMS(e / sc)
    for (int64_t r = 0; r < n; ++r) {
      const double scr = atol + rtol * std::max(std::fabs(x[r]), std::fabs(xn[r]));
      const double q = e[r] / scr;
      acc += q * q;
    }
    const double err = std::sqrt(acc / double(n));
    const double fac = err > 0.0 ? std::min(5.0, std::max(0.1, 0.8 / std::sqrt(std::sqrt(err)))) : 5.0;
    s.s_min = s.s_min ? std::min(s.s_min, sc) : sc;
    s.s_max = std::max(s.s_max, sc);
    if (err <= 1.0) {  // K5 accept
      for (int64_t r = 0; r < n; ++r) x[r] = xn[r];
      s.steps++;
      if (last) break;
      t += h;
      double hnew = h * fac;
      if (reject_prev) hnew = std::min(hnew, h);
      reject_prev = false;
      h = hnew;
    } else {
      s.rejects++;
      reject_prev = true;
      h = h * fac;
      if (s.rejects > 100000) return -4;
    }
  }
  if (st) {
    st->steps += s.steps; st->rejects += s.rejects; st->matvecs += s.matvecs;
    st->s_min = st->s_min ? std::min(st->s_min, s.s_min) : s.s_min;
    st->s_max = std::max(st->s_max, s.s_max);
  }
  if (hprop) *hprop = hwant;
  return 0;
}

// ============================================================== reaction / diffusion / Strang
namespace {
template <class F>
void parallel_for(int64_t n, int nthreads, F fn) {
  if (nthreads <= 1 || n < 2) {
    for (int64_t i = 0; i < n; ++i) fn(i, 0);
    return;
  }
  std::atomic<int64_t> next(0);
  std::vector<std::thread> th;
  for (int w = 0; w < nthreads; ++w)
    th.emplace_back([&, w]() {
      while (true) {
        int64_t b = next.fetch_add(64);
        if (b >= n) break;
        for (int64_t i = b; i < std::min(n, b + 64); ++i) fn(i, w);
      }
    });
  for (auto& t : th) t.join();
}
}  // namespace

int grid_react(Grid& g, const Model& M, double T, const R5Opts& o, int nthreads, R5Counters* total,
               int64_t* n_failed) {
  const int64_t n = int64_t(g.leaf_keys.size());
  std::vector<Node*> np(n);
  for (int64_t r = 0; r < n; ++r) np[r] = &g.nodes.at(g.leaf_keys[r]);
  std::vector<R5Counters> cs(n);
  std::vector<int> stv(n);
  parallel_for(n, nthreads, [&](int64_t r, int) { stv[r] = radau5_cell(M, np[r]->u.data(), T, o, &cs[r]); });
  int64_t nf = 0;
  for (int64_t r = 0; r < n; ++r) {
    if (stv[r]) ++nf;
    if (total) {
      total->n_attempt += cs[r].n_attempt; total->n_accept += cs[r].n_accept;
      total->n_reject += cs[r].n_reject; total->n_f += cs[r].n_f; total->n_jac += cs[r].n_jac;
      total->n_lu += cs[r].n_lu; total->n_newton += cs[r].n_newton;
    }
  }
  if (n_failed) *n_failed += nf;
  return nf ? -4 : 0;
}

int grid_diffuse(Grid& g, const double* eps_diff, double T, double rtol, double atol, int s_max,
                 int nthreads, Rock4Stats* st) {
  const int64_t n = int64_t(g.leaf_keys.size());
  std::vector<Node*> np(n);
  for (int64_t r = 0; r < n; ++r) np[r] = &g.nodes.at(g.leaf_keys[r]);
  std::vector<Rock4Stats> ss(g.m);
  std::vector<int> rc(g.m, 0);
  if (int(g.r4_hprop.size()) != g.m) g.r4_hprop.assign(g.m, 0.0);
  parallel_for(g.m, std::min(nthreads, g.m), [&](int64_t i, int) {
    if (eps_diff[i] == 0.0) return;  // D with eps = 0 is the identity
    std::vector<double> x(n);
    for (int64_t r = 0; r < n; ++r) x[r] = np[r]->u[i];
    rc[i] = rock4_integrate(g, x.data(), eps_diff[i], T, rtol, atol, s_max, &ss[i], &g.r4_hprop[i]);
    for (int64_t r = 0; r < n; ++r) np[r]->u[i] = x[r];
  });
  for (int i = 0; i < g.m; ++i) {
    if (st) {
      st->steps += ss[i].steps; st->rejects += ss[i].rejects; st->matvecs += ss[i].matvecs;
      if (ss[i].s_min) st->s_min = st->s_min ? std::min(st->s_min, ss[i].s_min) : ss[i].s_min;
      st->s_max = std::max(st->s_max, ss[i].s_max);
    }
    if (rc[i]) return rc[i];
  }
  return 0;
}

void grid_react_rk4(Grid& g, const Model& M, double T, int nsteps, int nthreads) {
  const int64_t n = int64_t(g.leaf_keys.size());
  std::vector<Node*> np(n);
  for (int64_t r = 0; r < n; ++r) np[r] = &g.nodes.at(g.leaf_keys[r]);
  parallel_for(n, nthreads, [&](int64_t r, int) { rk4_cell(M, np[r]->u.data(), T, nsteps); });
}

int strang_step(Grid& g, const Model& M, const double* eps_diff, double dt, int scheme,
                const R5Opts& ro, double krtol, double katol, int ks_max, int nthreads,
                R5Counters* rc, Rock4Stats* ks, int64_t* n_failed) {
  int r1 = 0, r2 = 0, r3 = 0;
  const bool rk4 = (scheme & STRANG_RK4) != 0;  // reaction by RK4, h_max = ro.h0 (reading R-K4)
  auto react = [&](double T) -> int {
    if (!rk4) return grid_react(g, M, T, ro, nthreads, rc, n_failed);
    const int ns = ro.h0 > 0.0 ? int(std::ceil(T / ro.h0)) : 1;
    grid_react_rk4(g, M, T, ns, nthreads);
    return 0;
  };
  if ((scheme & 0xff) == STRANG_RDR) {  // U_{n+1} = R_{dt/2} D_dt R_{dt/2} U_n
    r1 = react(0.5 * dt);
    r2 = grid_diffuse(g, eps_diff, dt, krtol, katol, ks_max, nthreads, ks);
    r3 = react(0.5 * dt);
  } else {  // D_{dt/2} R_dt D_{dt/2}
    r1 = grid_diffuse(g, eps_diff, 0.5 * dt, krtol, katol, ks_max, nthreads, ks);
    r2 = react(dt);
    r3 = grid_diffuse(g, eps_diff, 0.5 * dt, krtol, katol, ks_max, nthreads, ks);
  }
  if (r1) return r1;
  if (r2) return r2;
  return r3;
}

}  // namespace orc
