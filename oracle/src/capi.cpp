// ORACLE — test infrastructure only (see oracle.hpp).  Plain C entry points for
// ctypes (oracle/__init__.py).  Host arrays only.
#include <cstring>
#include <thread>

#include "oracle.hpp"

using namespace orc;

extern "C" {

typedef struct {
  int kind, m;
  double q, f_c, eps_b, mu;
  int n_reac;
  const int32_t* reactants;
  const int32_t* products;
  const double* rate;
  double k_nag;  // NAGUMO
} or_model;

typedef struct {
  double rtol, atol, h0;
  int nit;
  int64_t max_steps;
  int fixed_steps;
} or_r5opts;

static Model to_model(const or_model* om) {
  Model M;
  M.kind = om->kind;
  M.m = om->m;
  M.q = om->q; M.f_c = om->f_c; M.eps_b = om->eps_b; M.mu = om->mu;
  M.n_reac = om->n_reac;
  M.k_nag = om->k_nag;
  if (om->kind == MODEL_MASS_ACTION) {
    M.reactants.assign(om->reactants, om->reactants + 2 * om->n_reac);
    M.products.assign(om->products, om->products + 2 * om->n_reac);
    M.rate.assign(om->rate, om->rate + om->n_reac);
  }
  return M;
}

static R5Opts to_opts(const or_r5opts* o) {
  R5Opts r;
  if (o) {
    r.rtol = o->rtol; r.atol = o->atol; r.h0 = o->h0; r.nit = o->nit;
    r.max_steps = o->max_steps; r.fixed_steps = o->fixed_steps;
  }
  return r;
}

uint64_t or_key_encode(int dim, int level, const int32_t* k) { return make_key(dim, level, k); }
void or_key_decode(int dim, uint64_t key, int* level, int32_t* k) {
  *level = key_level(key);
  demorton(dim, *level, key_morton(key), k);
}

void or_model_f(const or_model* om, const double* u, double* f) { model_f(to_model(om), u, f); }
// u: [m][n] SoA (in place): RK4 with nsteps equal steps per cell
void or_rk4_batch(int64_t n, const or_model* om, double* u, double T, int nsteps, int nthreads) {
  const Model M = to_model(om);
  const int m = M.m;
  std::vector<std::thread> th;
  const int nt = nthreads < 1 ? 1 : nthreads;
  for (int t = 0; t < nt; ++t)
    th.emplace_back([&, t]() {
      std::vector<double> y(m);
      for (int64_t c = t; c < n; c += nt) {
        for (int i = 0; i < m; ++i) y[i] = u[i * n + c];
        rk4_cell(M, y.data(), T, nsteps);
        for (int i = 0; i < m; ++i) u[i * n + c] = y[i];
      }
    });
  for (auto& x : th) x.join();
}
void or_model_jac(const or_model* om, const double* u, double* J) { model_jac(to_model(om), u, J); }

// u: [m][n] SoA (in place).  counters: nullable [7][n] int64 (attempt, accept, reject, f, jac, lu, newton).
int or_radau5_batch(int64_t n, const or_model* om, double* u, double T, const or_r5opts* oo,
                    int nthreads, int64_t* counters, int32_t* status) {
  const Model M = to_model(om);
  const R5Opts o = to_opts(oo);
  const int m = M.m;
  std::vector<int> st(n, 0);
  auto work = [&](int64_t b, int64_t e) {
    std::vector<double> y(m);
    for (int64_t r = b; r < e; ++r) {
      for (int i = 0; i < m; ++i) y[i] = u[i * n + r];
      R5Counters c;
      st[r] = radau5_cell(M, y.data(), T, o, &c);
      for (int i = 0; i < m; ++i) u[i * n + r] = y[i];
      if (counters) {
        const int64_t v[7] = {c.n_attempt, c.n_accept, c.n_reject, c.n_f, c.n_jac, c.n_lu, c.n_newton};
        for (int q = 0; q < 7; ++q) counters[q * n + r] = v[q];
      }
    }
  };
  if (nthreads <= 1) {
    work(0, n);
  } else {
    std::vector<std::thread> th;
    const int64_t chunk = (n + nthreads - 1) / nthreads;
    for (int w = 0; w < nthreads; ++w) {
      const int64_t b = w * chunk, e = std::min(n, b + chunk);
      if (b < e) th.emplace_back(work, b, e);
    }
    for (auto& t : th) t.join();
  }
  int nf = 0;
  for (int64_t r = 0; r < n; ++r) {
    if (status) status[r] = st[r];
    if (st[r]) ++nf;
  }
  return nf;
}

int or_rock4_load(const char* path) { return rock4_load(path) ? rock4_smax() : -1; }
int or_rock4_get(int s, double* ell, double* sigma, double* mu, double* nu, double* kappa) {
  const Rock4Coeffs* c = rock4_get(s);
  if (!c) return -1;
  *ell = c->ell;
  for (int q = 0; q < 4; ++q) sigma[q] = c->sigma[q];
  for (int k = 0; k < s - 4; ++k) { mu[k] = c->mu[k]; nu[k] = c->nu[k]; kappa[k] = c->kappa[k]; }
  return 0;
}

void* or_grid_build(int dim, int lmin, int lmax, double eps, int m, const double* u_rowmajor, int* rc) {
  Grid* g = new Grid();
  *rc = grid_build(*g, dim, lmin, lmax, eps, m, u_rowmajor);
  return g;
}
void* or_grid_from_leaves(int dim, int lmin, int lmax, double eps, int m, int64_t n, const uint64_t* keys,
                          const double* u, int* rc) {
  Grid* g = new Grid();
  *rc = grid_from_leaves(*g, dim, lmin, lmax, eps, m, n, keys, u);
  return g;
}
void or_grid_free(void* g) { delete static_cast<Grid*>(g); }
int64_t or_grid_nleaves(void* g) { return int64_t(static_cast<Grid*>(g)->leaf_keys.size()); }
int64_t or_grid_nnodes(void* g) { return int64_t(static_cast<Grid*>(g)->nodes.size()); }
void or_grid_leaves(void* gp, uint64_t* keys, double* u) {
  Grid& g = *static_cast<Grid*>(gp);
  const int64_t n = int64_t(g.leaf_keys.size());
  for (int64_t r = 0; r < n; ++r) {
    if (keys) keys[r] = g.leaf_keys[r];
    if (u) {
      const Node& nd = g.nodes.at(g.leaf_keys[r]);
      for (int i = 0; i < g.m; ++i) u[i * n + r] = nd.u[i];
    }
  }
}
void or_grid_set_values(void* gp, const double* u) {
  Grid& g = *static_cast<Grid*>(gp);
  const int64_t n = int64_t(g.leaf_keys.size());
  for (int64_t r = 0; r < n; ++r) {
    Node& nd = g.nodes.at(g.leaf_keys[r]);
    for (int i = 0; i < g.m; ++i) nd.u[i] = u[i * n + r];
  }
}
int or_grid_adapt(void* g) { return grid_adapt(*static_cast<Grid*>(g)); }
double or_threshold_sq(int dim, int lmax, double eps, int j) { return mr_threshold_sq(dim, lmax, eps, j); }
double or_predict_vals(int dim, const double* v, const int* cb) { return mr_predict_vals(dim, v, cb); }
int or_grid_check(void* g) { return grid_check_graded(*static_cast<Grid*>(g)); }
double or_grid_rho1(void* g) { return static_cast<Grid*>(g)->rho1; }
// operator form at level jumps (OP_PREDICTION / OP_TWO_POINT); recompiles the operator
void or_grid_set_operator(void* gp, int mode) {
  Grid& g = *static_cast<Grid*>(gp);
  g.op_mode = mode;
  grid_compile(g);
}
void or_grid_apply(void* gp, const double* x, double* y) {
  std::vector<double> V;
  grid_apply(*static_cast<Grid*>(gp), x, y, V);
}
// stats: [steps, rejects, matvecs, s_min, s_max]
int or_grid_rock4_species(void* gp, double* x, double eps_i, double T, double rtol, double atol, int s_max,
                          int64_t* stats) {
  Rock4Stats st;
  int rc = rock4_integrate(*static_cast<Grid*>(gp), x, eps_i, T, rtol, atol, s_max, &st);
  if (stats) { stats[0] = st.steps; stats[1] = st.rejects; stats[2] = st.matvecs; stats[3] = st.s_min; stats[4] = st.s_max; }
  return rc;
}
int or_grid_rock4_forced(void* gp, const double* x, double eps_i, double h, int s, double* out, double* e) {
  return rock4_forced_step(*static_cast<Grid*>(gp), x, eps_i, h, s, out, e);
}
int or_grid_diffuse(void* gp, const double* eps_diff, double T, double rtol, double atol, int s_max,
                    int nthreads, int64_t* stats) {
  Rock4Stats st;
  int rc = grid_diffuse(*static_cast<Grid*>(gp), eps_diff, T, rtol, atol, s_max, nthreads, &st);
  if (stats) { stats[0] = st.steps; stats[1] = st.rejects; stats[2] = st.matvecs; stats[3] = st.s_min; stats[4] = st.s_max; }
  return rc;
}
int or_grid_react(void* gp, const or_model* om, double T, const or_r5opts* oo, int nthreads, int64_t* n_failed) {
  R5Counters c;
  int64_t nf = 0;
  int rc = grid_react(*static_cast<Grid*>(gp), to_model(om), T, to_opts(oo), nthreads, &c, &nf);
  if (n_failed) *n_failed = nf;
  return rc;
}
int or_strang_step(void* gp, const or_model* om, const double* eps_diff, double dt, int scheme,
                   const or_r5opts* oo, double krtol, double katol, int ks_max, int nthreads) {
  R5Counters c;
  Rock4Stats k;
  int64_t nf = 0;
  return strang_step(*static_cast<Grid*>(gp), to_model(om), eps_diff, dt, scheme, to_opts(oo), krtol, katol,
                     ks_max, nthreads, &c, &k, &nf);
}

}  // extern "C"
