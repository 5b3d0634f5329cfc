// ORACLE — test infrastructure only.
//
// A plain, slow, obviously-correct CPU implementation of the hot path of
// Descombes et al., "Task-based adaptive multiresolution on multi-core
// architectures" (arXiv 1506.04651; PAPER.md), written step by step from the
// paper and the readings of SURVEY.md §8(c) / DESIGN.md "Readings".  Only
// tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it.
// It shares no code with paper_1506_04651_b200/ (the product) and never calls
// it.  Scalar C++, compiled with -O2 -ffp-contract=off, no fast-math.
//
// Citations: "P:NNN" = line of PAPER.md.
#pragma once
#include <complex>
#include <cstdint>
#include <unordered_map>
#include <vector>

namespace orc {

// ---------------------------------------------------------------- keys (O.1)
// P:749-753 (§5.1): Morton abscissa by interlacing the binary digits of the
// coordinates, x_1 first.  Our key is level-major (reading C11):
// key = (level << 58) | morton_level(k).
constexpr int kLevelShift = 58;
uint64_t morton(int dim, int level, const int32_t* k);
void demorton(int dim, int level, uint64_t s, int32_t* k);
inline uint64_t make_key(int dim, int level, const int32_t* k) {
  return (uint64_t(level) << kLevelShift) | morton(dim, level, k);
}
inline int key_level(uint64_t key) { return int(key >> kLevelShift); }
inline uint64_t key_morton(uint64_t key) { return key & ((uint64_t(1) << kLevelShift) - 1); }
int level_cap(int dim);

// ---------------------------------------------------------------- models (O.2)
enum { MODEL_OREGONATOR = 1, MODEL_MASS_ACTION = 2, MODEL_NAGUMO = 3 };
struct Model {
  int kind = MODEL_OREGONATOR;
  int m = 3;
  double q = 2e-3, f_c = 1.6, eps_b = 1e-2, mu = 1e-5;  // Oregonator (BJ cfg 1)
  int n_reac = 0;
  std::vector<int32_t> reactants, products;  // [n_reac][2], -1 = none
  std::vector<double> rate;                  // [n_reac]
  double k_nag = 10.0;                       // NAGUMO f = k u^2 (1 - u), m = 1
};
void model_f(const Model& M, const double* u, double* f);
void model_jac(const Model& M, const double* u, double* J);  // row-major m x m, J[i*m+j] = df_i/du_j

// ---------------------------------------------------------------- RK4 (A10)
// Classical 4-stage explicit Runge-Kutta over [0, T] in n equal steps (reading R-K4: n = max(1,
// ceil(T / h_max)), h_max = 0 meaning one step), for non-stiff reaction terms (NAGUMO).
void rk4_cell(const Model& M, double* y, double T, int nsteps);

// ---------------------------------------------------------------- dense LU
bool lu_real(int n, std::vector<double>& A, std::vector<int>& piv);
void lu_real_solve(int n, const std::vector<double>& LU, const std::vector<int>& piv, double* b);
bool lu_cplx(int n, std::vector<std::complex<double>>& A, std::vector<int>& piv);
void lu_cplx_solve(int n, const std::vector<std::complex<double>>& LU, const std::vector<int>& piv,
                   std::complex<double>* b);

// ---------------------------------------------------------------- Radau5 (O.3)
struct R5Opts {
  double rtol = 1e-8, atol = 1e-8;  // used as given (reading C4)
  double h0 = 0.0;                  // 0 => whole interval (reading S2)
  int nit = 7;
  int64_t max_steps = 100000;
  int fixed_steps = 0;              // >0: that many equal steps, no error control (pins only)
};
enum { R5_OK = 0, R5_FAIL_STEPS = 1, R5_FAIL_SMALL_H = 2, R5_FAIL_NONFINITE = 3, R5_FAIL_NEWTON = 4 };
struct R5Counters {
  int64_t n_attempt = 0, n_accept = 0, n_reject = 0, n_f = 0, n_jac = 0, n_lu = 0, n_newton = 0;
};
int radau5_cell(const Model& M, double* y, double T, const R5Opts& o, R5Counters* cnt);

// ---------------------------------------------------------------- Rock4 table (O.4 K1)
struct Rock4Coeffs {
  int s = 0;
  double ell = 0, sigma[4] = {0, 0, 0, 0};
  std::vector<double> mu, nu, kappa;  // n = s - 4 entries
};
bool rock4_load(const char* path);
const Rock4Coeffs* rock4_get(int s);
int rock4_smax();

// ---------------------------------------------------------------- MR grid (O.6)
struct Node {
  bool leaf = true;
  bool is_new = false;
  double Q = 0.0;  // significance max_i (d_i/s_i)^2 (reading C6)
  std::vector<double> u;
};

struct Term {        // one face term of an FV row (O.5)
  int type;          // 0 same-level leaf, 1 ghost (coarser neighbour), 2 fine leaf
  int64_t idx;       // value index of the neighbour leaf (types 0, 2)
  int64_t sten;      // offset into stencil pool (types 1, 2): 3^d value indices
  int cbits[3];      // child bits of the predicted cell (types 1, 2)
  double coef;       // 1/h^2 factor (type 0, 1: 4^j; type 2: 4^(j+1) 2^-d)
};

struct Grid {
  int dim = 2, lmin = 0, lmax = 0, m = 1;
  double eps = 0.0;
  std::unordered_map<uint64_t, Node> nodes;
  // compiled operator (rebuilt after build / adapt / from_leaves)
  std::vector<uint64_t> leaf_keys;         // ascending key order
  std::vector<uint64_t> int_keys;          // internal nodes with level >= lmin, ascending
  std::vector<int64_t> proj_children;      // [n_int][2^d] value indices, aligned with proj_order
  std::vector<int64_t> proj_order;         // internal value indices, decreasing level
  std::vector<int64_t> row_start;          // [nleaf+1] into terms
  std::vector<Term> terms;
  std::vector<int64_t> sten_pool;
  double rho1 = 0.0;
  // operator at level jumps: 0 = ghost values by MR prediction (north_star, reading C3), 1 = two-point
  // fluxes between leaf centres (App. A's setting; reading R-T)
  int op_mode = 0;
  // Rock4 step size carried from one diffusion substep to the next, per species (reading R-K5b): the
  // step size the controller proposed when the previous substep ended; 0 = none yet (h0 = T)
  std::vector<double> r4_hprop;
};
enum { OP_PREDICTION = 0, OP_TWO_POINT = 1 };

int grid_build(Grid& g, int dim, int lmin, int lmax, double eps, int m, const double* u_rowmajor);
int grid_from_leaves(Grid& g, int dim, int lmin, int lmax, double eps, int m, int64_t n,
                     const uint64_t* keys, const double* u);
int grid_adapt(Grid& g);
double mr_threshold_sq(int dim, int lmax, double eps, int j);  // E_j = eps_j^2
double mr_predict_vals(int dim, const double* v /* 3^d */, const int* cb);  // Eq. inter_1d tensor
int grid_check_graded(const Grid& g);  // 0 = graded & consistent
void grid_compile(Grid& g);
void grid_apply(const Grid& g, const double* x, double* y, std::vector<double>& work);

struct Rock4Stats {
  int64_t steps = 0, rejects = 0, matvecs = 0;
  int s_min = 0, s_max = 0;
};
// hprop (nullable, in/out): in, the first step size if 0 < *hprop < T (else T); out, the step size the
// controller proposed for the step after the last one (before that step's end-of-interval clip)
int rock4_integrate(const Grid& g, double* x, double eps_i, double T, double rtol, double atol,
                    int s_max, Rock4Stats* st, double* hprop = nullptr);
int rock4_forced_step(const Grid& g, const double* x, double eps_i, double h, int s, double* out,
                      double* err_vec);

int grid_react(Grid& g, const Model& M, double T, const R5Opts& o, int nthreads,
               R5Counters* total, int64_t* n_failed);
int grid_diffuse(Grid& g, const double* eps_diff, double T, double rtol, double atol, int s_max,
                 int nthreads, Rock4Stats* st);
enum { STRANG_RDR = 0, STRANG_DRD = 1 };
// RK4 reaction substep on every leaf (n equal steps per leaf, see rk4_cell)
void grid_react_rk4(Grid& g, const Model& M, double T, int nsteps, int nthreads);
enum { STRANG_RK4 = 0x100 };  // scheme flag: reaction by RK4 (steps from R5Opts.h0) instead of Radau5
int strang_step(Grid& g, const Model& M, const double* eps_diff, double dt, int scheme,
                const R5Opts& ro, double krtol, double katol, int ks_max, int nthreads,
                R5Counters* rc, Rock4Stats* ks, int64_t* n_failed);

}  // namespace orc
