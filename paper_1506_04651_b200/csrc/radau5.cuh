// Radau5 internals shared by the thread-per-cell and warp-per-cell kernels (product side).
#pragma once
#include <cfloat>

#include "common.cuh"

namespace rdmr {

// ------------------------------------------------------------------ R1: Radau IIA constants
// c = ((4-sqrt6)/10, (4+sqrt6)/10, 1); eigenvalues of A^{-1}: gamma-hat, alpha-hat +- i beta-hat;
// T = [v_gamma | Re v_c | Im v_c] (third components 1), T^{-1}; dd = error weights.
namespace rk {
// Radau IIA constants live in the constant bank so DFMA/DMUL read them as c[] operands.  They are
// deliberately not `const`: a const initialised __constant__ double is folded into an immediate and
// re-materialised with two UMOVs on every use (8 % of the thread kernel's issue slots).
static __constant__ double c1 = 0.15505102572168219018;   // (4 - sqrt 6)/10
static __constant__ double c2 = 0.64494897427831780982;   // (4 + sqrt 6)/10
static __constant__ double gam = 3.6378342527444957322;
static __constant__ double alp = 2.6810828736277521339;
static __constant__ double bet = 3.0504301992474105694;
static __constant__ double T00 = 0.09443876248897524, T01 = -0.14125529502095421, T02 = -0.030029194105147424;
static __constant__ double T10 = 0.25021312296533331, T11 = 0.20412935229379993, T12 = 0.38294211275726194;
static __constant__ double Ti00 = 4.1787185915519047, Ti01 = 0.32768282076106239, Ti02 = 0.52337644549944955;
static __constant__ double Ti10 = -4.1787185915519047, Ti11 = -0.32768282076106239, Ti12 = 0.47662355450055045;
static __constant__ double Ti20 = -0.50287263494578688, Ti21 = 2.5719269498556054, Ti22 = -0.59603920482822492;
static __constant__ double dd1 = -10.048809399827416, dd2 = 1.3821427331607489, dd3 = -0.33333333333333333;
constexpr double uround = DBL_EPSILON;
constexpr double thet = 0.001;  // keep J when theta <= thet (R7)
constexpr float thetf = 0.001f;
constexpr double c1x = 0.15505102572168219018, c2x = 0.64494897427831780982;  // compile-time copies
}  // namespace rk

// ------------------------------------------------------------------ per-call parameters
struct R5Params {
  int64_t n;          // cells to integrate
  int64_t ld;         // species row stride of u and counters (>= every cell index + 1; = n for a full field)
  double* u;          // [m][ld]
  double T;
  double rtol, atol, h0;
  int nit;
  int64_t max_steps;
  double fnewt;       // kappa = max(10 uround / rtol, min(0.03, sqrt(rtol)))  (R5)
  int32_t* counters;  // nullable [8][ld]
  unsigned long long* work;     // atomic cell counter
  unsigned long long* totals;   // [9]: attempt, accept, reject, f, jac, lu, newton, failed, cells
  int sched;                    // thread kernel: lanes waiting for an event block before it runs
  const int32_t* order;         // nullable: cells are taken in this order (longest-first scheduling)
};

enum : int { PH_NEWCELL = 0, PH_ATTEMPT = 1, PH_NEWTON = 2, PH_ERR = 3, PH_EXIT = 4 };

// Lagrange cubic through (-1, -z3), (c1-1, z1-z3), (c2-1, z2-z3), (0, 0) evaluated at sg (R4).
__device__ __forceinline__ double extrap(double z1, double z2, double z3, double sg) {
  const double s0 = -1.0, s1 = rk::c1 - 1.0, s2 = rk::c2 - 1.0;
  // basis at the three nonzero nodes; the (0,0) node multiplies by (sg - 0)
  const double L0 = sg * (sg - s1) * (sg - s2) / (s0 * (s0 - s1) * (s0 - s2));
  const double L1 = sg * (sg - s0) * (sg - s2) / (s1 * (s1 - s0) * (s1 - s2));
  const double L2 = sg * (sg - s0) * (sg - s1) / (s2 * (s2 - s0) * (s2 - s1));
  return -z3 * L0 + (z1 - z3) * L1 + (z2 - z3) * L2;
}

rd_status launch_radau5_warp(const DevModel& md, const R5Params& P, cudaStream_t st);

}  // namespace rdmr
