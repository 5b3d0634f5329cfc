// Offline generator of the Rock4 coefficient family compiled into the product
// (paper_1506_04651_b200/csrc/rock4_coeffs.inc).  Independent of oracle/ (different code,
// different algorithms: long double, Lanczos instead of Stieltjes, a different exact quadrature
// size, peak-refined instead of plain sampled stability test); tests compare the two tables.
//
// PAPER.md P:957-975 (§5.3): Rock4 = a three-term recurrence of orthogonal polynomials whose
// length follows the spectral radius, composed with a 4-stage finishing procedure; for
// linear problems the finishing step is the polynomial w (with complex roots) applied by Horner.
// The ROCK4 tables of the cited paper are not in PAPER.md; reading R-K1 (SURVEY §8(c)
// O.4 K1) defines the family regenerated here:
//   n = s - 4; on z in [-l, 0], x = 1 + 2z/l, P_n orthogonal for w(z)^2 / sqrt(1 - x^2) with
//   P_n(0) = 1; w = 1 + s1 z + s2 z^2 + s3 z^3 + s4 z^4 fixed by R = w P_n = e^z + O(z^5);
//   P_n <-> sigma iterated to a fixed point; l_s = largest l with a converged fixed point and
//   max_{[-l,0)} |R| <= 1.
// Stage form (monic pi_{k+1} = (x - a_k) pi_k - b_k pi_{k-1}):
//   mu_k = (2/l) pi_k(1)/pi_{k+1}(1), nu_k = (1-a_k) pi_k(1)/pi_{k+1}(1),
//   kappa_k = -b_k pi_{k-1}(1)/pi_{k+1}(1);  g_{k+1} = mu_k hA g_k + nu_k g_k + kappa_k g_{k-1}.
//
// Build & run:  g++ -O2 -std=c++17 -pthread gen_rock4.cpp -o /tmp/gen_rock4 && /tmp/gen_rock4 200 > rock4_coeffs.inc
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <thread>
#include <vector>

typedef long double R;

struct Family {
  int s = 0;
  R ell = 0, sig[4] = {0, 0, 0, 0};
  std::vector<R> mu, nu, ka;
};

// Lanczos on diag(x) with start vector sqrt(weights): Jacobi matrix (alpha_k, beta_k);
// monic recurrence a_k = alpha_k, b_k = beta_{k-1}^2.  Full reorthogonalisation.
static void lanczos(const std::vector<R>& x, const std::vector<R>& wt, int n, std::vector<R>& a,
                    std::vector<R>& b) {
  const int N = int(x.size());
  std::vector<std::vector<R>> Q;
  std::vector<R> q(N), v(N);
  R nrm = 0;
  for (int i = 0; i < N; ++i) { q[i] = std::sqrt(wt[i]); nrm += wt[i]; }
  nrm = std::sqrt(nrm);
  for (int i = 0; i < N; ++i) q[i] /= nrm;
  a.assign(n, 0); b.assign(n, 0);
  R beta_prev = 0;
  std::vector<R> qprev(N, 0);
  for (int k = 0; k < n; ++k) {
    Q.push_back(q);
    R al = 0;
    for (int i = 0; i < N; ++i) al += q[i] * x[i] * q[i];
    a[k] = al;
    b[k] = k > 0 ? beta_prev * beta_prev : 0;
    for (int i = 0; i < N; ++i) v[i] = (x[i] - al) * q[i] - beta_prev * qprev[i];
    for (int pass = 0; pass < 1; ++pass)
      for (auto& u : Q) {
        R d = 0;
        for (int i = 0; i < N; ++i) d += u[i] * v[i];
        for (int i = 0; i < N; ++i) v[i] -= d * u[i];
      }
    R bt = 0;
    for (int i = 0; i < N; ++i) bt += v[i] * v[i];
    bt = std::sqrt(bt);
    qprev = q;
    for (int i = 0; i < N; ++i) q[i] = v[i] / bt;
    beta_prev = bt;
  }
}

static R wpoly(const R* s, R z) { return 1 + z * (s[0] + z * (s[1] + z * (s[2] + z * s[3]))); }

// Recurrence + Taylor coefficients (to z^4) of P_n for a given sigma; returns false on breakdown.
static bool recurrence(int s, R ell, const R* sig, Family& F, R* p) {
  const int n = s - 4;
  const int N = 3 * s + 64;  // Gauss-Chebyshev with N nodes is exact to degree 2N-1 >= 2n+8
  std::vector<R> x(N), wt(N);
  const R pi = std::acos(R(-1));
  for (int i = 0; i < N; ++i) {
    x[i] = std::cos((2 * i + 1) * pi / (2 * N));
    const R z = (x[i] - 1) * ell / 2;
    const R w = wpoly(sig, z);
    wt[i] = w * w;
  }
  std::vector<R> a, b;
  lanczos(x, wt, n, a, b);
  std::vector<R> pi1(n + 2, 0);  // pi1[k+1] = pi_k(1)
  pi1[1] = 1;
  for (int k = 0; k < n; ++k) pi1[k + 2] = (1 - a[k]) * pi1[k + 1] - b[k] * pi1[k];
  F.mu.assign(n, 0); F.nu.assign(n, 0); F.ka.assign(n, 0);
  for (int k = 0; k < n; ++k) {
    if (!(std::fabs(pi1[k + 2]) > 0) || !std::isfinite(pi1[k + 2])) return false;
    F.mu[k] = (2 / ell) * pi1[k + 1] / pi1[k + 2];
    F.nu[k] = (1 - a[k]) * pi1[k + 1] / pi1[k + 2];
    F.ka[k] = -b[k] * pi1[k] / pi1[k + 2];
  }
  R P[5] = {1, 0, 0, 0, 0}, Pm[5] = {0, 0, 0, 0, 0};
  for (int k = 0; k < n; ++k) {
    R Pn[5];
    for (int q = 0; q < 5; ++q)
      Pn[q] = F.nu[k] * P[q] + (q ? F.mu[k] * P[q - 1] : 0) + F.ka[k] * Pm[q];
    for (int q = 0; q < 5; ++q) { Pm[q] = P[q]; P[q] = Pn[q]; }
  }
  for (int q = 0; q < 5; ++q) p[q] = P[q];
  return true;
}

// Fixed point P_n <-> sigma (damped 1/2) from sig (in/out).
static bool fixed_point(int s, R ell, R* sig, Family& F) {
  for (int it = 0; it < 4000; ++it) {
    R p[5];
    if (!recurrence(s, ell, sig, F, p)) return false;
    R t[4];
    t[0] = 1 - p[1];
    t[1] = R(1) / 2 - t[0] * p[1] - p[2];
    t[2] = R(1) / 6 - t[1] * p[1] - t[0] * p[2] - p[3];
    t[3] = R(1) / 24 - t[2] * p[1] - t[1] * p[2] - t[0] * p[3] - p[4];
    R delta = 0;
    for (int q = 0; q < 4; ++q) {
      const R nx = (sig[q] + t[q]) / 2;
      if (!std::isfinite(nx)) return false;
      delta = std::fmax(delta, std::fabs(nx - sig[q]) / std::fmax(std::fabs(nx), R(1e-300)));
      sig[q] = nx;
    }
    if (delta < R(1e-16)) {
      R p2[5];
      return recurrence(s, ell, sig, F, p2);
    }
  }
  return false;
}

static R Rabs(const Family& F, const R* sig, R z) {
  R Pm = 0, P = 1;
  for (size_t k = 0; k < F.mu.size(); ++k) {
    const R Pn = (F.nu[k] + F.mu[k] * z) * P + F.ka[k] * Pm;
    Pm = P; P = Pn;
  }
  return std::fabs(wpoly(sig, z) * P);
}

// max |R| over samples z[0..M] (z[0] = 0 excluded), with golden-section refinement around every
// sampled local maximum.
static R max_abs_R_on(const Family& F, const R* sig, R zlo, int M) {
  std::vector<R> z(M + 1), v(M + 1);
  for (int i = 0; i <= M; ++i) { z[i] = zlo * R(i) / M; v[i] = Rabs(F, sig, z[i]); }
  R best = 0;
  for (int i = 1; i <= M; ++i) {  // i = 0 is z = 0 (R(0) = 1 exactly): excluded
    best = std::fmax(best, v[i]);
    const bool peak = (i < M) && v[i] >= v[i - 1] && v[i] >= v[i + 1];
    if (!peak) continue;
    R lo = z[i + 1], hi = z[i - 1];
    const R g = (std::sqrt(R(5)) - 1) / 2;
    R c = hi - g * (hi - lo), d = lo + g * (hi - lo);
    R fc = Rabs(F, sig, c), fd = Rabs(F, sig, d);
    for (int k = 0; k < 60; ++k) {
      if (fc > fd) { lo = d; d = c; fd = fc; c = hi - g * (hi - lo); fc = Rabs(F, sig, c); }
      else { hi = c; c = d; fc = fd; d = lo + g * (hi - lo); fd = Rabs(F, sig, d); }
    }
    if (hi < 0) best = std::fmax(best, std::fmax(fc, fd));
  }
  return best;
}

// max |R| on [-l, 0): the whole interval at ~60 samples per oscillation, plus [-min(l, 24), 0]
// densely, where the interior peak of |R| (the complex roots of w, z ~ -8) decides l_s.
static R max_abs_R(const Family& F, const R* sig, R ell) {
  const int n = int(F.mu.size());
  const R a = max_abs_R_on(F, sig, -ell, std::max(12000, 60 * (n + 4)));
  const R b = max_abs_R_on(F, sig, -std::fmin(ell, R(24)), 24000);
  return std::fmax(a, b);
}

static bool stable(int s, R ell, R* sig, Family& F) {
  if (!fixed_point(s, ell, sig, F)) return false;
  return max_abs_R(F, sig, ell) <= 1;
}

static Family make(int s) {
  Family F;
  F.s = s;
  R lo = (s < 7 ? R(0.2) : (s < 12 ? R(0.25) : R(0.28))) * s * s, hi = R(0.40) * s * s;
  R sig_lo[4] = {0, 0, 0, 0};
  if (!stable(s, lo, sig_lo, F)) { std::fprintf(stderr, "s=%d: lower bracket unstable\n", s); std::exit(1); }
  {
    R sg[4] = {sig_lo[0], sig_lo[1], sig_lo[2], sig_lo[3]};
    Family G;
    if (stable(s, hi, sg, G)) { std::fprintf(stderr, "s=%d: upper bracket stable\n", s); std::exit(1); }
  }
  for (int it = 0; it < 80 && hi - lo > R(1e-11) * hi; ++it) {
    const R mid = (lo + hi) / 2;
    R sg[4] = {sig_lo[0], sig_lo[1], sig_lo[2], sig_lo[3]};
    Family G;
    if (stable(s, mid, sg, G)) { lo = mid; for (int q = 0; q < 4; ++q) sig_lo[q] = sg[q]; }
    else hi = mid;
  }
  F.ell = lo;
  for (int q = 0; q < 4; ++q) F.sig[q] = sig_lo[q];
  R p[5];
  fixed_point(s, lo, F.sig, F);
  recurrence(s, lo, F.sig, F, p);
  return F;
}

int main(int argc, char** argv) {
  const int smax = argc > 1 ? std::atoi(argv[1]) : 200;
  const int ns = smax - 4;
  std::vector<Family> tab(ns);
  std::atomic<int> next(0);
  std::vector<std::thread> th;
  const int nt = std::max(1, int(std::thread::hardware_concurrency()) - 2);
  for (int w = 0; w < nt; ++w)
    th.emplace_back([&]() {
      for (int i; (i = next.fetch_add(1)) < ns;) {
        // largest s first (they take longest)
        const int s = smax - i;
        tab[s - 5] = make(s);
        std::fprintf(stderr, "s=%d ell=%.10Lg\n", s, tab[s - 5].ell);
      }
    });
  for (auto& t : th) t.join();
  std::printf("// GENERATED by paper_1506_04651_b200/tools/gen_rock4.cpp %d — do not edit.\n", smax);
  std::printf("// Rock4 family (DESIGN.md R-K1, PAPER.md P:957-997): per s = 5..%d: ell_s, sigma_1..4,\n", smax);
  std::printf("// then s-4 triples (mu_k, nu_k, kappa_k) at offset kRock4Off[s-5].\n");
  std::printf("#define RD_ROCK4_SMAX %d\n", smax);
  std::printf("static const double kRock4Ell[%d] = {\n", ns);
  for (auto& F : tab) std::printf("  %.17Lg,\n", F.ell);
  std::printf("};\nstatic const double kRock4Sig[%d][4] = {\n", ns);
  for (auto& F : tab) std::printf("  {%.17Lg, %.17Lg, %.17Lg, %.17Lg},\n", F.sig[0], F.sig[1], F.sig[2], F.sig[3]);
  std::printf("};\nstatic const int kRock4Off[%d] = {", ns + 1);
  int off = 0;
  for (int i = 0; i <= ns; ++i) {
    std::printf("%s%d", i ? ", " : "", off);
    if (i < ns) off += tab[i].s - 4;
  }
  std::printf("};\nstatic const double kRock4Rec[%d][3] = {\n", off);
  for (auto& F : tab)
    for (int k = 0; k < F.s - 4; ++k) std::printf("  {%.17Lg, %.17Lg, %.17Lg},\n", F.mu[k], F.nu[k], F.ka[k]);
  std::printf("};\n");
  return 0;
}
