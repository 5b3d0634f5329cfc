// Multiresolution grid on the B200 (readings R-B, R-A, R-G2, R-F):
// build, adapt (projection, details + significance, refinement + graded repair, prediction of
// new nodes, coarsening fixed point, compaction) and the FV operator topology with ghost stencils.
//
// Every pass is a data-parallel kernel over a dense per-level node map (see mr.cuh); the fixed
// points of graded refinement and coarsening are level-synchronous sweeps whose termination flag
// the host reads (the paper's "loop as long as ...").  The detail arithmetic
// (projection P1, prediction P2, significance P4) is FMA-free with a fixed operation order so the
// adapted leaf set is bit-identical to the oracle's (SURVEY §8(c) parity rule 3, reading S19).
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "mr.cuh"

namespace rdmr {

namespace {
constexpr int kTB = 256;

// RDMR_ADAPT_PROFILE=1: per-section wall times of mr_adapt (synchronises; stderr)
struct SecTimer {
  bool on;
  cudaStream_t st;
  std::chrono::steady_clock::time_point t0;
  explicit SecTimer(cudaStream_t s) : on(getenv("RDMR_ADAPT_PROFILE") != nullptr), st(s) {
    if (on) { cudaStreamSynchronize(st); t0 = std::chrono::steady_clock::now(); }
  }
  void mark(const char* name) {
    if (!on) return;
    cudaStreamSynchronize(st);
    const auto t1 = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[adapt] %-12s %8.1f us\n", name, std::chrono::duration<double, std::micro>(t1 - t0).count());
    t0 = t1;
  }
};
constexpr int kGradeRadius = 2;  // DESIGN.md R-G2: ghost stencils of coarse leaves must exist

inline unsigned nblk(int64_t n) { return unsigned(std::max<int64_t>(1, std::min<int64_t>((n + kTB - 1) / kTB, 1 << 20))); }

__device__ __forceinline__ int level_of(const GridDev& G, int64_t p) {
  int j = 0;
  while (p >= G.off[j + 1]) ++j;
  return j;
}
__device__ __forceinline__ int mir(int i, int n) { return i < 0 ? 0 : (i >= n ? n - 1 : i); }

template <int D>
__device__ __forceinline__ int64_t posk(const GridDev& G, int j, const int* k) {
  return G.off[j] + int64_t(morton_enc<D>(k));
}

// Eq. inter_1d, one axis: u0 + s * (u_- - u_+)/8, s = +1 for child bit 0, -1 for bit 1.
// Round-to-nearest intrinsics: no FMA contraction, fixed order (bit-exact with the oracle's P2).
__device__ __forceinline__ double step1d_rn(double um, double u0, double up, int bit) {
  double t = __dmul_rn(0.125, __dsub_rn(um, up));
  if (bit) t = -t;
  return __dadd_rn(u0, t);
}
// Tensor product, x first then y then z; v = 3^D values, x fastest.
template <int D>
__device__ __forceinline__ double predict_rn(const double* v, int cb) {
  if (D == 2) {
    double r[3];
#pragma unroll
    for (int oy = 0; oy < 3; ++oy) r[oy] = step1d_rn(v[oy * 3], v[oy * 3 + 1], v[oy * 3 + 2], cb & 1);
    return step1d_rn(r[0], r[1], r[2], (cb >> 1) & 1);
  }
  double q[3];
#pragma unroll
  for (int oz = 0; oz < 3; ++oz) {
    double r[3];
#pragma unroll
    for (int oy = 0; oy < 3; ++oy) {
      const double* w = v + (oz * 3 + oy) * 3;
      r[oy] = step1d_rn(w[0], w[1], w[2], cb & 1);
    }
    q[oz] = step1d_rn(r[0], r[1], r[2], (cb >> 1) & 1);
  }
  return step1d_rn(q[0], q[1], q[2], (cb >> 2) & 1);
}

// 3^D neighbourhood positions of (j, k) at level j, mirrored at the boundary (S10), x fastest.
template <int D>
__device__ __forceinline__ void stencil_pos(const GridDev& G, int j, const int* k, int64_t* out) {
  const int n = 1 << j;
  int c = 0;
#pragma unroll
  for (int oz = 0; oz < (D == 3 ? 3 : 1); ++oz)
#pragma unroll
    for (int oy = 0; oy < 3; ++oy)
#pragma unroll
      for (int ox = 0; ox < 3; ++ox) {
        int q[3] = {mir(k[0] + ox - 1, n), mir(k[1] + oy - 1, n), D == 3 ? mir(k[2] + oz - 1, n) : 0};
        out[c++] = posk<D>(G, j, q);
      }
}

// ------------------------------------------------------------------ kernels
__global__ void k_rowmajor_to_morton2(int J, int m, const double* src, double* dst) {
  const int64_t n1 = int64_t(1) << J, NJ = n1 * n1;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < NJ; idx += int64_t(gridDim.x) * blockDim.x) {
    int k[2] = {int(idx % n1), int(idx / n1)};
    const int64_t s = int64_t(morton_enc<2>(k));
    for (int i = 0; i < m; ++i) dst[i * NJ + s] = src[i * NJ + idx];
  }
}
__global__ void k_rowmajor_to_morton3(int J, int m, const double* src, double* dst) {
  const int64_t n1 = int64_t(1) << J, NJ = n1 * n1 * n1;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < NJ; idx += int64_t(gridDim.x) * blockDim.x) {
    int k[3] = {int(idx % n1), int((idx / n1) % n1), int(idx / (n1 * n1))};
    const int64_t s = int64_t(morton_enc<3>(k));
    for (int i = 0; i < m; ++i) dst[i * NJ + s] = src[i * NJ + idx];
  }
}

__global__ void k_scatter_leaves(GridDev G) {
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < G.N; r += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t key = G.keys[r];
    const int j = int(key >> kLevelShift);
    const int64_t p = G.off[j] + int64_t(key & ((1ull << kLevelShift) - 1));
    for (int i = 0; i < G.m; ++i) G.val[i * G.total + p] = G.u[i * G.N + r];
  }
}

// P1: parent = (((c0 + c1) + c2) + ...) * 2^-D, children in Morton child order.
template <int D>
__global__ void k_project(GridDev G, int j) {
  const int64_t nj = int64_t(1) << (D * j);
  const double scale = D == 2 ? 0.25 : 0.125;
  for (int64_t s = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; s < nj; s += int64_t(gridDim.x) * blockDim.x) {
    const int64_t p = G.off[j] + s;
    if ((G.st[p] & ST_KIND) != ST_INTERNAL) continue;
    const int64_t c = G.off[j + 1] + (s << D);
    for (int i = 0; i < G.m; ++i) {
      const double* v = G.val + i * G.total + c;
      double acc = v[0];
#pragma unroll
      for (int d = 1; d < (1 << D); ++d) acc = __dadd_rn(acc, v[d]);
      G.val[i * G.total + p] = __dmul_rn(acc, scale);
    }
  }
}

__global__ void k_fill_u64(unsigned long long* p, int n, unsigned long long v) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) p[i] = v;
}

// max_leaves |u_i| (reading C6 scale), as ordered bits of non-negative doubles.
// from_leaves: the compact leaf array G.u holds the same leaf values (adaptation): a coalesced sweep of
// N values instead of the dense map (the maximum does not depend on the order).
__global__ void k_absmax(GridDev G, unsigned long long* out, int from_leaves) {
  __shared__ double sm[kTB];
  for (int i = 0; i < G.m; ++i) {
    double mx = 0.0;
    if (from_leaves) {
      for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < G.N; r += int64_t(gridDim.x) * blockDim.x)
        mx = fmax(mx, fabs(G.u[i * G.N + r]));
    } else {
      for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < G.total; p += int64_t(gridDim.x) * blockDim.x)
        if ((G.st[p] & ST_KIND) == ST_LEAF) mx = fmax(mx, fabs(G.val[i * G.total + p]));
    }
    sm[threadIdx.x] = mx;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
      if (threadIdx.x < o) sm[threadIdx.x] = fmax(sm[threadIdx.x], sm[threadIdx.x + o]);
      __syncthreads();
    }
    if (threadIdx.x == 0) atomicMax(out + i, (unsigned long long)__double_as_longlong(sm[0]));
    __syncthreads();
  }
}

// P3 details + P4 significance Q = max_i (d_i / s_i)^2 (reading C6), nodes at level >= lo.  One
// thread per PARENT position at levels lo-1 .. J-1: the 2^D children of an internal node share its 3^D
// stencil, so the stencil is read once per species for all of them (each child's prediction keeps
// the oracle's P2 order, bit for bit).  Levels < lo get Q = 0.
template <int D>
__global__ void k_significance(GridDev G, const unsigned long long* smax_bits, int lo, int* err) {
  constexpr int NS = D == 2 ? 9 : 27;
  constexpr int NC = 1 << D;
  const int64_t gs = int64_t(gridDim.x) * blockDim.x;
  const int64_t t0 = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  for (int64_t p = t0; p < G.off[lo]; p += gs) G.Q[p] = 0.0;
  for (int64_t pp = G.off[lo - 1] + t0; pp < G.off[G.J]; pp += gs) {
    const int jp = level_of(G, pp);
    const int64_t c0 = G.off[jp + 1] + ((pp - G.off[jp]) << D);
    if ((G.st[pp] & ST_KIND) != ST_INTERNAL) {  // children absent
#pragma unroll
      for (int d = 0; d < NC; ++d) G.Q[c0 + d] = 0.0;
      continue;
    }
    int kp[3] = {0, 0, 0};
    morton_dec<D>(uint64_t(pp - G.off[jp]), kp);
    int64_t sp[NS];
    stencil_pos<D>(G, jp, kp, sp);
    bool ok = true;
#pragma unroll
    for (int q = 0; q < NS; ++q) ok = ok && (G.st[sp[q]] & ST_KIND) != ST_ABSENT;
    if (!ok) {
      atomicExch(err, 1);
#pragma unroll
      for (int d = 0; d < NC; ++d) G.Q[c0 + d] = 0.0;
      continue;
    }
    double Q[NC];
#pragma unroll
    for (int d = 0; d < NC; ++d) Q[d] = 0.0;
    for (int i = 0; i < G.m; ++i) {
      double v[NS];
#pragma unroll
      for (int q = 0; q < NS; ++q) v[q] = G.val[i * G.total + sp[q]];
      const double si = __longlong_as_double((long long)smax_bits[i]);
#pragma unroll
      for (int d = 0; d < NC; ++d) {
        // child d in Morton child order: digit group (b_x, b_y[, b_z]), x most significant (C10)
        const int bx = (d >> (D - 1)) & 1, by = (d >> (D - 2)) & 1, bz = D == 3 ? (d & 1) : 0;
        const int cb = bx | (by << 1) | (bz << 2);
        const double uh = predict_rn<D>(v, cb);
        const double dd = __dsub_rn(G.val[i * G.total + c0 + d], uh);
        const double t = __ddiv_rn(dd, si);
        Q[d] = fmax(Q[d], __dmul_rn(t, t));
      }
    }
#pragma unroll
    for (int d = 0; d < NC; ++d) G.Q[c0 + d] = Q[d];
  }
}

struct Thresh { double E[kMaxLevels + 1]; };  // E_j = eps^2 2^{d (j - J)}

// The refine / grade / coarsen sweeps visit levels < J only (positions [0, off[J])): leaves at the
// finest level cannot refine, and internal nodes (whose grading / collapse is tested) live below J.
// P6 step 1: R0 = {leaf n : level < J, D(n) > eps_level} (strict).
// "something changed" flags are raised once per warp (a store per marked node to one address serialises)
__device__ __forceinline__ void raise_flag(bool any, int* flag) {
  if (__any_sync(0xffffffffu, any) && (threadIdx.x & 31) == 0) *flag = 1;
}

__global__ void k_refine_initial(GridDev G, Thresh Th, int* flag) {
  bool any = false;
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < G.off[G.J]; p += int64_t(gridDim.x) * blockDim.x) {
    if ((G.st[p] & ST_KIND) != ST_LEAF) continue;
    const int j = level_of(G, p);
    if (j < G.J && G.Q[p] > Th.E[j]) { G.mark[p] = 1; any = true; }
  }
  raise_flag(any, flag);
}

// P5/P6 grading repair: every internal node needs all level-j cells within radius 2 (inside Omega);
// a missing one marks the leaf covering it (its first present ancestor) for refinement.  A level-j
// position exists iff its parent is internal, so the 5^D box is tested through its 3^D parents at
// level j-1: a non-internal parent is either the covering leaf itself or absent (then the covering
// leaf is its first present ancestor) -- the same marks as testing the 5^D positions one by one.
template <int D>
__global__ void k_grade_mark(GridDev G, int* flag) {
  bool any = false;
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < G.off[G.J]; p += int64_t(gridDim.x) * blockDim.x) {
    if ((G.st[p] & ST_KIND) != ST_INTERNAL) continue;
    const int j = level_of(G, p);
    if (j == 0) continue;  // the root's box is the root itself
    const int n = 1 << j;
    int k[3] = {0, 0, 0};
    morton_dec<D>(uint64_t(p - G.off[j]), k);
    const int R = kGradeRadius;
    int lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
    for (int a = 0; a < D; ++a) {
      lo[a] = max(k[a] - R, 0) >> 1;
      hi[a] = min(k[a] + R, n - 1) >> 1;
    }
    for (int z = lo[2]; z <= hi[2]; ++z)
      for (int y = lo[1]; y <= hi[1]; ++y)
        for (int x = lo[0]; x <= hi[0]; ++x) {
          int q[3] = {x, y, z};
          const int64_t pq = posk<D>(G, j - 1, q);
          const uint8_t sq = G.st[pq] & ST_KIND;
          if (sq == ST_INTERNAL) continue;
          if (sq == ST_LEAF) {
            if (!G.mark[pq]) G.mark[pq] = 1;
            any = true;
            continue;
          }
          int la = j - 1;
          while (la > 0) {
            q[0] >>= 1; q[1] >>= 1; if (D == 3) q[2] >>= 1;
            --la;
            const int64_t pa = posk<D>(G, la, q);
            if ((G.st[pa] & ST_KIND) != ST_ABSENT) {
              if (!G.mark[pa]) G.mark[pa] = 1;
              any = true;
              break;
            }
          }
        }
  }
  raise_flag(any, flag);
}

// Refine every marked leaf: it becomes internal, its 2^D children are new leaves.
template <int D>
__global__ void k_refine_apply(GridDev G) {
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < G.off[G.J]; p += int64_t(gridDim.x) * blockDim.x) {
    if (!G.mark[p]) continue;
    G.mark[p] = 0;
    if ((G.st[p] & ST_KIND) != ST_LEAF) continue;
    const int j = level_of(G, p);
    G.st[p] = ST_INTERNAL | (G.st[p] & ST_NEW);
    const int64_t c = G.off[j + 1] + ((p - G.off[j]) << D);
    for (int d = 0; d < (1 << D); ++d) {
      G.st[c + d] = ST_LEAF | ST_NEW;
      G.Q[c + d] = 0.0;
    }
  }
}

// H6.4 new-node values by prediction (P2), one level at a time in increasing order.
template <int D>
__global__ void k_predict_new(GridDev G, int j, int* err) {
  constexpr int NS = D == 2 ? 9 : 27;
  const int64_t nj = int64_t(1) << (D * j);
  for (int64_t s = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; s < nj; s += int64_t(gridDim.x) * blockDim.x) {
    const int64_t p = G.off[j] + s;
    if (!(G.st[p] & ST_NEW)) continue;
    int k[3] = {0, 0, 0};
    morton_dec<D>(uint64_t(s), k);
    int kp[3] = {k[0] >> 1, k[1] >> 1, D == 3 ? k[2] >> 1 : 0};
    const int cb = (k[0] & 1) | ((k[1] & 1) << 1) | (D == 3 ? ((k[2] & 1) << 2) : 0);
    int64_t sp[NS];
    stencil_pos<D>(G, j - 1, kp, sp);
    bool ok = true;
#pragma unroll
    for (int q = 0; q < NS; ++q) ok = ok && (G.st[sp[q]] & ST_KIND) != ST_ABSENT;
    if (!ok) { atomicExch(err, 1); continue; }
    for (int i = 0; i < G.m; ++i) {
      double v[NS];
#pragma unroll
      for (int q = 0; q < NS; ++q) v[q] = G.val[i * G.total + sp[q]];
      G.val[i * G.total + p] = predict_rn<D>(v, cb);
    }
  }
}

// P7 coarsening sweep, in two passes.  A node P = (j, k) may not collapse while an internal node of level
// j+1 lies within distance 2 of one of its children (grading, R-G2), i.e. in the box [2k-2, 2k+3]^D --
// exactly the children of the 3^D level-j neighbours of P.  Pass 1 sets bit 2 of mark on every internal
// node with an internal child (levels L_min .. J-2; at J-1 all children are leaves); pass 2 marks (bit 1)
// every collapsible node: internal, level in [L_min, J), all children leaves that are not new with
// D < eps_{j+1} (strict), and no neighbour within distance 1 (inside Omega) carrying bit 2 -- 3^D byte
// reads per candidate instead of (2R+2)^D.  The apply pass collapses bit-1 nodes and clears the marks.
template <int D>
__global__ void k_coarsen_hic(GridDev G) {
  for (int64_t p = G.off[G.lmin] + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < G.off[G.J - 1];
       p += int64_t(gridDim.x) * blockDim.x) {
    if ((G.st[p] & ST_KIND) != ST_INTERNAL) continue;
    const int j = level_of(G, p);
    const int64_t c = G.off[j + 1] + ((p - G.off[j]) << D);
    bool hic = false;
#pragma unroll
    for (int d = 0; d < (1 << D); ++d) hic = hic || (G.st[c + d] & ST_KIND) == ST_INTERNAL;
    if (hic) G.mark[p] = 2;
  }
}

template <int D>
__global__ void k_coarsen_mark(GridDev G, Thresh Th, int* flag) {
  bool any = false;
  for (int64_t p = G.off[G.lmin] + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < G.off[G.J];
       p += int64_t(gridDim.x) * blockDim.x) {
    if ((G.st[p] & ST_KIND) != ST_INTERNAL) continue;
    const int j = level_of(G, p);
    const int64_t c = G.off[j + 1] + ((p - G.off[j]) << D);
    const double E = Th.E[j + 1];
    bool ok = true;
    for (int d = 0; d < (1 << D) && ok; ++d) {
      const uint8_t s = G.st[c + d];
      ok = (s == ST_LEAF) && (G.Q[c + d] < E);  // leaf, not new, D < eps_{j+1} (strict)
    }
    if (!ok) continue;
    int k[3] = {0, 0, 0};
    morton_dec<D>(uint64_t(p - G.off[j]), k);
    const int n = 1 << j;
    for (int z = (D == 3 ? k[2] - 1 : 0); ok && z <= (D == 3 ? k[2] + 1 : 0); ++z)
      for (int y = k[1] - 1; ok && y <= k[1] + 1; ++y)
        for (int x = k[0] - 1; ok && x <= k[0] + 1; ++x) {
          if (x < 0 || x >= n || y < 0 || y >= n || (D == 3 && (z < 0 || z >= n))) continue;
          int q[3] = {x, y, z};
          if (G.mark[posk<D>(G, j, q)] & 2) ok = false;
        }
    if (ok) { G.mark[p] |= 1; any = true; }
  }
  raise_flag(any, flag);
}

template <int D>
__global__ void k_coarsen_apply(GridDev G) {
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < G.off[G.J]; p += int64_t(gridDim.x) * blockDim.x) {
    const uint8_t mk = G.mark[p];
    if (!mk) continue;
    G.mark[p] = 0;
    if (!(mk & 1)) continue;
    const int j = level_of(G, p);
    G.st[p] = ST_LEAF;  // value = its projection, already stored
    const int64_t c = G.off[j + 1] + ((p - G.off[j]) << D);
    for (int d = 0; d < (1 << D); ++d) G.st[c + d] = ST_ABSENT;
  }
}


// Tree invariants: leaves at level >= L_min, internal nodes have all children and satisfy the
// radius-2 grading (DESIGN.md R-G2).
// Also clears the NEW bits of the adaptation (H6.5: new nodes are excluded only during this call).
template <int D>
__global__ void k_check(GridDev G, int* err) {
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < G.total; p += int64_t(gridDim.x) * blockDim.x) {
    const uint8_t s0 = G.st[p];
    if (s0 & ST_NEW) G.st[p] = s0 & ST_KIND;
    const uint8_t s = s0 & ST_KIND;
    if (s == ST_ABSENT) continue;
    const int j = level_of(G, p);
    if (s == ST_LEAF) {
      if (j < G.lmin) atomicExch(err, 2);
      continue;
    }
    if (j >= G.J) { atomicExch(err, 3); continue; }
    const int64_t c = G.off[j + 1] + ((p - G.off[j]) << D);
    for (int d = 0; d < (1 << D); ++d)
      if ((G.st[c + d] & ST_KIND) == ST_ABSENT) atomicExch(err, 4);
    if (j == 0) continue;
    // grading: every level-j position within radius 2 (inside Omega) exists, i.e. its parent is internal
    // (a parent with a missing child is caught by the children test above): 3^D parents, not 5^D cells
    int k[3] = {0, 0, 0};
    morton_dec<D>(uint64_t(p - G.off[j]), k);
    const int n = 1 << j, R = kGradeRadius;
    int lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
    for (int a = 0; a < D; ++a) {
      lo[a] = max(k[a] - R, 0) >> 1;
      hi[a] = min(k[a] + R, n - 1) >> 1;
    }
    for (int z = lo[2]; z <= hi[2]; ++z)
      for (int y = lo[1]; y <= hi[1]; ++y)
        for (int x = lo[0]; x <= hi[0]; ++x) {
          int q[3] = {x, y, z};
          if ((G.st[posk<D>(G, j - 1, q)] & ST_KIND) != ST_INTERNAL) atomicExch(err, 5);
        }
  }
}

struct IsLeaf {
  const uint8_t* st;
  __device__ int operator()(int64_t p) const { return (st[p] & ST_KIND) == ST_LEAF ? 1 : 0; }
};
struct IsFineFace {  // interface record with finer leaves (type 2)
  const int8_t* t;
  __device__ bool operator()(int64_t r) const { return t[r] == 2; }
};
struct IsMarked {
  const uint8_t* mk;
  __device__ int operator()(int64_t p) const { return mk[p] ? 1 : 0; }
};

__global__ void k_gather_leaves(GridDev G) {
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < G.total; p += int64_t(gridDim.x) * blockDim.x) {
    if ((G.st[p] & ST_KIND) != ST_LEAF) continue;
    const int j = level_of(G, p);
    const int64_t r = G.lidx[p];
    G.keys[r] = (uint64_t(j) << kLevelShift) | uint64_t(p - G.off[j]);
    G.lev[r] = uint8_t(j);
    for (int i = 0; i < G.m; ++i) G.u[i * G.N + r] = G.val[i * G.total + p];
  }
}

// ------------------------------------------------------------------ FV operator topology (O.5)
// Face order (-x, +x, -y, +y, -z, +z).  Per face: same-level leaf (F2), boundary (F3, no term),
// internal neighbour => 2^{D-1} fine-leaf terms with C's stencil (F5), absent neighbour => one ghost
// term from the coarse leaf L = parent(nb) and L's stencil (F4).
template <int D>
__device__ __forceinline__ int face_kind(const GridDev& G, int j, const int* k, int a, int dir, int64_t* pnb) {
  int nb[3] = {k[0], k[1], D == 3 ? k[2] : 0};
  nb[a] += dir;
  const int n = 1 << j;
  if (nb[a] < 0 || nb[a] >= n) return 0;
  const int64_t pn = posk<D>(G, j, nb);
  *pnb = pn;
  const uint8_t s = G.st[pn] & ST_KIND;
  return s == ST_LEAF ? 1 : (s == ST_INTERNAL ? 2 : 3);
}

// Per-row interface-record count (faces toward a coarser or finer neighbour, O.5 F4/F5).
template <int D>
__global__ void k_op_count(GridDev G, int32_t* cnt, int* err) {
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < G.N; r += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t key = G.keys[r];
    const int j = int(key >> kLevelShift);
    int k[3] = {0, 0, 0};
    morton_dec<D>(key & ((1ull << kLevelShift) - 1), k);
    int c = 0;
    for (int a = 0; a < D; ++a)
      for (int dir = -1; dir <= 1; dir += 2) {
        int64_t pn = -1;
        const int kind = face_kind<D>(G, j, k, a, dir, &pn);
        if (kind == 3 && j == 0) atomicExch(err, 6);
        c += kind >= 2;
      }
    cnt[r] = c;
  }
}

template <int D>
__device__ __forceinline__ int32_t vindex(const GridDev& G, int64_t p) {
  return (G.st[p] & ST_KIND) == ST_LEAF ? G.lidx[p] : int32_t(G.N + G.iidx[p]);
}

// Row topology: face codes, interface record headers (type, child bits, fine leaves) and each record's
// stencil centre (the 3^D stencils themselves are written by k_rec_mark / k_rec_sten, one thread per
// stencil entry), and the Gershgorin row sums for rho_1 (reading R-K2; the terms are dyadic with short
// mantissas, so the sums are exact in any order).
template <int D>
__global__ void k_op_fill(GridDev G, const int32_t* rec_off, int64_t* ctr, unsigned long long* rho_bits) {
  const double gw = 1.0 + (D == 2 ? 1.5625 : 1.953125);  // 1 + (5/4)^D: abs weights of a predicted ghost
  unsigned long long rmax = 0;  // bit pattern of the largest row sum (>= 0: ordered like the value)
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < G.N; r += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t key = G.keys[r];
    const int j = int(key >> kLevelShift);
    int k[3] = {0, 0, 0};
    morton_dec<D>(key & ((1ull << kLevelShift) - 1), k);
    const double cj = ldexp(1.0, 2 * j);
    const double cf = ldexp(1.0, 2 * (j + 1) - D);
    int32_t rec = rec_off[r];
    double rowsum = 0.0;
    int f = 0;
    for (int a = 0; a < D; ++a)
      for (int dir = -1; dir <= 1; dir += 2, ++f) {
        int64_t pn = -1;
        const int kind = face_kind<D>(G, j, k, a, dir, &pn);
        int32_t code = -1;
        if (kind == 1) {
          code = G.lidx[pn];
          rowsum += 2.0 * cj;
        } else if (kind == 3) {  // coarse neighbour: ghost = prediction of nb from L = parent(nb)
          int nb[3] = {k[0], k[1], D == 3 ? k[2] : 0};
          nb[a] += dir;
          int L[3] = {nb[0] >> 1, nb[1] >> 1, nb[2] >> 1};
          code = -2 - rec;
          G.if_type[rec] = 1;
          G.if_cb[rec] = int8_t((nb[0] & 1) | ((nb[1] & 1) << 1) | ((nb[2] & 1) << 2));
          *reinterpret_cast<int4*>(G.if_fine + int64_t(rec) * 4) = make_int4(-1, -1, -1, -1);
          ctr[rec] = posk<D>(G, j - 1, L);
          ++rec;
          rowsum += G.op_mode ? 2.0 * (cj / 1.5) : gw * cj;  // two-point: one link to L (reading R-T)
        } else if (kind == 2) {  // finer neighbours: one record per face (mirror of their ghost terms)
          int nb[3] = {k[0], k[1], D == 3 ? k[2] : 0};
          nb[a] += dir;
          code = -2 - rec;
          G.if_type[rec] = 2;
          G.if_cb[rec] = int8_t(a | ((dir > 0 ? 1 : 0) << 2));
          int fine[4] = {-1, -1, -1, -1};
          for (int d = 0; d < (1 << D); ++d) {
            int fc[3] = {0, 0, 0};
            for (int x = 0; x < D; ++x) fc[x] = 2 * nb[x] + ((d >> (D - 1 - x)) & 1);
            if (fc[a] != (dir > 0 ? 2 * nb[a] : 2 * nb[a] + 1)) continue;
            int q = 0, t = 0;  // bits of the other axes, increasing axis order
            for (int x = 0; x < D; ++x) {
              if (x == a) continue;
              q |= (fc[x] & 1) << t;
              ++t;
            }
            fine[q] = G.lidx[posk<D>(G, j + 1, fc)];
            rowsum += G.op_mode ? 2.0 * (cf / 1.5) : gw * cf;
          }
          *reinterpret_cast<int4*>(G.if_fine + int64_t(rec) * 4) = make_int4(fine[0], fine[1], fine[2], fine[3]);
          ctr[rec] = posk<D>(G, j, k);
          ++rec;
        }
        G.nbr[int64_t(f) * G.N + r] = code;
      }
    const unsigned long long b = (unsigned long long)__double_as_longlong(rowsum);
    rmax = b > rmax ? b : rmax;
  }
  // one atomic per warp (a per-leaf atomic on one address serialised ~10^6 updates)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long v = __shfl_xor_sync(0xffffffffu, rmax, o);
    rmax = v > rmax ? v : rmax;
  }
  if ((threadIdx.x & 31) == 0 && rmax) atomicMax(rho_bits, rmax);
}

// One thread per (record, z layer of its mirrored 3^D stencil): the centre is decoded once for the
// layer's 9 entries (x fastest, then y).
template <int D>
__device__ __forceinline__ void sten_layer(const GridDev& G, int64_t c, int oz, int64_t* out) {
  const int j = level_of(G, c);
  int k[3] = {0, 0, 0};
  morton_dec<D>(uint64_t(c - G.off[j]), k);
  const int n = 1 << j;
  const int z = D == 3 ? mir(k[2] + oz - 1, n) : 0;
#pragma unroll
  for (int oy = 0; oy < 3; ++oy)
#pragma unroll
    for (int ox = 0; ox < 3; ++ox) {
      int e[3] = {mir(k[0] + ox - 1, n), mir(k[1] + oy - 1, n), z};
      out[oy * 3 + ox] = posk<D>(G, j, e);
    }
}

// Internal stencil nodes are marked as needed (their values are projections of the current vector,
// F6); an absent one is a structure error.
template <int D>
__global__ void k_rec_mark(GridDev G, const int64_t* ctr, int* err) {
  constexpr int NZ = D == 2 ? 1 : 3;
  const int64_t tot = G.n_if * NZ;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < tot; t += int64_t(gridDim.x) * blockDim.x) {
    int64_t sp[9];
    sten_layer<D>(G, ctr[t / NZ], int(t % NZ), sp);
#pragma unroll
    for (int q = 0; q < 9; ++q) {
      const uint8_t s = G.st[sp[q]] & ST_KIND;
      if (s == ST_ABSENT) atomicExch(err, 7);
      else if (s == ST_INTERNAL && !G.mark[sp[q]]) G.mark[sp[q]] = 1;
    }
  }
}

// The value indices into V = [leaves | needed internal nodes] of every stencil entry.
template <int D>
__global__ void k_rec_sten(GridDev G, const int64_t* ctr) {
  constexpr int NZ = D == 2 ? 1 : 3;
  const int64_t tot = G.n_if * NZ;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < tot; t += int64_t(gridDim.x) * blockDim.x) {
    int64_t sp[9];
    sten_layer<D>(G, ctr[t / NZ], int(t % NZ), sp);
    const int64_t rec = t / NZ, oz = t % NZ;  // entry-major layout: entry e of record r at e * n_if + r
#pragma unroll
    for (int q = 0; q < 9; ++q) G.if_sten[(oz * 9 + q) * G.n_if + rec] = vindex<D>(G, sp[q]);
  }
}

// Ghost links: a coarse-neighbour record (type 1) of fine leaf C reads the ghost computed once for
// the coarse leaf L's face record (type 2) toward C: if_fine[rec*4] = rec2 * 4 + q with q = C's bits
// on the axes other than the face normal (the order of the fine leaves in rec2).
template <int D>
__global__ void k_op_link(GridDev G, int* err) {
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < G.N; r += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t key = G.keys[r];
    const int j = int(key >> kLevelShift);
    int k[3] = {0, 0, 0};
    morton_dec<D>(key & ((1ull << kLevelShift) - 1), k);
    int f = 0;
    for (int a = 0; a < D; ++a)
      for (int dir = -1; dir <= 1; dir += 2, ++f) {
        const int32_t code = G.nbr[int64_t(f) * G.N + r];
        if (code > -2) continue;
        const int32_t rec = -2 - code;
        if (G.if_type[rec] != 1) continue;
        int L[3] = {k[0], k[1], D == 3 ? k[2] : 0};
        L[a] += dir;
        L[0] >>= 1; L[1] >>= 1; L[2] >>= 1;
        const int64_t pl = posk<D>(G, j - 1, L);
        const int32_t rowL = G.lidx[pl];
        const int fL = 2 * a + (dir < 0 ? 1 : 0);  // L's face toward C
        const int32_t codeL = G.nbr[int64_t(fL) * G.N + rowL];
        if (codeL > -2 || G.if_type[-2 - codeL] != 2) { atomicExch(err, 8); continue; }
        int q = 0, t = 0;
        for (int x = 0; x < D; ++x) {
          if (x == a) continue;
          q |= (k[x] & 1) << t;
          ++t;
        }
        G.if_fine[int64_t(rec) * 4] = (-2 - codeL) * 4 + q;
      }
  }
}

// Cost of each chunk of kR4Chunk rows of the matrix-free Rock4 stage: its interface faces (from the
// record offsets), and the identity order the sort permutes.
__global__ void k_chunk_cost(int64_t N, const int32_t* rec_off, int32_t* cost, int32_t* idx) {
  const int64_t nch = (N + kR4Chunk - 1) / kR4Chunk;
  for (int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; c < nch; c += int64_t(gridDim.x) * blockDim.x) {
    const int64_t a = c * kR4Chunk, b = a + kR4Chunk < N ? a + kR4Chunk : N;
    cost[c] = rec_off[b] - rec_off[a];
    idx[c] = int32_t(c);
  }
}

// 3-D ghost-phase face codes (GridDev::nbrg): the coarse-neighbour link is resolved here once instead of
// through two dependent loads per face and stage.
__global__ void k_nbr_ghost(GridDev G, int nf) {
  const int64_t tot = int64_t(nf) * G.N;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < tot; t += int64_t(gridDim.x) * blockDim.x) {
    const int32_t c = G.nbr[t];
    int32_t o = c;
    if (c <= -2) {
      const int32_t rec = -2 - c;
      o = G.if_type[rec] == 1 ? -2 - 2 * G.if_fine[int64_t(rec) * 4] : -3 - 2 * rec;
    }
    G.nbrg[t] = o;
  }
}

// Needed internal nodes (marked; internal nodes live below level J).
__global__ void k_need_list(GridDev G, int64_t* need_pos) {
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < G.off[G.J]; p += int64_t(gridDim.x) * blockDim.x)
    if (G.mark[p]) need_pos[G.iidx[p]] = p;
}

// Projection expansion of a needed internal node: its leaf descendants with weights 2^{-D(l'-l)}
// (F6: internal value = projection of the current vector).  pass 0 counts, pass 1 fills.
template <int D>
__global__ void k_expand(GridDev G, const int64_t* need_pos, int32_t* cnt, int pass) {
  for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < G.n_need; q += int64_t(gridDim.x) * blockDim.x) {
    const int64_t p0 = need_pos[q];
    const int l0 = level_of(G, p0);
    int64_t stk_s[128];
    int8_t stk_l[128];
    int top = 0;
    stk_s[0] = p0 - G.off[l0];
    stk_l[0] = int8_t(l0);
    top = 1;
    int32_t c = 0;
    int32_t w0 = pass ? G.exp_start[q] : 0;
    while (top > 0) {
      --top;
      const int64_t s = stk_s[top];
      const int l = stk_l[top];
      const int64_t p = G.off[l] + s;
      const uint8_t st = G.st[p] & ST_KIND;
      if (st == ST_LEAF) {
        if (pass) {
          G.exp_leaf[w0 + c] = G.lidx[p];
          G.exp_w[w0 + c] = ldexp(1.0, -D * (l - l0));
        }
        ++c;
      } else if (st == ST_INTERNAL && top + (1 << D) <= 128) {
        for (int d = (1 << D) - 1; d >= 0; --d) {
          stk_s[top] = (s << D) + d;
          stk_l[top] = int8_t(l + 1);
          ++top;
        }
      }
    }
    if (!pass) cnt[q] = c;
  }
}

// 3-D Rock4 projection work (GridDev::proj_*): "simple" = the expansion is 2^D consecutive leaf
// indices inside one stage chunk (the node's children, all leaves).  pass 0 counts per chunk and lists
// the other nodes, pass 1 fills the per-chunk lists (order inside a chunk is immaterial: each node's
// projection is computed on its own).
template <int D>
__global__ void k_proj_class(GridDev G, int32_t* ccnt, int pass) {
  constexpr int NC = 1 << D;
  for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < G.n_need; q += int64_t(gridDim.x) * blockDim.x) {
    const int32_t e0 = G.exp_start[q], e1 = G.exp_start[q + 1];
    bool simple = e1 - e0 == NC;  // the node's 2^D children, all leaves (consecutive leaf indices) ...
    const int32_t l0 = G.exp_leaf[e0];
    for (int k = 1; k < NC && simple; ++k) simple = G.exp_leaf[e0 + k] == l0 + k;
    simple = simple && (l0 / kR4Chunk) == ((l0 + NC - 1) / kR4Chunk);  // ... inside one chunk
    if (pass == 0) {
      if (simple) atomicAdd(ccnt + l0 / kR4Chunk, 1);
      else G.proj_ns[atomicAdd(G.proj_ns_count, 1)] = int32_t(q);
    } else if (simple) {
      const int c = l0 / kR4Chunk;
      G.proj_cnode[G.proj_cstart[c] + atomicAdd(ccnt + c, 1)] = make_int2(int32_t(q), l0);
    }
  }
}

// ------------------------------------------------------------------ FV apply (rd_fv_apply, Rock4)
template <int D>
__global__ void k_need_values(GridDev G, double* V) {
  for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < G.n_need; q += int64_t(gridDim.x) * blockDim.x) {
    double acc = 0.0;
    for (int32_t e = G.exp_start[q]; e < G.exp_start[q + 1]; ++e) acc += G.exp_w[e] * V[G.exp_leaf[e]];
    V[G.N + q] = acc;
  }
}

}  // namespace

template <int D>
__global__ void k_fv_apply(GridDev G, const double* V, double* y) {
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < G.N; r += int64_t(gridDim.x) * blockDim.x)
    y[r] = fv_row<D>(G, V, r);
}

void fv_apply_launch(const GridDev& G, double* V, double* y, cudaStream_t st) {
  if (G.dim == 2) {
    if (G.n_need) { k_need_values<2><<<nblk(G.n_need), kTB, 0, st>>>(G, V); RD_COUNT_LAUNCH(1); }
    k_fv_apply<2><<<nblk(G.N), kTB, 0, st>>>(G, V, y);
    RD_COUNT_LAUNCH(1);
  } else {
    if (G.n_need) { k_need_values<3><<<nblk(G.n_need), kTB, 0, st>>>(G, V); RD_COUNT_LAUNCH(1); }
    k_fv_apply<3><<<nblk(G.N), kTB, 0, st>>>(G, V, y);
    RD_COUNT_LAUNCH(1);
  }
}

// ------------------------------------------------------------------ host side
namespace {

template <class T>
rd_status grow(T** p, int64_t* cap, int64_t need, cudaStream_t st) {
  if (need <= *cap && *p) return RD_OK;
  rd_free(*p, st);
  *p = nullptr;
  const int64_t c = std::max<int64_t>(need + need / 4, 1024);
  RD_CUDA_TRY(rd_malloc(reinterpret_cast<void**>(p), size_t(c) * sizeof(T), st));
  *cap = c;
  return RD_OK;
}

rd_status cub_tmp(mr_grid* g, size_t bytes, cudaStream_t st) {
  if (bytes <= g->cub_bytes) return RD_OK;
  if (g->cub_tmp) rd_free(g->cub_tmp, st);
  g->cub_tmp = nullptr;
  RD_CUDA_TRY(rd_malloc(&g->cub_tmp, bytes, st));
  g->cub_bytes = bytes;
  return RD_OK;
}

template <class It>
rd_status excl_scan(mr_grid* g, It in, int32_t* out, int64_t n, cudaStream_t st) {
  size_t bytes = 0;
  RD_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n, st));
  RD_TRY(cub_tmp(g, bytes, st));
  RD_CUDA_TRY(cub::DeviceScan::ExclusiveSum(g->cub_tmp, bytes, in, out, n, st));
  RD_COUNT_LAUNCH(2);  // CUB init + scan kernels
  return RD_OK;
}

// read device int flag idx (synchronises), and reset it.  Flag 1 is the sticky structure-error flag of
// the stencil kernels (k_significance, k_predict_new): it is not read where it is raised but at the
// next synchronisation of the call, which then fails with RD_ESTRUCT (saves two host round trips per
// adaptation).
rd_status read_flag(mr_grid* g, int idx, int* out, cudaStream_t st) {
  RD_CUDA_TRY(cudaMemcpyAsync(g->hflag, g->dflag, 4 * sizeof(int), cudaMemcpyDeviceToHost, st));
  RD_CUDA_TRY(cudaStreamSynchronize(st));
  *out = g->hflag[idx];
  RD_CUDA_TRY(cudaMemsetAsync(g->dflag + idx, 0, sizeof(int), st));
  if (g->hflag[1]) {
    RD_CUDA_TRY(cudaMemsetAsync(g->dflag + 1, 0, sizeof(int), st));
    return RD_ESTRUCT;
  }
  return RD_OK;
}

Thresh thresholds(const mr_grid* g) {
  Thresh t{};
  for (int j = 0; j <= g->d.J; ++j) t.E[j] = std::ldexp(g->eps * g->eps, g->d.dim * (j - g->d.J));
  return t;
}

template <int D>
rd_status significance(mr_grid* g, cudaStream_t st, int from_leaves) {
  GridDev& G = g->d;
  for (int j = G.J - 1; j >= 0; --j) {
    k_project<D><<<nblk(int64_t(1) << (D * j)), kTB, 0, st>>>(G, j);
    RD_COUNT_LAUNCH(1);
  }
  unsigned long long* smax = reinterpret_cast<unsigned long long*>(g->dflag + 8);
  k_fill_u64<<<1, 32, 0, st>>>(smax, G.m, (unsigned long long)__builtin_bit_cast(long long, 1.0));  // s_i >= 1
  RD_COUNT_LAUNCH(1);
  k_absmax<<<std::min<unsigned>(nblk(from_leaves ? G.N : G.total), 1184), kTB, 0, st>>>(G, smax, from_leaves);
  RD_COUNT_LAUNCH(1);
  k_significance<D><<<nblk(G.total), kTB, 0, st>>>(G, smax, std::max(1, G.lmin), g->dflag + 1);
  RD_COUNT_LAUNCH(1);
  RD_CUDA_TRY(cudaGetLastError());
  return RD_OK;  // a stencil error raises flag 1, reported at the call's next read_flag
}

template <int D>
rd_status coarsen_fixed_point(mr_grid* g, cudaStream_t st) {
  GridDev& G = g->d;
  const Thresh th = thresholds(g);
  if (G.lmin >= G.J) return RD_OK;  // nothing may coarsen
  const unsigned nb = nblk(G.off[G.J] - G.off[G.lmin]);
  auto sweep = [&]() {  // internal-child bits + mark (2 launches)
    if (G.lmin + 2 <= G.J) k_coarsen_hic<D><<<nblk(G.off[G.J - 1] - G.off[G.lmin]), kTB, 0, st>>>(G);
    k_coarsen_mark<D><<<nb, kTB, 0, st>>>(G, th, g->dflag);
    RD_COUNT_LAUNCH(2);
  };
  RD_CUDA_TRY(cudaMemsetAsync(g->dflag, 0, sizeof(int), st));
  for (int it = 0; it < 64 * (G.J + 1); it += 2) {  // checked every second iteration (see adapt_impl)
    sweep();
    k_coarsen_apply<D><<<nblk(G.off[G.J]), kTB, 0, st>>>(G);
    RD_CUDA_TRY(cudaMemsetAsync(g->dflag, 0, sizeof(int), st));
    sweep();
    RD_COUNT_LAUNCH(1);
    int any = 0;
    RD_TRY(read_flag(g, 0, &any, st));
    if (!any) return RD_OK;
    k_coarsen_apply<D><<<nblk(G.off[G.J]), kTB, 0, st>>>(G);
    RD_COUNT_LAUNCH(1);
  }
  return RD_ESTRUCT;
}

template <int D>
rd_status compact_and_compile(mr_grid* g, cudaStream_t st) {
  GridDev& G = g->d;
  SecTimer tm(st);
  k_check<D><<<nblk(G.total), kTB, 0, st>>>(G, g->dflag + 2);
  RD_COUNT_LAUNCH(1);
  // leaf numbering in (level, Morton) order = ascending key
  cub::CountingInputIterator<int64_t> cnt_it(0);
  cub::TransformInputIterator<int, IsLeaf, cub::CountingInputIterator<int64_t>> leaf_it(cnt_it, IsLeaf{G.st});
  RD_TRY(excl_scan(g, leaf_it, G.lidx, G.total, st));
  int32_t* hl = reinterpret_cast<int32_t*>(g->hflag + 40);  // pinned: last leaf index, last state
  uint8_t* hs = reinterpret_cast<uint8_t*>(g->hflag + 41);
  RD_CUDA_TRY(cudaMemcpyAsync(hl, G.lidx + G.total - 1, 4, cudaMemcpyDeviceToHost, st));
  RD_CUDA_TRY(cudaMemcpyAsync(hs, G.st + G.total - 1, 1, cudaMemcpyDeviceToHost, st));
  int bad = 0;
  RD_TRY(read_flag(g, 2, &bad, st));  // synchronises: the check's flag and the two values above
  if (bad) return RD_ESTRUCT;
  const int32_t last = hl[0];
  const uint8_t lst = hs[0];
  G.N = int64_t(last) + ((lst & ST_KIND) == ST_LEAF ? 1 : 0);
  int64_t capk = g->cap_leaf;
  RD_TRY(grow(&G.keys, &capk, G.N, st));
  int64_t capu = g->cap_leaf * G.m;
  if (capk != g->cap_leaf || !G.u) {
    if (G.u) rd_free(G.u, st);
    G.u = nullptr;
    RD_CUDA_TRY(rd_malloc(&G.u, size_t(capk) * G.m * sizeof(double), st));
    if (G.nbr) rd_free(G.nbr, st);
    G.nbr = nullptr;
    RD_CUDA_TRY(rd_malloc(&G.nbr, size_t(capk) * 2 * D * sizeof(int32_t), st));
    if (G.nbrg) rd_free(G.nbrg, st);
    G.nbrg = nullptr;
    if (D == 3) RD_CUDA_TRY(rd_malloc(&G.nbrg, size_t(capk) * 2 * D * sizeof(int32_t), st));
    if (G.lev) rd_free(G.lev, st);
    G.lev = nullptr;
    RD_CUDA_TRY(rd_malloc(&G.lev, size_t(capk), st));
    g->cap_leaf = capk;
  }
  (void)capu;
  k_gather_leaves<<<nblk(G.total), kTB, 0, st>>>(G);
  RD_COUNT_LAUNCH(1);
  RD_CUDA_TRY(cudaGetLastError());
  tm.mark("  check+gather");
  return grid_rebuild_operator(g, st);
}

// The operator build's last host read, shared with the expansion count: rho_1 (its bits), the leaf
// level range (first / last key) and the flags (a structure error raised by the record, link or
// expansion-count kernels; the expansion fill repeats the count pass's walk).  Synchronises.
rd_status op_tail_reads(mr_grid* g, const unsigned long long* rho_bits, cudaStream_t st) {
  GridDev& G = g->d;
  unsigned long long* hrb = reinterpret_cast<unsigned long long*>(g->hflag + 28);
  uint64_t* hk = reinterpret_cast<uint64_t*>(g->hflag + 48);  // pinned [48..52)
  RD_CUDA_TRY(cudaMemcpyAsync(hrb, rho_bits, 8, cudaMemcpyDeviceToHost, st));
  if (G.N > 0) {
    RD_CUDA_TRY(cudaMemcpyAsync(hk, G.keys, 8, cudaMemcpyDeviceToHost, st));
    RD_CUDA_TRY(cudaMemcpyAsync(hk + 1, G.keys + G.N - 1, 8, cudaMemcpyDeviceToHost, st));
  }
  int bad = 0;
  RD_TRY(read_flag(g, 3, &bad, st));
  if (bad) return RD_ESTRUCT;
  g->rho1 = __builtin_bit_cast(double, *hrb);
  if (G.N > 0) {
    g->level_lo = int(hk[0] >> kLevelShift);
    g->level_hi = int(hk[1] >> kLevelShift);
  }
  return RD_OK;
}

template <int D>
rd_status rebuild_op(mr_grid* g, cudaStream_t st) {
  constexpr int NS = D == 2 ? 9 : 27;
  GridDev& G = g->d;
  SecTimer tm(st);
  // per-leaf record counts + needed internal marks
  RD_CUDA_TRY(cudaMemsetAsync(G.mark, 0, size_t(G.total), st));
  if (G.N + 1 > g->cap_scr) {
    rd_free(g->scr_cnt, st);
    rd_free(g->scr_off, st);
    g->scr_cnt = g->scr_off = nullptr;
    const int64_t c = (G.N + 1) * 5 / 4 + 1024;
    RD_CUDA_TRY(rd_malloc(&g->scr_cnt, size_t(c) * 4, st));
    RD_CUDA_TRY(rd_malloc(&g->scr_off, size_t(c) * 4, st));
    g->cap_scr = c;
  }
  int32_t* cnt = g->scr_cnt;
  int32_t* rec_off = g->scr_off;
  RD_CUDA_TRY(cudaMemsetAsync(cnt, 0, size_t(G.N + 1) * 4, st));
  k_op_count<D><<<nblk(G.N), kTB, 0, st>>>(G, cnt, g->dflag + 3);
  RD_COUNT_LAUNCH(1);
  RD_TRY(excl_scan(g, cnt, rec_off, G.N + 1, st));
  {  // longest-first chunk order for the matrix-free Rock4 stage's tickets
    const int64_t nch = (G.N + kR4Chunk - 1) / kR4Chunk;
    if (2 * nch > g->cap_chunk) {
      rd_free(g->scr_ccost, st); rd_free(g->scr_cidx, st); rd_free(G.chunk_order, st);
      rd_free(g->scr_pcnt, st); rd_free(G.proj_cstart, st);
      const int64_t c = 2 * nch + 1024;
      RD_CUDA_TRY(rd_malloc(&g->scr_ccost, size_t(c) * 4, st));
      RD_CUDA_TRY(rd_malloc(&g->scr_cidx, size_t(c) * 4, st));
      RD_CUDA_TRY(rd_malloc(&G.chunk_order, size_t(c) * 4, st));
      RD_CUDA_TRY(rd_malloc(&g->scr_pcnt, size_t(c) * 4, st));
      RD_CUDA_TRY(rd_malloc(&G.proj_cstart, size_t(c) * 4, st));
      g->cap_chunk = c;
    }
    int32_t* cost = g->scr_ccost;
    int32_t* idx = g->scr_cidx;
    k_chunk_cost<<<nblk(nch), kTB, 0, st>>>(G.N, rec_off, cost, idx);
    RD_COUNT_LAUNCH(1);
    size_t bytes = 0;
    RD_CUDA_TRY(cub::DeviceRadixSort::SortPairsDescending(nullptr, bytes, cost, cost + nch, idx, G.chunk_order, nch));
    RD_TRY(cub_tmp(g, bytes, st));
    RD_CUDA_TRY(cub::DeviceRadixSort::SortPairsDescending(g->cub_tmp, bytes, cost, cost + nch, idx, G.chunk_order,
                                                           nch, 0, 32, st));
    RD_COUNT_LAUNCH(3);
  }
  int32_t* hv = reinterpret_cast<int32_t*>(g->hflag + 16);  // pinned
  uint8_t* hm = reinterpret_cast<uint8_t*>(g->hflag + 20);
  RD_CUDA_TRY(cudaMemcpyAsync(hv, rec_off + G.N, 4, cudaMemcpyDeviceToHost, st));
  int bad = 0;
  RD_TRY(read_flag(g, 3, &bad, st));
  if (bad) return RD_ESTRUCT;
  tm.mark("  op count+scans");
  const int32_t nif = hv[0];
  G.n_if = nif;
  int64_t c1 = g->cap_if;
  RD_TRY(grow(&G.if_type, &c1, G.n_if + 1, st));
  if (c1 != g->cap_if) {
    rd_free(G.if_cb, st); rd_free(G.if_fine, st); rd_free(G.if_sten, st); rd_free(g->scr_ctr, st);
    rd_free(G.if2_list, st);
    RD_CUDA_TRY(rd_malloc(&G.if2_list, size_t(c1) * 4, st));
    RD_CUDA_TRY(rd_malloc(&G.if_cb, size_t(c1), st));
    RD_CUDA_TRY(rd_malloc(&G.if_fine, size_t(c1) * 4 * 4, st));
    RD_CUDA_TRY(rd_malloc(&G.if_sten, size_t(c1) * NS * 4, st));
    RD_CUDA_TRY(rd_malloc(&g->scr_ctr, size_t(c1) * 8, st));
    g->cap_if = c1;
  }
  unsigned long long* rho_bits = reinterpret_cast<unsigned long long*>(g->dflag + 4);
  RD_CUDA_TRY(cudaMemsetAsync(rho_bits, 0, 8, st));
  k_op_fill<D><<<nblk(G.N), kTB, 0, st>>>(G, rec_off, g->scr_ctr, rho_bits);
  RD_COUNT_LAUNCH(1);
  if (G.n_if) {
    k_rec_mark<D><<<nblk(G.n_if * NS / 9), kTB, 0, st>>>(G, g->scr_ctr, g->dflag + 3);
    RD_COUNT_LAUNCH(1);
  }
  cub::CountingInputIterator<int64_t> cnt_it(0);
  cub::TransformInputIterator<int, IsMarked, cub::CountingInputIterator<int64_t>> mk_it(cnt_it, IsMarked{G.mark});
  RD_TRY(excl_scan(g, mk_it, G.iidx, G.total, st));
  RD_CUDA_TRY(cudaMemcpyAsync(hv + 1, G.iidx + G.total - 1, 4, cudaMemcpyDeviceToHost, st));
  RD_CUDA_TRY(cudaMemcpyAsync(hm, G.mark + G.total - 1, 1, cudaMemcpyDeviceToHost, st));
  if (G.n_if) {
    k_rec_sten<D><<<nblk(G.n_if * NS / 9), kTB, 0, st>>>(G, g->scr_ctr);
    RD_COUNT_LAUNCH(1);
  }
  k_op_link<D><<<nblk(G.N), kTB, 0, st>>>(G, g->dflag + 3);
  RD_COUNT_LAUNCH(1);
  if (D == 3) {
    k_nbr_ghost<<<nblk(G.N * 2 * D), kTB, 0, st>>>(G, 2 * D);
    RD_COUNT_LAUNCH(1);
    // the ghost phase's work list: the type-2 records (about a fifth of them), count left on the device
    if (G.n_if > 0) {
      cub::CountingInputIterator<int32_t> rec_it(0);
      cub::TransformInputIterator<bool, IsFineFace, cub::CountingInputIterator<int64_t>> fl_it(
          cub::CountingInputIterator<int64_t>(0), IsFineFace{G.if_type});
      size_t bytes = 0;
      RD_CUDA_TRY(cub::DeviceSelect::Flagged(nullptr, bytes, rec_it, fl_it, G.if2_list, G.if2_count, G.n_if, st));
      RD_TRY(cub_tmp(g, bytes, st));
      RD_CUDA_TRY(cub::DeviceSelect::Flagged(g->cub_tmp, bytes, rec_it, fl_it, G.if2_list, G.if2_count, G.n_if, st));
      RD_COUNT_LAUNCH(2);
    } else {
      RD_CUDA_TRY(cudaMemsetAsync(G.if2_count, 0, sizeof(int32_t), st));
    }
  }
  RD_TRY(read_flag(g, 3, &bad, st));  // stencil structure + ghost links; synchronises (hv[1], hm valid)
  if (bad) return RD_ESTRUCT;
  const int32_t nneed = hv[1];
  const uint8_t lmk = hm[0];
  G.n_need = int64_t(nneed) + (lmk ? 1 : 0);
  tm.mark("  op fill+link");
  // projection expansions of the needed internal nodes
  int64_t c2 = g->cap_need;
  RD_TRY(grow(&G.exp_start, &c2, G.n_need + 2, st));
  g->cap_need = c2;
  if (G.n_need) {
    if (G.n_need + 1 > g->cap_scr_need) {
      rd_free(g->scr_need, st);
      rd_free(g->scr_ecnt, st);
      g->scr_need = nullptr;
      g->scr_ecnt = nullptr;
      const int64_t c = (G.n_need + 1) * 5 / 4 + 1024;
      RD_CUDA_TRY(rd_malloc(&g->scr_need, size_t(c) * 8, st));
      RD_CUDA_TRY(rd_malloc(&g->scr_ecnt, size_t(c) * 4, st));
      g->cap_scr_need = c;
    }
    int64_t* need_pos = g->scr_need;
    int32_t* ecnt = g->scr_ecnt;
    RD_CUDA_TRY(cudaMemsetAsync(ecnt, 0, size_t(G.n_need + 1) * 4, st));
    k_need_list<<<nblk(G.off[G.J]), kTB, 0, st>>>(G, need_pos);
    RD_COUNT_LAUNCH(1);
    k_expand<D><<<nblk(G.n_need), kTB, 0, st>>>(G, need_pos, ecnt, 0);
    RD_COUNT_LAUNCH(1);
    RD_TRY(excl_scan(g, ecnt, G.exp_start, G.n_need + 1, st));
    int32_t* hn = reinterpret_cast<int32_t*>(g->hflag + 24);
    RD_CUDA_TRY(cudaMemcpyAsync(hn, G.exp_start + G.n_need, 4, cudaMemcpyDeviceToHost, st));
    RD_TRY(op_tail_reads(g, rho_bits, st));  // + rho_1 bits, level range, flags; synchronises
    const int32_t nexp = hn[0];
    g->n_exp = nexp;
    int64_t c3 = g->cap_exp;
    RD_TRY(grow(&G.exp_leaf, &c3, nexp + 1, st));
    if (c3 != g->cap_exp) {
      rd_free(G.exp_w, st);
      RD_CUDA_TRY(rd_malloc(&G.exp_w, size_t(c3) * 8, st));
      g->cap_exp = c3;
    }
    k_expand<D><<<nblk(G.n_need), kTB, 0, st>>>(G, need_pos, ecnt, 1);
    RD_COUNT_LAUNCH(1);
  } else {
    g->n_exp = 0;
    RD_TRY(op_tail_reads(g, rho_bits, st));
  }
  if (D == 3) {  // the 3-D Rock4 stage's per-chunk projection lists
    const int64_t nch = (G.N + kR4Chunk - 1) / kR4Chunk;
    if (G.n_need + 1 > g->cap_proj) {
      rd_free(G.proj_cnode, st);
      rd_free(G.proj_ns, st);
      const int64_t c = (G.n_need + 1) * 5 / 4 + 1024;
      RD_CUDA_TRY(rd_malloc(&G.proj_cnode, size_t(c) * 8, st));
      RD_CUDA_TRY(rd_malloc(&G.proj_ns, size_t(c) * 4, st));
      g->cap_proj = c;
    }
    // cap_chunk (chunk-order arrays, >= 2 nch) also sizes the per-chunk counts and offsets
    RD_CUDA_TRY(cudaMemsetAsync(g->scr_pcnt, 0, size_t(nch + 1) * 4, st));
    RD_CUDA_TRY(cudaMemsetAsync(G.proj_ns_count, 0, 4, st));
    if (G.n_need) {
      k_proj_class<D><<<nblk(G.n_need), kTB, 0, st>>>(G, g->scr_pcnt, 0);
      RD_COUNT_LAUNCH(1);
    }
    RD_TRY(excl_scan(g, g->scr_pcnt, G.proj_cstart, nch + 1, st));
    if (G.n_need) {
      RD_CUDA_TRY(cudaMemsetAsync(g->scr_pcnt, 0, size_t(nch + 1) * 4, st));
      k_proj_class<D><<<nblk(G.n_need), kTB, 0, st>>>(G, g->scr_pcnt, 1);
      RD_COUNT_LAUNCH(1);
    }
  }
  RD_CUDA_TRY(cudaMemsetAsync(G.mark, 0, size_t(G.total), st));
  tm.mark("  need+expand");
  RD_CUDA_TRY(cudaGetLastError());
  return RD_OK;
}

}  // namespace

rd_status grid_rebuild_operator(mr_grid* g, cudaStream_t st) {
  g->mat_state = 0;  // the assembled matrix (fvmat.cu) belongs to the previous leaf set
  return g->d.dim == 2 ? rebuild_op<2>(g, st) : rebuild_op<3>(g, st);  // (sets the level range too)
}

namespace {

rd_status alloc_grid(mr_grid* g, int dim, int lmin, int J, int m, double eps, cudaStream_t st) {
  GridDev& G = g->d;
  G.dim = dim; G.J = J; G.lmin = lmin; G.m = m;
  g->eps = eps;
  int64_t off = 0;
  for (int j = 0; j <= J + 1 && j < kMaxLevels + 2; ++j) {
    G.off[j] = off;
    if (j <= J) off += int64_t(1) << (dim * j);
  }
  for (int j = J + 2; j < kMaxLevels + 2; ++j) G.off[j] = off;
  G.total = off;
  RD_CUDA_TRY(rd_malloc(&G.st, size_t(G.total), st));
  RD_CUDA_TRY(rd_malloc(&G.mark, size_t(G.total), st));
  RD_CUDA_TRY(rd_malloc(&G.val, size_t(G.total) * m * 8, st));
  RD_CUDA_TRY(rd_malloc(&G.Q, size_t(G.total) * 8, st));
  RD_CUDA_TRY(rd_malloc(&G.lidx, size_t(G.total) * 4, st));
  RD_CUDA_TRY(rd_malloc(&G.iidx, size_t(G.total) * 4, st));
  RD_CUDA_TRY(rd_malloc(&g->dflag, 256 * sizeof(int), st));  // flags [0..8), rho [4..6), smax [8..8+2m)
  G.if2_count = g->dflag + 192;                                // [192]: type-2 record count (op build)
  G.proj_ns_count = g->dflag + 193;                            // [193]: non-simple projection count
  RD_CUDA_TRY(cudaMemsetAsync(g->dflag, 0, 256 * sizeof(int), st));
  RD_CUDA_TRY(cudaMemsetAsync(G.mark, 0, size_t(G.total), st));
  RD_CUDA_TRY(cudaMallocHost(&g->hflag, 64 * sizeof(int)));
  // rd_strang_step's once-per-step status buffers, allocated with the grid (pinned host allocations
  // are slow; the step itself then makes no allocation of its own)
  RD_CUDA_TRY(cudaMalloc(&g->r5_acc, 16 * sizeof(unsigned long long)));
  RD_CUDA_TRY(cudaMallocHost(&g->r5_host, 16 * sizeof(unsigned long long)));
  RD_CUDA_TRY(cudaMallocHost(&g->r4_host, 2 * kR4HostWords * sizeof(long long)));
  return RD_OK;
}

template <int D>
rd_status build_impl(mr_grid* g, const double* u_finest, cudaStream_t st) {
  GridDev& G = g->d;
  const int J = G.J;
  RD_CUDA_TRY(cudaMemsetAsync(G.st, ST_INTERNAL, size_t(G.off[J]), st));
  RD_CUDA_TRY(cudaMemsetAsync(G.st + G.off[J], ST_LEAF, size_t(G.off[J + 1] - G.off[J]), st));
  const int64_t NJ = G.off[J + 1] - G.off[J];
  for (int i = 0; i < G.m; ++i)
    RD_CUDA_TRY(cudaMemcpyAsync(G.val + i * G.total + G.off[J], u_finest + i * NJ, size_t(NJ) * 8,
                                cudaMemcpyDeviceToDevice, st));
  RD_TRY(significance<D>(g, st, 0));
  RD_TRY(coarsen_fixed_point<D>(g, st));
  return compact_and_compile<D>(g, st);
}


template <int D>
rd_status adapt_impl(mr_grid* g, cudaStream_t st) {
  GridDev& G = g->d;
  SecTimer tm(st);
  // H6.1/H6.2: current leaf values -> tree, projection, details, significance
  RD_CUDA_TRY(cudaMemsetAsync(G.mark, 0, size_t(G.total), st));
  k_scatter_leaves<<<nblk(G.N), kTB, 0, st>>>(G);
  RD_COUNT_LAUNCH(1);
  RD_TRY(significance<D>(g, st, 1));
  tm.mark("significance");  // (no NEW bits here: every build / adapt ends with k_check, which clears them)
  // H6.3: refinement of significant leaves, then graded repair to a fixed point
  const Thresh th = thresholds(g);
  // Fixed points are checked every second iteration: an iteration after convergence marks nothing and
  // its apply is a no-op, so the states are those of the check-every-time loop with half the host
  // round trips.
  k_refine_initial<<<nblk(G.off[G.J]), kTB, 0, st>>>(G, th, g->dflag);
  k_refine_apply<D><<<nblk(G.off[G.J]), kTB, 0, st>>>(G);  // no-op when nothing is marked
  RD_COUNT_LAUNCH(2);
  int any = 0;
  for (int it = 0;; it += 2) {
    if (it > 64 * (G.J + 1)) return RD_ESTRUCT;
    k_grade_mark<D><<<nblk(G.off[G.J]), kTB, 0, st>>>(G, g->dflag);
    k_refine_apply<D><<<nblk(G.off[G.J]), kTB, 0, st>>>(G);
    RD_CUDA_TRY(cudaMemsetAsync(g->dflag, 0, sizeof(int), st));
    k_grade_mark<D><<<nblk(G.off[G.J]), kTB, 0, st>>>(G, g->dflag);
    RD_COUNT_LAUNCH(3);
    RD_TRY(read_flag(g, 0, &any, st));
    if (!any) break;
    k_refine_apply<D><<<nblk(G.off[G.J]), kTB, 0, st>>>(G);
    RD_COUNT_LAUNCH(1);
  }
  tm.mark("refine+grade");
  // H6.4: predicted values of the new nodes, increasing level
  for (int j = 1; j <= G.J; ++j) {
    k_predict_new<D><<<nblk(int64_t(1) << (D * j)), kTB, 0, st>>>(G, j, g->dflag + 1);
    RD_COUNT_LAUNCH(1);
  }
  tm.mark("predict");  // (a stencil error raises flag 1: reported by the coarsening's read_flag)
  // H6.5: coarsening fixed point (nodes created in this call excluded), H6.6 compaction
  RD_TRY(coarsen_fixed_point<D>(g, st));
  tm.mark("coarsen");
  const rd_status rc = compact_and_compile<D>(g, st);
  tm.mark("compact+op");
  return rc;
}

void free_grid(mr_grid* g) {
  GridDev& G = g->d;
  void* ps[] = {G.st, G.mark, G.val, G.Q, G.lidx, G.iidx, G.keys, G.lev, G.u, G.nbr, G.nbrg, G.if_type, G.if_cb, G.if_fine,
                G.if_sten, G.if2_list, G.proj_cstart, G.proj_cnode, G.proj_ns, g->scr_pcnt, G.exp_start, G.exp_leaf, G.exp_w, g->r4_work, g->r4_part, g->r4_ctl, g->cub_tmp, g->dflag,
                g->scr_cnt, g->scr_off, g->scr_need, g->scr_ctr, g->scr_ccost, g->scr_cidx, G.chunk_order, g->scr_ecnt, g->lpt_cnt, g->lpt_keys, g->lpt_iota,
                g->lpt_order, g->lpt_tmp, G.m_row, G.m_slc, G.m_col, G.m_w, g->mat_cnt, g->mat_tmp, g->mat_stage, G.m_wd};
  cudaDeviceSynchronize();  // no stream of its own: the grid's pending work must finish first
  for (void* p : ps)
    if (p) cudaFreeAsync(p, 0);
  if (g->hflag) cudaFreeHost(g->hflag);
  if (g->r5_acc) cudaFree(g->r5_acc);
  if (g->r5_host) cudaFreeHost(g->r5_host);
  if (g->r4_host) cudaFreeHost(g->r4_host);
}

}  // namespace
}  // namespace rdmr

using namespace rdmr;

extern "C" rd_status mr_grid_build(const mr_params* p, int m, const double* u_finest, void* stream, mr_grid** out) {
  if (!p || !out || !u_finest || m < 1 || m > kMaxSpecies) return RD_EINVAL;
  if (p->dim != 2 && p->dim != 3) return RD_EINVAL;
  const int cap = p->dim == 2 ? 14 : 9;
  if (p->level_min < 0 || p->level_min > p->level_max || p->level_max > cap || p->level_max < 1) return RD_EINVAL;
  if (!(p->eps_mr >= 0) || (reinterpret_cast<uintptr_t>(u_finest) & 7)) return RD_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int dev = 0;
  cudaMemPool_t pool;
  uint64_t used0 = 0;
  const bool pool_ok = pool_init() == cudaSuccess && cudaGetDevice(&dev) == cudaSuccess &&
                       cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess &&
                       cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used0) == cudaSuccess;
  mr_grid* g = new mr_grid();
  rd_status rc = alloc_grid(g, p->dim, p->level_min, p->level_max, m, p->eps_mr, st);
  if (rc == RD_OK) rc = p->dim == 2 ? build_impl<2>(g, u_finest, st) : build_impl<3>(g, u_finest, st);
  if (rc != RD_OK) {
    free_grid(g);
    delete g;
    return rc;
  }
  rc = grid_reserve_step_workspace(g, st);
  if (rc != RD_OK) {
    free_grid(g);
    delete g;
    return rc;
  }
  // Pool headroom: the buffers a grid grows while it steps and adapts (and the blocks a freed grid
  // leaves behind, fragmented) would otherwise make the stream-ordered pool map new memory inside a
  // step (~80 ms once on BJ configs[3], tools/first_step.py).  One block of kPoolHeadroom x this
  // grid's build footprint is allocated and released on the grid's stream: the pool keeps it mapped
  // (release threshold unbounded) and the grid's later growth is carved from it.
  if (pool_ok) {
    constexpr uint64_t kPoolHeadroom = 6;
    uint64_t used1 = 0;
    size_t fr = 0, tot = 0;
    if (cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used1) == cudaSuccess && used1 > used0 &&
        cudaMemGetInfo(&fr, &tot) == cudaSuccess) {
      // bounded: the pool keeps what it maps, and other allocators (torch's) share the device
      const uint64_t want = std::min<uint64_t>(std::min<uint64_t>(kPoolHeadroom * (used1 - used0), fr / 8),
                                               uint64_t(16) << 30);
      void* p = nullptr;
      if (cudaMallocAsync(&p, size_t(want), st) == cudaSuccess) cudaFreeAsync(p, st);
      else cudaGetLastError();
    }
  }
  *out = g;
  return RD_OK;
}

extern "C" rd_status mr_set_operator(mr_grid* g, int mode, void* stream) {
  if (!g || mode < RD_OP_PREDICTION || mode > RD_OP_TWO_POINT_COMPACT) return RD_EINVAL;
  g->d.op_mode = mode;
  return grid_rebuild_operator(g, static_cast<cudaStream_t>(stream));  // also invalidates the matrix
}

extern "C" rd_status mr_adapt(mr_grid* g, void* stream) {
  if (!g) return RD_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  NvtxRange nvtx("mr_adapt");
  return g->d.dim == 2 ? adapt_impl<2>(g, st) : adapt_impl<3>(g, st);
}

extern "C" rd_status mr_grid_leaves(const mr_grid* g, int64_t* n, const uint64_t** keys, double** u) {
  if (!g) return RD_EINVAL;
  if (n) *n = g->d.N;
  if (keys) *keys = g->d.keys;
  if (u) *u = g->d.u;
  return RD_OK;
}

extern "C" rd_status mr_grid_info(const mr_grid* g, int64_t* n_internal, int* level_lo, int* level_hi, double* cr,
                                  double* rho1) {
  if (!g) return RD_EINVAL;
  const GridDev& G = g->d;
  if (n_internal) {
    // internal nodes at levels >= L_min (count on the dense map)
    const int64_t a = G.off[G.lmin], b = G.off[G.J + 1];
    std::vector<uint8_t> h(size_t(b - a));
    if (cudaDeviceSynchronize() != cudaSuccess) return RD_ECUDA;
    if (cudaMemcpy(h.data(), G.st + a, size_t(b - a), cudaMemcpyDeviceToHost) != cudaSuccess) return RD_ECUDA;
    int64_t c = 0;
    for (uint8_t s : h) c += (s & ST_KIND) == ST_INTERNAL;
    *n_internal = c;
  }
  if (level_lo) *level_lo = g->level_lo;
  if (level_hi) *level_hi = g->level_hi;
  if (cr) *cr = 1.0 - double(G.N) / std::ldexp(1.0, G.dim * G.J);
  if (rho1) *rho1 = g->rho1;
  return RD_OK;
}

extern "C" rd_status mr_grid_stats(const mr_grid* g, int64_t* out, int n) {
  if (!g || !out || n < 1) return RD_EINVAL;
  const int64_t v[8] = {g->d.N, g->d.n_if, g->d.n_need, g->n_exp, g->d.total, g->d.dim, g->d.J, g->d.lmin};
  for (int q = 0; q < n && q < 8; ++q) out[q] = v[q];
  return RD_OK;
}

extern "C" void mr_grid_free(mr_grid* g) {
  if (!g) return;
  free_grid(g);
  delete g;
}

extern "C" rd_status mr_rowmajor_to_morton(int dim, int level, int m, const double* src, double* dst, void* stream) {
  if ((dim != 2 && dim != 3) || level < 0 || level > (dim == 2 ? 14 : 9) || m < 1 || !src || !dst || src == dst)
    return RD_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t NJ = int64_t(1) << (dim * level);
  if (dim == 2) { k_rowmajor_to_morton2<<<nblk(NJ), kTB, 0, st>>>(level, m, src, dst); RD_COUNT_LAUNCH(1); }
  else { k_rowmajor_to_morton3<<<nblk(NJ), kTB, 0, st>>>(level, m, src, dst); RD_COUNT_LAUNCH(1); }
  RD_CUDA_TRY(cudaGetLastError());
  return RD_OK;
}

extern "C" rd_status rd_fv_apply(mr_grid* g, const double* x, double* y, void* stream) {
  if (!g || !x || !y || x == y) return RD_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (use_assembled_operator(g)) {  // the operator form the Rock4 kernel uses (rd_fv_apply is its test hook)
    RD_TRY(grid_assemble_matrix(g, assembled_launch_blocks(), st));
    if (g->mat_state == 1) return grid_mat_apply(g, x, y, st);
    if (g->d.op_mode != RD_OP_PREDICTION) return RD_ENOTSUP;
  }
  double* V = nullptr;  // [x | projections of the needed internal nodes]
  RD_CUDA_TRY(cudaMallocAsync(&V, size_t(g->d.N + g->d.n_need + 1) * 8, st));
  RD_CUDA_TRY(cudaMemcpyAsync(V, x, size_t(g->d.N) * 8, cudaMemcpyDeviceToDevice, st));
  fv_apply_launch(g->d, V, y, st);
  RD_CUDA_TRY(cudaFreeAsync(V, st));
  RD_CUDA_TRY(cudaGetLastError());
  return RD_OK;
}
