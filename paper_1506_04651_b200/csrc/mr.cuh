// MR grid internals (product side).  Data layout:
//  * dense per-level node maps, levels concatenated, Morton order inside a level:
//      position p = off[j] + morton_j(k);  st[p] in {ABSENT, LEAF, INTERNAL} (+ NEW bit)
//      val[i * total + p] node values (leaf values, projections, predictions), Q[p] significance
//    O(1) neighbour / parent / children lookups instead of the paper's block store
//  * compact leaf arrays in ascending key order (level-major, Morton-minor):
//      keys[N], u[i * N + r] (SoA)
//  * FV operator topology rebuilt per adaptation: per-leaf face codes nbr[f * N + r] and
//    interface records (ghost terms, P:602-625 prediction stencils), plus projection expansions of
//    the internal nodes the ghost stencils read.
#pragma once
#include "common.cuh"

namespace rdmr {

constexpr int kMaxLevels = 16;
enum : uint8_t { ST_ABSENT = 0, ST_LEAF = 1, ST_INTERNAL = 2, ST_KIND = 3, ST_NEW = 4 };

struct GridDev {
  int dim, J, lmin, m;
  int64_t off[kMaxLevels + 2];
  int64_t total;
  uint8_t* st;
  double* val;      // [m][total]
  double* Q;        // [total]
  uint8_t* mark;    // [total]
  int32_t* lidx;    // [total] leaf index at leaf positions (after compaction)
  int32_t* iidx;    // [total] needed-internal index at needed internal positions
  int64_t N;
  uint64_t* keys;   // [N]
  double* u;        // [m][N]
  // FV operator (eps = 1)
  int32_t* nbr;     // [2d][N]: >= 0 same-level leaf, -1 boundary, <= -2: interface record -2-code
  int64_t n_if;
  int8_t* if_type;  // 1 coarse neighbour (ghost from L's stencil), 2 fine neighbour (conservative mirror)
  int8_t* if_cb;    // child bits of the predicted cell (bit a = axis a)
  int32_t* if_fine; // type 2: fine leaf index
  int32_t* if_sten; // [n_if][3^d] value indices (< N leaf, >= N needed internal N + q)
  int64_t n_need;
  int32_t* exp_start;  // [n_need + 1]
  int32_t* exp_leaf;   // leaf indices
  double* exp_w;       // weights 2^{-d (l_leaf - l)}
};

}  // namespace rdmr

struct mr_grid {
  rdmr::GridDev d;
  double eps;
  double rho1;
  int64_t cap_leaf = 0, cap_if = 0, cap_need = 0, cap_exp = 0, n_exp = 0, n_internal = 0;
  int level_lo = 0, level_hi = 0;
  // Rock4 workspace (rock4.cu)
  double* r4_work = nullptr;
  int64_t r4_cap = 0;
  double* r4_part = nullptr;
  int64_t r4_part_cap = 0;
  void* r4_ctl = nullptr;
  // scratch
  void* cub_tmp = nullptr;
  size_t cub_bytes = 0;
  int* dflag = nullptr;        // device flags / counters
  int* hflag = nullptr;        // pinned host mirror
};

namespace rdmr {
// Row r of A x (eps = 1): same-level faces (x_N - x_C)/h_j^2, coarse faces (ghost - x_C)/h_j^2,
// fine faces sum (x_F - ghost_F) 2^{2(j+1)-D}; boundary faces 0 (O.5 F1-F6).
template <int D>
__device__ __forceinline__ double fv_row(const GridDev& G, const double* x, const double* xint, int64_t r) {
  constexpr int NS = D == 2 ? 9 : 27;
  const int j = int(G.keys[r] >> kLevelShift);
  const double cj = ldexp(1.0, 2 * j);
  const double xr = x[r];
  double acc = 0.0;
#pragma unroll
  for (int f = 0; f < 2 * D; ++f) {
    const int32_t code = G.nbr[int64_t(f) * G.N + r];
    if (code >= 0) {
      acc += (x[code] - xr) * cj;
    } else if (code <= -2) {
      int32_t rec = -2 - code;
      const int ty = G.if_type[rec];
      const int nrec = ty == 1 ? 1 : (1 << (D - 1));
      for (int t = 0; t < nrec; ++t, ++rec) {
        double v[NS];
        const int32_t* sp = G.if_sten + int64_t(rec) * NS;
#pragma unroll
        for (int q = 0; q < NS; ++q) {
          const int32_t vi = sp[q];
          v[q] = vi < G.N ? x[vi] : xint[vi - G.N];
        }
        const int cb = G.if_cb[rec];
        double gh;
        if (D == 2) {
          double rr[3];
#pragma unroll
          for (int oy = 0; oy < 3; ++oy) {
            const double dl = v[oy * 3] - v[oy * 3 + 2];
            rr[oy] = v[oy * 3 + 1] + ((cb & 1) ? -0.125 : 0.125) * dl;
          }
          gh = rr[1] + (((cb >> 1) & 1) ? -0.125 : 0.125) * (rr[0] - rr[2]);
        } else {
          double qq[3];
#pragma unroll
          for (int oz = 0; oz < 3; ++oz) {
            double rr[3];
#pragma unroll
            for (int oy = 0; oy < 3; ++oy) {
              const double* w = v + (oz * 3 + oy) * 3;
              rr[oy] = w[1] + ((cb & 1) ? -0.125 : 0.125) * (w[0] - w[2]);
            }
            qq[oz] = rr[1] + (((cb >> 1) & 1) ? -0.125 : 0.125) * (rr[0] - rr[2]);
          }
          gh = qq[1] + (((cb >> 2) & 1) ? -0.125 : 0.125) * (qq[0] - qq[2]);
        }
        if (ty == 1) acc += (gh - xr) * cj;
        else acc += (x[G.if_fine[rec]] - gh) * ldexp(1.0, 2 * (j + 1) - D);
      }
    }
  }
  return acc;
}

rd_status grid_rebuild_operator(mr_grid* g, cudaStream_t st);  // mr.cu
void fv_apply_launch(const GridDev& G, const double* x, double* y, double* xint, cudaStream_t st);
}  // namespace rdmr
