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
  uint8_t* lev;     // [N] level of each leaf (= keys >> 58; the 1-byte copy the matrix-free stage reads)
  double* u;        // [m][N]
  // FV operator (eps = 1)
  int32_t* nbr;     // [2d][N]: >= 0 same-level leaf, -1 boundary, <= -2: interface record -2-code
  int32_t* nbrg;    // [2d][N] 3-D ghost-phase form of nbr: >= -1 as nbr; -2 - 2 gi: a coarse neighbour whose
                    // ghost is gh[gi] (the linked record resolved); -3 - 2 rec: a face record with finer leaves
  int64_t n_if;
  int8_t* if_type;  // 1 coarse neighbour (ghost from L's stencil), 2 face with finer neighbours (mirror)
  int8_t* if_cb;    // type 1: child bits of the predicted cell (bit a = axis a); type 2: axis | (dir>0) << 2
  int32_t* if_fine; // type 2: [n_if][4] fine leaf indices, ordered by the bits of the other axes
  int32_t* chunk_order;  // [ceil(N / kR4Chunk)] chunks of the matrix-free Rock4 stage, most interface
                        // faces first (longest-processing-time order of the dynamic tickets)
  int32_t* if2_list;   // [n_if] the type-2 records (faces toward finer leaves), ascending: the 3-D ghost
                       // phase's work list; their count at *if2_count (device, written at operator build)
  int32_t* if2_count;
  // 3-D Rock4 projections (operator build): a needed internal node whose expansion is its 2^d children,
  // all leaves with consecutive indices inside one stage chunk ("simple") is projected by the block that
  // ran that chunk, right after writing it; proj_cstart [nch + 1] / proj_cnode list them per chunk.  The
  // other needed nodes (proj_ns, count at *proj_ns_count) go through the projection phase.
  int32_t* proj_cstart;
  int2* proj_cnode;  // (node, its first child's leaf index)
  int32_t* proj_ns;
  int32_t* proj_ns_count;
  int32_t* if_sten; // [3^d][n_if] value indices into V = [leaves | needed internal nodes], entry-major
                    // (consecutive records load coalesced); read through sten_at
  int64_t n_need;
  int32_t* exp_start;  // [n_need + 1]
  int32_t* exp_leaf;   // leaf indices
  double* exp_w;       // weights 2^{-d (l_leaf - l)}
  // The same operator assembled over leaf values only (fvmat.cu): ghost predictions and internal
  // projections folded into explicit row weights.  Sliced ELL, one warp per slice: a slice holds
  // 32/G rows with G = 1, 2, 4, 8 lanes per row (each lane <= kMatLane entries of its row, entry
  // e of a row on lane e % G), rows sorted by length inside windows of kMatWin rows.  Slice s:
  // m_slc[s] = {first position in m_row, first slot, width | nrows << 8 | log2 G << 16, 0};
  // slot (s, k, lane) at m_slc[s].y + 32 k + lane.
  int op_mode;         // RD_OP_* (mr_set_operator)
  int64_t n_slice;
  int4* m_slc;         // [n_slice]
  int32_t* m_row;      // [N] leaf rows in slice order
  int32_t* m_col;      // [slots]
  float* m_w;          // [slots] (exact: dyadic weights with short mantissas, checked at assembly)
  double* m_wd;        // [slots] FP64 weights (RD_OP_TWO_POINT)
  // RD_OP_TWO_POINT_COMPACT: m_col holds column | type << 30 (type 0 same level, 1 to coarser, 2 to
  // finer; no diagonal: a row is sum_t w_type 4^j (x_col - x_row))
};

#ifndef RD_R4_CHUNK
#define RD_R4_CHUNK 256
#endif
constexpr int kR4Chunk = RD_R4_CHUNK;  // rows per ticket of the matrix-free Rock4 stage (= its block size)
constexpr int kMatWin = 512;  // rows per length-sorting window (one block)
// weight storage of the assembled operator: 0 FP32 (prediction ghosts), 1 FP64 (two-point), 2 link
// types (two-point compact); shared-memory words per slot in the Rock4 cache
__host__ __device__ constexpr int mat_wk(int op_mode) { return op_mode; }
__host__ __device__ constexpr int mat_slot_words(int wk) { return wk == 0 ? 2 : (wk == 1 ? 3 : 1); }
// two-point coefficients divided by 4^j (reading R-T): same level 1, to the coarser leaf 2/3, to each
// finer leaf 4 / (1.5 2^d); the compact form rebuilds them from the level and the link type
// (x / 1.5 == x * fl(2/3) bit for bit when x is a power of two, so no FP64 division is needed)
__host__ __device__ inline double tp_coef(int type, int dim, int j) {
#ifdef __CUDA_ARCH__
  const double cj = __hiloint2double((1023 + 2 * j) << 20, 0);  // 4^j
#else
  const double cj = ldexp(1.0, 2 * j);
#endif
  constexpr double kTwoThirds = 2.0 / 3.0;
  return type == 0 ? cj : (type == 1 || dim == 2 ? cj * kTwoThirds : cj * (0.5 * kTwoThirds));
}
constexpr int kMatCap = 64;   // max distinct columns per assembled row (2-D max on BJ configs[2]: 50)
#ifndef RD_MAT_LANE
#define RD_MAT_LANE 8
#endif
constexpr int kMatLane = RD_MAT_LANE;  // max entries per lane: long rows are split over 2..8 lanes
#ifndef RD_MAT_WARPS
#define RD_MAT_WARPS 32
#endif
constexpr int kMatWarps = RD_MAT_WARPS;  // warps per block of the Rock4 kernel on the assembled operator

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
  // operator-build scratch (persistent, grown on demand; no allocation in the steady state)
  int32_t* scr_cnt = nullptr;
  int32_t* scr_off = nullptr;
  int64_t cap_scr = 0;
  int64_t* scr_ctr = nullptr;
  int32_t* scr_ccost = nullptr;   // [cap_chunk] chunk costs, and their sort scratch (op build)
  int32_t* scr_cidx = nullptr;
  int64_t cap_chunk = 0;  // [cap_if] stencil centre of each interface record (op build)
  int32_t* scr_pcnt = nullptr;  // [cap_chunk] per-chunk simple-node counts / cursors (op build)
  int64_t cap_proj = 0;         // capacity of proj_cnode / proj_ns (needed nodes)
  int64_t* scr_need = nullptr;
  int32_t* scr_ecnt = nullptr;
  int64_t cap_scr_need = 0;
  // longest-first order of the second reaction half step (strang.cu)
  int32_t* lpt_cnt = nullptr;
  int32_t* lpt_keys = nullptr;
  int32_t* lpt_iota = nullptr;
  int32_t* lpt_order = nullptr;
  // assembled operator (fvmat.cu); valid until the next build / adapt
  int mat_state = 0;  // 0 not built, 1 built, -1 not assemblable (row over kMatCap)
  int64_t cap_mat_wd = 0;
  int64_t cap_mat_cnt = 0, cap_mat_row = 0, cap_mat_col = 0, cap_mat_w = 0;
  int32_t* mat_cnt = nullptr;
  int4* mat_tmp = nullptr;
  int2* mat_stage = nullptr;  // [N][kMatCap] assembled rows (column, FP32 weight bits)
  int64_t cap_mat_stage = 0;
  int64_t cap_mat_tmp = 0, cap_mat_slc = 0;
  int64_t mat_slots = 0;
  int mat_blocks = 0;       // Rock4 launch the shared-memory footprint was computed for
  int mat_smem_words = 0;   // max over blocks of the slices' footprint (4-byte words)
  void* lpt_tmp = nullptr;
  size_t lpt_tmp_bytes = 0;
  int64_t cap_lpt = 0;
  // scratch
  void* cub_tmp = nullptr;
  size_t cub_bytes = 0;
  int* dflag = nullptr;        // device flags / counters
  int* hflag = nullptr;        // pinned host mirror
  // rd_strang_step's once-per-step status read: Radau5 work counter + totals (device) and their pinned
  // host copy; the Rock4 controller results of up to two launches (pinned)
  unsigned long long* r5_acc = nullptr;
  unsigned long long* r5_host = nullptr;
  long long* r4_host = nullptr;
};

namespace rdmr {
// Stencil entry q (x fastest) of interface record rec.
__device__ __forceinline__ int32_t sten_at(const GridDev& G, int64_t rec, int q) {
  return G.if_sten[int64_t(q) * G.n_if + rec];
}

// Results of a Rock4 launch whose controller statistics are read after the caller's synchronisation.
struct R4Pending {
  long long* hs = nullptr;  // pinned host [6 * kMaxSpecies + 8]
  int nsp = 0;
  cudaEvent_t ev[2] = {nullptr, nullptr};
  double rho1 = 0.0;
  int64_t mat_slots = 0;
  bool armed = false;
};
rd_status rock4_finish(R4Pending& pd, rd_stats* stats);
constexpr int kR4HostWords = 6 * kMaxSpecies + 8;

// Eq. inter_1d on one axis for child bit `bit`: u0 + (u_- - u_+)/8 (bit 0), - (bit 1).
__device__ __forceinline__ double pstep(double um, double u0, double up, int bit) {
  return u0 + (bit ? -0.125 : 0.125) * (um - up);
}

// All 2^D children of the cell whose 3^D neighbourhood is v (x fastest), tensor product x, y, z
// (P:619-621); ch[bx | by << 1 | bz << 2].
template <int D>
__device__ __forceinline__ void predict_children(const double* v, double* ch) {
  if (D == 2) {
    double r[3][2];
#pragma unroll
    for (int oy = 0; oy < 3; ++oy)
#pragma unroll
      for (int bx = 0; bx < 2; ++bx) r[oy][bx] = pstep(v[oy * 3], v[oy * 3 + 1], v[oy * 3 + 2], bx);
#pragma unroll
    for (int bx = 0; bx < 2; ++bx)
#pragma unroll
      for (int by = 0; by < 2; ++by) ch[bx | (by << 1)] = pstep(r[0][bx], r[1][bx], r[2][bx], by);
  } else {
    double r[9][2];
#pragma unroll
    for (int l = 0; l < 9; ++l)
#pragma unroll
      for (int bx = 0; bx < 2; ++bx) r[l][bx] = pstep(v[l * 3], v[l * 3 + 1], v[l * 3 + 2], bx);
    double q[3][2][2];
#pragma unroll
    for (int oz = 0; oz < 3; ++oz)
#pragma unroll
      for (int bx = 0; bx < 2; ++bx)
#pragma unroll
        for (int by = 0; by < 2; ++by) q[oz][bx][by] = pstep(r[oz * 3][bx], r[oz * 3 + 1][bx], r[oz * 3 + 2][bx], by);
#pragma unroll
    for (int bx = 0; bx < 2; ++bx)
#pragma unroll
      for (int by = 0; by < 2; ++by)
#pragma unroll
        for (int bz = 0; bz < 2; ++bz) ch[bx | (by << 1) | (bz << 2)] = pstep(q[0][bx][by], q[1][bx][by], q[2][bx][by], bz);
  }
}

// One child (bits cb) of the cell whose 3^D neighbourhood is v.
template <int D>
__device__ __forceinline__ double predict_child(const double* v, int cb) {
  if (D == 2) {
    double r[3];
#pragma unroll
    for (int oy = 0; oy < 3; ++oy) r[oy] = pstep(v[oy * 3], v[oy * 3 + 1], v[oy * 3 + 2], cb & 1);
    return pstep(r[0], r[1], r[2], (cb >> 1) & 1);
  }
  double q[3];
#pragma unroll
  for (int oz = 0; oz < 3; ++oz) {
    double r[3];
#pragma unroll
    for (int oy = 0; oy < 3; ++oy) {
      const double* w = v + (oz * 3 + oy) * 3;
      r[oy] = pstep(w[0], w[1], w[2], cb & 1);
    }
    q[oz] = pstep(r[0], r[1], r[2], (cb >> 1) & 1);
  }
  return pstep(q[0], q[1], q[2], (cb >> 2) & 1);
}

// Row r of A x (eps = 1) on V = [x (N leaves) | projections of the needed internal nodes]:
// same-level faces (x_N - x_C)/h_j^2; a face toward a coarser leaf L: (g - x_C)/h_j^2 with g the
// predicted level-j child of L adjacent to C; a face toward finer leaves F: sum_F (x_F - g_F)
// 2^{2(j+1)-D} with g_F the predicted child of C adjacent to F (the conservative mirror); boundary
// faces 0 (O.5 F1-F6).  C's 2^D children are predicted once per row.
template <int D>
__device__ __forceinline__ double fv_row(const GridDev& G, const double* V, int64_t r) {
  constexpr int NS = D == 2 ? 9 : 27;
  constexpr int NF = 1 << (D - 1);
  const int j = G.lev[r];
  const double cj = ldexp(1.0, 2 * j);
  const double xr = V[r];
  double acc = 0.0;
  double ch[1 << D];
  bool have = false;
#pragma unroll
  for (int f = 0; f < 2 * D; ++f) {
    const int32_t code = G.nbr[int64_t(f) * G.N + r];
    if (code >= 0) {
      acc += (V[code] - xr) * cj;
    } else if (code <= -2) {
      const int32_t rec = -2 - code;
      const int cb = G.if_cb[rec];
      if (G.if_type[rec] == 1) {
        double v[NS];
#pragma unroll
        for (int q = 0; q < NS; ++q) v[q] = V[sten_at(G, rec, q)];
        acc += (predict_child<D>(v, cb) - xr) * cj;
      } else {
        if (!have) {
          double v[NS];
#pragma unroll
          for (int q = 0; q < NS; ++q) v[q] = V[sten_at(G, rec, q)];
          predict_children<D>(v, ch);
          have = true;
        }
        const int a = cb & 3, bit = (cb >> 2) & 1;
        const double cf = ldexp(1.0, 2 * (j + 1) - D);
#pragma unroll
        for (int q = 0; q < NF; ++q) {
          // bits of the other axes in increasing axis order, axis a fixed to `bit`
          int cidx = 0, t = 0;
#pragma unroll
          for (int ax = 0; ax < D; ++ax) {
            int b;
            if (ax == a) b = bit;
            else { b = (q >> t) & 1; ++t; }
            cidx |= b << ax;
          }
          acc += (V[G.if_fine[int64_t(rec) * 4 + q]] - ch[cidx]) * cf;
        }
      }
    }
  }
  return acc;
}

// Values of the 3^D stencil entries sp[] for S species.  Entries >= N are internal nodes: either
// read from the V tail (filled by a projection phase) or, with `inl`, computed here from their
// projection expansion (leaf indices loaded once for all species).
template <int D, int S>
__device__ __forceinline__ void stencil_values(const GridDev& G, const double* const (&V)[S], const int32_t* sp, bool inl,
                                               double (*v)[D == 2 ? 9 : 27]) {
  constexpr int NS = D == 2 ? 9 : 27;
#pragma unroll
  for (int q = 0; q < NS; ++q) {
    const int32_t vi = sp[q];
    if (!inl || vi < G.N) {
#pragma unroll
      for (int s = 0; s < S; ++s) v[s][q] = V[s][vi];
    } else {
      const int64_t nq = vi - G.N;
      double acc[S];
#pragma unroll
      for (int s = 0; s < S; ++s) acc[s] = 0.0;
      for (int32_t e = G.exp_start[nq]; e < G.exp_start[nq + 1]; ++e) {
        const int32_t l = G.exp_leaf[e];
        const double w = G.exp_w[e];
#pragma unroll
        for (int s = 0; s < S; ++s) acc[s] += w * V[s][l];
      }
#pragma unroll
      for (int s = 0; s < S; ++s) v[s][q] = acc[s];
    }
  }
}

// fv_row for S species at once on the same row: the topology (level, face codes, interface records,
// stencil indices) is loaded once and the S value gathers are independent (memory-level
// parallelism).  out[s] = (A V_s)_r.
template <int D, int S>
__device__ __forceinline__ void fv_row_multi(const GridDev& G, const double* const (&V)[S], int64_t r, double (&out)[S],
                                             bool inl = false) {
  constexpr int NS = D == 2 ? 9 : 27;
  constexpr int NF = 1 << (D - 1);
  const int j = G.lev[r];
  const double cj = ldexp(1.0, 2 * j);
  int32_t code[2 * D];
#pragma unroll
  for (int f = 0; f < 2 * D; ++f) code[f] = G.nbr[int64_t(f) * G.N + r];
  double xr[S];
#pragma unroll
  for (int s = 0; s < S; ++s) { xr[s] = V[s][r]; out[s] = 0.0; }
#pragma unroll
  for (int f = 0; f < 2 * D; ++f) {
    if (code[f] >= 0) {
      double nb[S];
#pragma unroll
      for (int s = 0; s < S; ++s) nb[s] = V[s][code[f]];
#pragma unroll
      for (int s = 0; s < S; ++s) out[s] += (nb[s] - xr[s]) * cj;
    }
  }
#pragma unroll 1
  for (int f = 0; f < 2 * D; ++f) {
    if (code[f] > -2) continue;
    const int32_t rec = -2 - code[f];
    const int cb = G.if_cb[rec];
    int32_t sp[NS];
#pragma unroll
    for (int q = 0; q < NS; ++q) sp[q] = sten_at(G, rec, q);
    if (G.if_type[rec] == 1) {
#pragma unroll
      for (int s = 0; s < S; ++s) {
        double v[NS];
#pragma unroll
        for (int q = 0; q < NS; ++q) v[q] = V[s][sp[q]];
        out[s] += (predict_child<D>(v, cb) - xr[s]) * cj;
      }
    } else {
      const int a = cb & 3, bit = (cb >> 2) & 1;
      const double cf = ldexp(1.0, 2 * (j + 1) - D);
      int32_t fine[NF];
      int cidx[NF];
#pragma unroll
      for (int q = 0; q < NF; ++q) {
        fine[q] = G.if_fine[int64_t(rec) * 4 + q];
        int c = 0, t = 0;
#pragma unroll
        for (int ax = 0; ax < D; ++ax) {
          int b;
          if (ax == a) b = bit;
          else { b = (q >> t) & 1; ++t; }
          c |= b << ax;
        }
        cidx[q] = c;
      }
#pragma unroll
      for (int s = 0; s < S; ++s) {
        double v[NS], ch[1 << D];
#pragma unroll
        for (int q = 0; q < NS; ++q) v[q] = V[s][sp[q]];
        predict_children<D>(v, ch);
#pragma unroll
        for (int q = 0; q < NF; ++q) {
          double g = ch[0];
#pragma unroll
          for (int c = 1; c < (1 << D); ++c) g = (cidx[q] == c) ? ch[c] : g;
          out[s] += (V[s][fine[q]] - g) * cf;
        }
      }
    }
  }
}

// Ghost phase of a stage: for a face record of coarse leaf L toward finer leaves (type 2), the
// 2^{D-1} predicted children of L adjacent to that face, for S species at once (stencil indices
// loaded once).  gh[s][rec*4 + q] is read by L's row (mirror term) and by the fine leaves' rows
// (their coarse-neighbour term): each ghost is computed once, so both sides use the same value.
template <int D, int S>
__device__ __forceinline__ void ghost_record(const GridDev& G, const double* const (&V)[S], double* const (&gh)[S],
                                             int64_t rec) {
  constexpr int NS = D == 2 ? 9 : 27;
  constexpr int NF = 1 << (D - 1);
  const int cb = G.if_cb[rec];
  const int a = cb & 3, bit = (cb >> 2) & 1;
  int32_t sp[NS];
#pragma unroll
  for (int q = 0; q < NS; ++q) sp[q] = sten_at(G, rec, q);
#pragma unroll
  for (int s = 0; s < S; ++s) {
    double v[NS], ch[1 << D];
#pragma unroll
    for (int q = 0; q < NS; ++q) v[q] = V[s][sp[q]];
    predict_children<D>(v, ch);
#pragma unroll
    for (int q = 0; q < NF; ++q) {
      int c = 0, t = 0;
#pragma unroll
      for (int ax = 0; ax < D; ++ax) {
        int b;
        if (ax == a) b = bit;
        else { b = (q >> t) & 1; ++t; }
        c |= b << ax;
      }
      double g = ch[0];
#pragma unroll
      for (int cc = 1; cc < (1 << D); ++cc) g = (c == cc) ? ch[cc] : g;
      gh[s][rec * 4 + q] = g;
    }
  }
}

// Row r of A V_s for S species, ghosts read from the ghost phase's buffers gh[s].
template <int D, int S>
__device__ __forceinline__ void fv_row_ghosts(const GridDev& G, const double* const (&V)[S], const double* const (&gh)[S],
                                              int64_t r, double (&out)[S]) {
  constexpr int NF = 1 << (D - 1);
  const int j = G.lev[r];
  const double cj = ldexp(1.0, 2 * j);
  const double cf = ldexp(1.0, 2 * (j + 1) - D);
  int32_t code[2 * D];
#pragma unroll
  for (int f = 0; f < 2 * D; ++f) code[f] = G.nbrg[int64_t(f) * G.N + r];
  double xr[S];
#pragma unroll
  for (int s = 0; s < S; ++s) { xr[s] = V[s][r]; out[s] = 0.0; }
  // same-level neighbours: all 2D x S gathers are issued unconditionally (a face without one reads the
  // row's own value, which it then ignores), so they are in flight together instead of one memory
  // latency per face behind each face's branch
  double nb[S][2 * D];
#pragma unroll
  for (int f = 0; f < 2 * D; ++f) {
    const int64_t q = code[f] >= 0 ? int64_t(code[f]) : r;
#pragma unroll
    for (int s = 0; s < S; ++s) nb[s][f] = V[s][q];
  }
#pragma unroll
  for (int f = 0; f < 2 * D; ++f)
    if (code[f] >= 0)
#pragma unroll
      for (int s = 0; s < S; ++s) out[s] += (nb[s][f] - xr[s]) * cj;
#pragma unroll
  for (int f = 0; f < 2 * D; ++f) {
    const int32_t c = code[f];
    if (c >= 0) {
    } else if (c <= -2) {
      if (((-2 - c) & 1) == 0) {  // coarse neighbour: the linked ghost
        const int32_t gi = (-2 - c) >> 1;
#pragma unroll
        for (int s = 0; s < S; ++s) out[s] += (gh[s][gi] - xr[s]) * cj;
      } else {
        const int32_t rec = (-3 - c) >> 1;
        int32_t fine[NF];
#pragma unroll
        for (int q = 0; q < NF; ++q) fine[q] = G.if_fine[int64_t(rec) * 4 + q];
#pragma unroll
        for (int s = 0; s < S; ++s)
#pragma unroll
          for (int q = 0; q < NF; ++q) out[s] += (V[s][fine[q]] - gh[s][int64_t(rec) * 4 + q]) * cf;
      }
    }
  }
}

rd_status grid_rebuild_operator(mr_grid* g, cudaStream_t st);  // mr.cu
rd_status grid_assemble_matrix(mr_grid* g, int nb, cudaStream_t st);  // fvmat.cu (lazy; sets g->mat_state)
rd_status grid_reserve_step_workspace(mr_grid* g, cudaStream_t st);  // strang.cu (Rock4 stage vectors, LPT scratch, status buffers)
rd_status grid_mat_apply(mr_grid* g, const double* x, double* y, cudaStream_t st);  // fvmat.cu
bool use_assembled_operator(const mr_grid* g);  // rock4.cu: 2-D default, RDMR_R4_MODE=mat|free overrides
int assembled_launch_blocks();                  // rock4.cu: blocks of the assembled-operator Rock4 launch
void fv_apply_launch(const GridDev& G, double* V, double* y, cudaStream_t st);
}  // namespace rdmr
