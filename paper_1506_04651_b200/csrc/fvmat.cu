// The FV operator of mr.cuh assembled over LEAF values (2-D MR grids; used by the Rock4 kernel).
//
// Row r of A (eps = 1, P:324-333 with MR ghosts P:602-625, reading R-F) is linear in the leaf values:
// a same-level face contributes (x_N - x_C)/h_j^2; a ghost is the tensor-product prediction Eq.
// inter_1d of a 3^d stencil whose internal entries are projections (F6) of
// their leaf descendants.  Folding prediction weights (+-1/8, 1 per axis) and projection weights
// 2^{-d dl} into explicit coefficients gives a sparse row over leaves, so one Rock4 stage becomes one
// sparse mat-vec with no internal-value phase and no dependent topology chain (face code -> record
// -> stencil -> value): one grid barrier per stage instead of two.  All weights are dyadic rationals
// with short mantissas; they are stored as FP32 after an exactness check (else: matrix-free form).
//
// Storage: sliced ELL, one warp per slice, coalesced column/weight loads (slot (s, k, lane) at
// m_slc[s].y + 32 k + lane).  A warp's stage is as slow as its longest lane chain, and the slowest warp
// holds the grid barrier, so rows longer than kMatLane entries are split over G = 2, 4, 8 lanes
// (entry e on lane e % G, partial sums joined by G-lane shuffles).  Rows are sorted by length
// (descending) inside windows of kMatWin consecutive rows (Morton order keeps windows spatially
// compact); a slice takes 32/G rows of equal class, so padding stays small.
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "mr.cuh"

namespace rdmr {
namespace {

constexpr int kTB = 256;
inline unsigned nblk(int64_t n) { return unsigned(std::max<int64_t>(1, std::min<int64_t>((n + kTB - 1) / kTB, 1 << 20))); }

// weight of stencil offset o (0: minus, 1: centre, 2: plus) in one axis of Eq. inter_1d, child bit b
__device__ __forceinline__ double w1(int o, int b) {
  return o == 1 ? 1.0 : ((o == 0) == (b == 0) ? 0.125 : -0.125);
}
// weight of stencil entry q (x fastest) in the prediction of the child with bits cb
template <int D>
__device__ __forceinline__ double wpred(int q, int cb) {
  double w = w1(q % 3, cb & 1) * w1((q / 3) % 3, (cb >> 1) & 1);
  if (D == 3) w *= w1(q / 9, (cb >> 2) & 1);
  return w;
}

// Row assembly, one pass (k_mat_rows): a thread takes a row whose faces are all same-level or boundary
// (entries in face order, the diagonal second, so equal-kind entries of neighbouring rows share a
// slot column); a row with ghost terms is assembled by the whole warp: every lane expands some of its
// (face, stencil entry) units into leaf terms and merges them into a per-warp open-addressing table
// in shared memory (atomicCAS on the column).  Every weight of a row is 4^j times a dyadic rational
// with a short mantissa (prediction 1/8 per axis, projection 2^-d per level), so the row is summed
// EXACTLY in 32-bit fixed point, w 4^-j 2^kFix, with native integer atomics (order-independent; a
// floating-point atomicAdd would be a CAS loop spinning under contention).  Then the entries are ranked
// by column (a deterministic order) and staged as (column, FP32 weight) at stage[r * kMatCap].
#ifndef RD_ASM_WARPS
#define RD_ASM_WARPS 8
#endif
constexpr int kAsmWarps = RD_ASM_WARPS;  // warps per block of the irregular-row assembly
constexpr int kHash = 2 * kMatCap;
constexpr int kFix = 20;  // scaled weights are multiples of 2^-18 (3-D: 1/512 prediction x 2^-9 projection)

// v: the weight divided by 4^j
__device__ __forceinline__ void hash_add(int32_t* hk, int* hv, int32_t c, double v, int* over) {
  const double sv = ldexp(v, kFix);
  const int iv = __double2int_rn(sv);
  if (double(iv) != sv) atomicExch(over + 1, 1);  // not exact in the fixed-point format: matrix-free form
  uint32_t h = (uint32_t(c) * 2654435761u) >> 25;  // 7 bits: kHash = 128
  for (int probe = 0; probe < kHash; ++probe) {
    const int32_t old = atomicCAS(hk + h, -1, c);
    if (old == -1 || old == c) { atomicAdd(hv + h, iv); return; }
    h = (h + 1) & (kHash - 1);
  }
  atomicExch(over, 1);
}

template <int D>
__device__ void warp_row(const GridDev& G, int64_t r, int32_t* hk, int* hv, int2* stage, int32_t* cnt, int* over,
                         int lane) {
  constexpr int NS = D == 2 ? 9 : 27;
  constexpr int NF = 1 << (D - 1);
  for (int i = lane; i < kHash; i += 32) { hk[i] = -1; hv[i] = 0; }
  __syncwarp();
  const int j = int(G.keys[r] >> kLevelShift);
  const double cj = 1.0;                        // 4^j / 4^j: weights are accumulated divided by 4^j
  const double cf = ldexp(1.0, 2 - D);          // 2^{2(j+1)-d} / 4^j
  // units: per face 1 + NF * (1 + NS) slots: [0] same-level / diagonal term, then per fine leaf qf
  // the fine term and NS stencil entries (type 2), or NS stencil entries of L's stencil (type 1, qf = 0)
  constexpr int U = 1 + NF * (1 + NS);
  // phase 1: every lane resolves ALL its units first (the loads of different units are independent and
  // stay in flight together; interleaving them with the table atomics would serialise them)
  constexpr int UPL = (2 * D * U + 31) / 32;
  int32_t uc[UPL], uc2[UPL];  // unit leaf column (or value index >= N), second column (same-level face)
  double uw[UPL], uw2[UPL];
#pragma unroll
  for (int t = 0; t < UPL; ++t) {
    uc[t] = uc2[t] = -1;
    uw[t] = uw2[t] = 0.0;
    const int u = lane + 32 * t;
    if (u >= 2 * D * U) continue;
    const int f = u / U, k = u % U;
    const int32_t code = G.nbr[int64_t(f) * G.N + r];
    if (code == -1) continue;
    if (code >= 0) {
      if (k == 0) { uc[t] = code; uw[t] = cj; uc2[t] = int32_t(r); uw2[t] = -cj; }
      continue;
    }
    const int32_t rec = -2 - code;
    const int cb = G.if_cb[rec];
    if (G.if_type[rec] == 1) {
      if (k == 0) { uc[t] = int32_t(r); uw[t] = -cj; continue; }
      if (k > NS) continue;
      uc[t] = sten_at(G, rec, k - 1);
      uw[t] = cj * wpred<D>(k - 1, cb);
    } else {
      if (k == 0) continue;
      const int qf = (k - 1) / (1 + NS), q = (k - 1) % (1 + NS);
      if (q == 0) { uc[t] = G.if_fine[int64_t(rec) * 4 + qf]; uw[t] = cf; continue; }
      const int a = cb & 3, bit = (cb >> 2) & 1;
      int cidx = 0, tt = 0;
      for (int ax = 0; ax < D; ++ax) {
        int bb;
        if (ax == a) bb = bit;
        else { bb = (qf >> tt) & 1; ++tt; }
        cidx |= bb << ax;
      }
      uc[t] = sten_at(G, rec, q - 1);
      uw[t] = -cf * wpred<D>(q - 1, cidx);
    }
  }
  // phase 2: expansion ranges of the internal stencil entries, all units at once
  int32_t e0[UPL], e1[UPL];
#pragma unroll
  for (int t = 0; t < UPL; ++t) {
    e0[t] = e1[t] = 0;
    if (uc[t] >= G.N) {
      const int64_t qn = uc[t] - G.N;
      e0[t] = G.exp_start[qn];
      e1[t] = G.exp_start[qn + 1];
    }
  }
  // phase 3: merge into the table
#pragma unroll
  for (int t = 0; t < UPL; ++t) {
    if (uc2[t] >= 0) hash_add(hk, hv, uc2[t], uw2[t], over);
    if (uc[t] < 0) continue;
    if (uc[t] < G.N) {
      hash_add(hk, hv, uc[t], uw[t], over);
      continue;
    }
    for (int32_t e = e0[t]; e < e1[t]; e += 8) {  // loads of a batch first
      int32_t lf[8];
      double lw[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        lf[q] = e + q < e1[t] ? G.exp_leaf[e + q] : -1;
        lw[q] = e + q < e1[t] ? G.exp_w[e + q] : 0.0;
      }
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (lf[q] >= 0) hash_add(hk, hv, lf[q], uw[t] * lw[q], over);
    }
  }
  __syncwarp();
  // nonzero entries: compacted (ballot prefix) into the front of the table, then ranked by column
  int n = 0;
  int32_t ec[kHash / 32];
  int ev[kHash / 32];
#pragma unroll
  for (int t = 0; t < kHash / 32; ++t) {
    ec[t] = hk[32 * t + lane];
    ev[t] = hv[32 * t + lane];
  }
  __syncwarp();
#pragma unroll
  for (int t = 0; t < kHash / 32; ++t) {
    const bool live = ec[t] >= 0 && ev[t] != 0;
    const unsigned b = __ballot_sync(0xffffffffu, live);
    if (live) {
      const int pos = n + __popc(b & ((1u << lane) - 1));
      hk[pos] = ec[t];
      hv[pos] = ev[t];
    }
    n += __popc(b);
  }
  __syncwarp();
  const int nn = min(n, kHash);
  for (int i = lane; i < nn; i += 32) {
    const int32_t c = hk[i];
    const double w = ldexp(double(hv[i]), 2 * j - kFix);
    int rank = 0;
    for (int q = 0; q < nn; ++q) rank += hk[q] < c;
    if (rank < kMatCap) stage[r * kMatCap + rank] = make_int2(c, __float_as_int(float(w)));
    if (double(float(w)) != w) atomicExch(over + 1, 1);
  }
  if (lane == 0) {
    cnt[r] = min(n, kMatCap);  // over kMatCap: flagged, the matrix is discarded after the sort
    if (n > kMatCap) atomicExch(over, 1);
  }
  __syncwarp();
}

// Rows with only same-level / boundary faces, one thread each; the others are listed (irr, n_irr) for
// k_mat_rows_irr.
template <int D>
__global__ void k_mat_rows_reg(GridDev G, int2* stage, int32_t* cnt, int32_t* irr, int* n_irr, int* over) {
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < G.N; r += int64_t(gridDim.x) * blockDim.x) {
    int32_t code[2 * D];
    bool regular = true;
    for (int f = 0; f < 2 * D; ++f) {
      code[f] = G.nbr[int64_t(f) * G.N + r];
      regular = regular && code[f] >= -1;
    }
    if (!regular) {
      irr[atomicAdd(n_irr, 1)] = int32_t(r);  // order is irrelevant: each row is assembled on its own
      continue;
    }
    const double cj = ldexp(1.0, 2 * int(G.keys[r] >> kLevelShift));
    int n = 0, nf = 0;
    for (int f = 0; f < 2 * D; ++f)
      if (code[f] >= 0) {
        stage[r * kMatCap + n] = make_int2(code[f], __float_as_int(float(cj)));
        ++n;
        ++nf;
        if (nf == 1) ++n;  // the diagonal goes second
      }
    if (nf) stage[r * kMatCap + 1] = make_int2(int32_t(r), __float_as_int(float(-cj * nf)));
    if (double(float(cj)) != cj || double(float(-cj * nf)) != -cj * nf) atomicExch(over + 1, 1);
    cnt[r] = n;
  }
}

// Rows with ghost terms, one warp each (listed by k_mat_rows_reg).
template <int D>
__global__ void __launch_bounds__(32 * kAsmWarps) k_mat_rows_irr(GridDev G, const int32_t* irr, const int* n_irr,
                                                                 int2* stage, int32_t* cnt, int* over) {
  __shared__ int32_t s_hk[kAsmWarps][kHash];
  __shared__ int s_hv[kAsmWarps][kHash];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int n = *n_irr;
  for (int64_t i = blockIdx.x * int64_t(kAsmWarps) + wid; i < n; i += int64_t(gridDim.x) * kAsmWarps)
    warp_row<D>(G, irr[i], s_hk[wid], s_hv[wid], stage, cnt, over, lane);
}

// Two-point-flux rows (RD_OP_TWO_POINT*, reading R-T), one thread per row, no merging needed (a neighbour
// leaf touches a leaf through one face only): staged as (column, link type): 0 same level, 1 the
// coarser leaf L (centre of the type-1 record's stencil), 2 each finer leaf of a type-2 record, 3 the
// diagonal (explicit form only; the compact form sums w (x_col - x_row) and stores no diagonal).
template <int D>
__global__ void k_mat_rows_tp(GridDev G, int2* stage, int32_t* cnt, bool diag) {
  constexpr int NS = D == 2 ? 9 : 27;
  constexpr int NF = 1 << (D - 1);
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < G.N; r += int64_t(gridDim.x) * blockDim.x) {
    int n = 0;
    int2* out = stage + r * kMatCap;
    for (int f = 0; f < 2 * D; ++f) {
      const int32_t code = G.nbr[int64_t(f) * G.N + r];
      if (code >= 0) {
        out[n++] = make_int2(code, 0);
      } else if (code <= -2) {
        const int32_t rec = -2 - code;
        if (G.if_type[rec] == 1) {
          out[n++] = make_int2(sten_at(G, rec, NS / 2), 1);  // the coarse leaf itself
        } else {
          for (int q = 0; q < NF; ++q) out[n++] = make_int2(G.if_fine[int64_t(rec) * 4 + q], 2);
        }
      }
    }
    if (diag) out[n++] = make_int2(int32_t(r), 3);
    cnt[r] = n;
  }
}

constexpr int kWinSlices = 32 * kMatWin / 128;  // max slices per window (>= 4 rows per slice)
static_assert(kMatCap <= 8 * kMatLane, "rows must fit 8 lanes");

// One block per window: rows sorted by length, descending (stable), padding rows last; thread 0 cuts
// the sorted window into slices (class of the first = longest row of each slice).
__global__ void __launch_bounds__(kMatWin) k_mat_sort(int64_t N, const int32_t* cnt, int32_t* m_row, int4* tmp,
                                                      int32_t* wcnt) {
  using Sort = cub::BlockRadixSort<int, kMatWin, 1, int>;
  __shared__ typename Sort::TempStorage st;
  __shared__ int s_cnt[kMatWin];
  const int64_t w0 = blockIdx.x * int64_t(kMatWin);
  const int64_t r = w0 + threadIdx.x;
  int key[1], val[1];
  key[0] = r < N ? kMatCap - cnt[r] : kMatCap + 1;
  val[0] = r < N ? int(r) : -1;
  Sort(st).Sort(key, val, 0, 8);
  m_row[w0 + threadIdx.x] = val[0];  // blocked arrangement: thread t holds rank t
  s_cnt[threadIdx.x] = kMatCap - key[0];
  __syncthreads();
  if (threadIdx.x == 0) {
    const int nvalid = int(N - w0 < kMatWin ? N - w0 : kMatWin);
    int p = 0, ns = 0;
    while (p < nvalid) {
      const int nnz = s_cnt[p];
      int lg = 0;
      while ((kMatLane << lg) < nnz) ++lg;
      const int rows = min(32 >> lg, nvalid - p);
      const int width = (nnz + (1 << lg) - 1) >> lg;
      tmp[blockIdx.x * int64_t(kWinSlices) + ns] = make_int4(int(w0 + p), 0, width | (rows << 8) | (lg << 16), 0);
      ++ns;
      p += rows;
    }
    wcnt[blockIdx.x] = ns;
  }
}

// Slices of every window into their global order, slot counts for the offset scan, and the inverse
// map row -> 32 * slice + position in the slice.
__global__ void k_mat_slices(int64_t nwin, const int4* tmp, const int32_t* wcnt, const int32_t* woff, int4* slc,
                             int32_t* scnt, const int32_t* m_row, int32_t* inv) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < nwin * kWinSlices; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t w = i / kWinSlices;
    const int k = int(i % kWinSlices);
    if (k >= wcnt[w]) continue;
    const int4 t = tmp[i];
    const int32_t s = woff[w] + k;
    slc[s] = t;
    scnt[s] = 32 * (t.z & 0xff);
    const int rows = (t.z >> 8) & 0xff;
    for (int q = 0; q < rows; ++q) inv[m_row[t.x + q]] = 32 * s + q;
  }
}

__global__ void k_mat_setoff(int64_t ns, int4* slc, const int32_t* soff) {
  for (int64_t s = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; s < ns; s += int64_t(gridDim.x) * blockDim.x)
    slc[s].y = soff[s];
}

// One thread per row: its staged entries into the slots of its G lanes (entry e at k = e / G, lane
// q G + e % G), padded to the slice width with zero weights on the row's own column.  Lanes of rows a
// slice does not hold keep the memset zeros.
__global__ void k_mat_fill(GridDev G, const int32_t* inv, const int2* stage, const int32_t* cnt) {
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < G.N; r += int64_t(gridDim.x) * blockDim.x) {
    const int32_t p = inv[r];
    const int4 md = G.m_slc[p >> 5];
    const int q = p & 31;
    const int wdt = md.z & 0xff, lg = md.z >> 16;
    const int n = cnt[r];
    for (int e = 0; e < (wdt << lg); ++e) {
      const int64_t slot = md.y + 32 * (e >> lg) + (q << lg) + (e & ((1 << lg) - 1));
      const int2 v = e < n ? stage[r * kMatCap + e] : make_int2(int32_t(r), 0);
      G.m_col[slot] = v.x;
      G.m_w[slot] = __int_as_float(v.y);
    }
  }
}

// Two-point rows: explicit FP64 weights (wk 1; the diagonal = minus the sum of the links, summed in
// entry order) or columns tagged with the link type (wk 2, compact).  Padding: the row's own column
// with a zero weight (wk 1) or type 0 (wk 2: its term w (x_row - x_row) vanishes).
__global__ void k_mat_fill_tp(GridDev G, const int32_t* inv, const int2* stage, const int32_t* cnt, int wk) {
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < G.N; r += int64_t(gridDim.x) * blockDim.x) {
    const int32_t p = inv[r];
    const int4 md = G.m_slc[p >> 5];
    const int q = p & 31;
    const int wdt = md.z & 0xff, lg = md.z >> 16;
    const int n = cnt[r];
    const int j = int(G.keys[r] >> kLevelShift);
    double sum = 0.0;
    for (int e = 0; e < (wdt << lg); ++e) {
      const int64_t slot = md.y + 32 * (e >> lg) + (q << lg) + (e & ((1 << lg) - 1));
      const int2 v = e < n ? stage[r * kMatCap + e] : make_int2(int32_t(r), -1);
      if (wk == 2) {
        G.m_col[slot] = v.x | ((v.y < 0 ? 0 : v.y) << 30);
      } else {
        double w = 0.0;
        if (v.y >= 0 && v.y < 3) { w = tp_coef(v.y, G.dim, j); sum += w; }
        else if (v.y == 3) w = -sum;
        G.m_col[slot] = v.x;
        G.m_wd[slot] = w;
      }
    }
  }
}

// Shared-memory footprint (4-byte words) of each block's slices for the Rock4 launch with nb blocks of
// kMatWarps warps (warp gw owns slices gw, gw + nw, ...): per slice 2 words of metadata + 32 row
// indices + mat_slot_words(wk) words per slot.  Max over blocks -> need.
__global__ void k_mat_need(int64_t ns, const int4* slc, int nb, int wk, int* need) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  const int64_t nw = int64_t(nb) * kMatWarps;
  int64_t words = 0;
  for (int w = 0; w < kMatWarps; ++w)
    for (int64_t s = int64_t(b) * kMatWarps + w; s < ns; s += nw)
      words += 34 + mat_slot_words(wk) * 32 * (slc[s].z & 0xff);
  atomicMax(need, int(words < (1 << 30) ? words : (1 << 30)));
}

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

// RDMR_ADAPT_PROFILE=1: per-section wall times of the assembly (synchronises; stderr)
struct AsmTimer {
  bool on;
  cudaStream_t st;
  std::chrono::steady_clock::time_point t0;
  explicit AsmTimer(cudaStream_t s) : on(getenv("RDMR_ADAPT_PROFILE") != nullptr), st(s) {
    if (on) { cudaStreamSynchronize(st); t0 = std::chrono::steady_clock::now(); }
  }
  void mark(const char* name) {
    if (!on) return;
    cudaStreamSynchronize(st);
    const auto t1 = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[assemble] %-12s %8.1f us\n", name, std::chrono::duration<double, std::micro>(t1 - t0).count());
    t0 = t1;
  }
};

template <int D>
rd_status assemble(mr_grid* g, int nb, cudaStream_t st) {
  GridDev& G = g->d;
  AsmTimer tm(st);
  const int64_t N = G.N;
  const int64_t nwin = (N + kMatWin - 1) / kMatWin;
  const int64_t nsmax = nwin * kWinSlices;
  // mat_cnt: row lengths [N] | window slice counts [nwin + 1] | their offsets [nwin + 1]
  //          | slot counts [nsmax + 1] | slot offsets [nsmax + 1] | inverse row map [N]
  RD_TRY(grow(&g->mat_cnt, &g->cap_mat_cnt, 2 * N + 2 * (nwin + 1) + 2 * (nsmax + 1), st));
  RD_TRY(grow(&G.m_row, &g->cap_mat_row, nwin * kMatWin, st));
  RD_TRY(grow(&g->mat_tmp, &g->cap_mat_tmp, nsmax, st));
  RD_TRY(grow(&G.m_slc, &g->cap_mat_slc, nsmax, st));
  int32_t* cnt = g->mat_cnt;
  int32_t* wcnt = cnt + N;
  int32_t* woff = wcnt + nwin + 1;
  int32_t* scnt = woff + nwin + 1;
  int32_t* soff = scnt + nsmax + 1;
  int32_t* inv = soff + nsmax + 1;
  int* flag = g->dflag + 200;  // [0] row over kMatCap, [1] inexact FP32 weight, [2] smem need, [3] irregular rows
  RD_CUDA_TRY(cudaMemsetAsync(flag, 0, 4 * sizeof(int), st));
  RD_CUDA_TRY(cudaMemsetAsync(wcnt, 0, size_t(nwin + 1) * 4, st));
  RD_CUDA_TRY(cudaMemsetAsync(scnt, 0, size_t(nsmax + 1) * 4, st));
  RD_TRY(grow(&g->mat_stage, &g->cap_mat_stage, N * kMatCap, st));
  const int wk = mat_wk(G.op_mode);
  if (wk == 2 && N >= (int64_t(1) << 27)) { g->mat_state = -1; return RD_OK; }  // 30-bit columns, 27-bit cached rows
  if (wk == 0) {
    int32_t* irr = inv;  // the inverse row map is written later: its space holds the irregular-row list first
    k_mat_rows_reg<D><<<nblk(N), kTB, 0, st>>>(G, g->mat_stage, cnt, irr, flag + 3, flag);
    k_mat_rows_irr<D><<<unsigned(std::min<int64_t>((N + kAsmWarps - 1) / kAsmWarps, 148 * 16)), 32 * kAsmWarps, 0, st>>>(
        G, irr, flag + 3, g->mat_stage, cnt, flag);
  } else {
    k_mat_rows_tp<D><<<nblk(N), kTB, 0, st>>>(G, g->mat_stage, cnt, wk == 1);
  }
  RD_COUNT_LAUNCH(1);
  tm.mark("rows");
  k_mat_sort<<<unsigned(nwin), kMatWin, 0, st>>>(N, cnt, G.m_row, g->mat_tmp, wcnt);
  RD_COUNT_LAUNCH(2);
  size_t b1 = 0, b2 = 0;
  RD_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, b1, wcnt, woff, nwin + 1, st));
  RD_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, b2, scnt, soff, nsmax + 1, st));
  const size_t bytes = std::max(b1, b2);
  if (bytes > g->cub_bytes) {
    if (g->cub_tmp) rd_free(g->cub_tmp, st);
    g->cub_tmp = nullptr;
    RD_CUDA_TRY(rd_malloc(&g->cub_tmp, bytes, st));
    g->cub_bytes = bytes;
  }
  RD_CUDA_TRY(cub::DeviceScan::ExclusiveSum(g->cub_tmp, b1, wcnt, woff, nwin + 1, st));
  k_mat_slices<<<nblk(nsmax), kTB, 0, st>>>(nwin, g->mat_tmp, wcnt, woff, G.m_slc, scnt, G.m_row, inv);
  RD_CUDA_TRY(cub::DeviceScan::ExclusiveSum(g->cub_tmp, b2, scnt, soff, nsmax + 1, st));
  k_mat_setoff<<<nblk(nsmax), kTB, 0, st>>>(nsmax, G.m_slc, soff);
  RD_COUNT_LAUNCH(6);
  int32_t* h = reinterpret_cast<int32_t*>(g->hflag + 32);  // pinned
  RD_CUDA_TRY(cudaMemcpyAsync(h, woff + nwin, 4, cudaMemcpyDeviceToHost, st));
  RD_CUDA_TRY(cudaMemcpyAsync(h + 1, soff + nsmax, 4, cudaMemcpyDeviceToHost, st));
  RD_CUDA_TRY(cudaMemcpyAsync(h + 2, flag, 8, cudaMemcpyDeviceToHost, st));
  RD_CUDA_TRY(cudaStreamSynchronize(st));
  if (h[2] || h[3]) {  // a row over kMatCap distinct columns / a weight FP32 does not hold: matrix-free
    if (getenv("RDMR_MAT_DEBUG")) {  // diagnostics: row-length histogram (saturated rows count as kMatCap)
      std::vector<int32_t> hc(static_cast<size_t>(N));
      RD_CUDA_TRY(cudaMemcpy(hc.data(), cnt, size_t(N) * 4, cudaMemcpyDeviceToHost));
      int64_t hist[9] = {0}, tot = 0;
      for (int32_t c : hc) { ++hist[std::min(c / 8, 8)]; tot += c; }
      fprintf(stderr, "[mat] not assembled (over cap %d, inexact %d): N %lld, entries %lld, rows by length/8:",
              h[2], h[3], (long long)N, (long long)tot);
      for (int k = 0; k <= 8; ++k) fprintf(stderr, " %lld", (long long)hist[k]);
      fprintf(stderr, "\n");
    }
    g->mat_state = -1;
    return RD_OK;
  }
  tm.mark("sort+slices");
  G.n_slice = h[0];
  const int64_t slots = h[1];
  g->mat_slots = slots;
  RD_TRY(grow(&G.m_col, &g->cap_mat_col, slots + 1, st));
  if (wk == 0) RD_TRY(grow(&G.m_w, &g->cap_mat_w, slots + 1, st));
  if (wk == 1) RD_TRY(grow(&G.m_wd, &g->cap_mat_wd, slots + 1, st));
  RD_CUDA_TRY(cudaMemsetAsync(G.m_col, 0, size_t(slots) * 4, st));
  if (wk == 0) {
    RD_CUDA_TRY(cudaMemsetAsync(G.m_w, 0, size_t(slots) * 4, st));
    k_mat_fill<<<nblk(N), kTB, 0, st>>>(G, inv, g->mat_stage, cnt);
  } else {
    if (wk == 1) RD_CUDA_TRY(cudaMemsetAsync(G.m_wd, 0, size_t(slots) * 8, st));
    k_mat_fill_tp<<<nblk(N), kTB, 0, st>>>(G, inv, g->mat_stage, cnt, wk);
  }
  k_mat_need<<<unsigned((nb + 127) / 128), 128, 0, st>>>(G.n_slice, G.m_slc, nb, wk, flag + 2);
  RD_COUNT_LAUNCH(2);
  RD_CUDA_TRY(cudaMemcpyAsync(h, flag + 2, 4, cudaMemcpyDeviceToHost, st));
  RD_CUDA_TRY(cudaStreamSynchronize(st));
  tm.mark("fill+need");
  g->mat_blocks = nb;
  g->mat_smem_words = h[0];
  g->mat_state = 1;
  if (getenv("RDMR_MAT_DEBUG")) {  // diagnostics: slice widths and the per-warp load of the Rock4 stage
    std::vector<int4> hs(size_t(G.n_slice));
    RD_CUDA_TRY(cudaMemcpy(hs.data(), G.m_slc, hs.size() * sizeof(int4), cudaMemcpyDeviceToHost));
    const int64_t nw = int64_t(nb) * kMatWarps;
    std::vector<int64_t> wsl(size_t(nw), 0), wsum(size_t(nw), 0), wrows(size_t(nw), 0);
    int64_t hist[33] = {0};
    for (int64_t q = 0; q < G.n_slice; ++q) {
      const int wdt = hs[q].z & 0xff, nr = (hs[q].z >> 8) & 0xff;
      ++wsl[q % nw]; wsum[q % nw] += wdt; wrows[q % nw] += nr;
      ++hist[std::min(wdt, 32)];
    }
    int64_t msl = 0, msum = 0, tsum = 0, mrows = 0;
    for (int64_t w = 0; w < nw; ++w) {
      msl = std::max(msl, wsl[w]); msum = std::max(msum, wsum[w]); tsum += wsum[w]; mrows = std::max(mrows, wrows[w]);
    }
    fprintf(stderr, "[mat] N %lld slices %lld warps %lld slots %lld | slices/warp max %lld avg %.2f | sum wdt/warp max %lld avg %.2f | rows/warp max %lld avg %.1f\n[mat] wdt hist:",
            (long long)N, (long long)G.n_slice, (long long)nw, (long long)slots, (long long)msl, double(G.n_slice) / nw,
            (long long)msum, double(tsum) / nw, (long long)mrows, double(N) / nw);
    for (int k = 0; k <= 32; ++k)
      if (hist[k]) fprintf(stderr, " %d:%lld", k, (long long)hist[k]);
    fprintf(stderr, "\n");
  }
  return RD_OK;
}

// y = A x with the assembled operator (rd_fv_apply in the assembled form): warp per slice, G lanes per
// row joined by shuffles, as in the Rock4 stage.
__global__ void k_mat_apply(GridDev G, const double* x, double* y) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5, nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t sl = w0; sl < G.n_slice; sl += nw) {
    const int4 md = G.m_slc[sl];
    const int wdt = md.z & 0xff, nrows = (md.z >> 8) & 0xff, lg = md.z >> 16;
    const int q = lane >> lg;
    const int32_t r = q < nrows ? G.m_row[md.x + q] : -1;
    double a = 0.0;
    const int wk = mat_wk(G.op_mode);
    if (r >= 0) {
      const int j = wk == 2 ? int(G.keys[r] >> kLevelShift) : 0;
      const double xr = wk == 2 ? x[r] : 0.0;
      for (int e = 0; e < wdt; ++e) {
        const int32_t c = G.m_col[md.y + 32 * e + lane];
        if (wk == 0) a = fma(double(G.m_w[md.y + 32 * e + lane]), x[c], a);
        else if (wk == 1) a = fma(G.m_wd[md.y + 32 * e + lane], x[c], a);
        else a = fma(tp_coef(int(uint32_t(c) >> 30), G.dim, j), x[c & 0x3fffffff] - xr, a);
      }
    }
    for (int o = 1; o < (1 << lg); o <<= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (r >= 0 && (lane & ((1 << lg) - 1)) == 0) y[r] = a;
  }
}

}  // namespace

rd_status grid_mat_apply(mr_grid* g, const double* x, double* y, cudaStream_t st) {
  if (g->mat_state != 1) return RD_ENOTSUP;
  k_mat_apply<<<nblk(g->d.n_slice * 32), kTB, 0, st>>>(g->d, x, y);
  RD_COUNT_LAUNCH(1);
  RD_CUDA_TRY(cudaGetLastError());
  return RD_OK;
}

rd_status grid_assemble_matrix(mr_grid* g, int nb, cudaStream_t st) {
  if (g->mat_state == -1 || (g->mat_state == 1 && g->mat_blocks == nb)) return RD_OK;
  if (g->d.N == 0) { g->mat_state = -1; return RD_OK; }
  return g->d.dim == 2 ? assemble<2>(g, nb, st) : assemble<3>(g, nb, st);
}

}  // namespace rdmr
