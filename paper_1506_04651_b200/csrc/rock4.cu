// Diffusion substep: Rock4 on the MR leaves (readings R-K1..R-K5 =
// SURVEY §8(c) O.4), matrix-free with the FV operator of mr.cuh (ghosts by MR prediction).
//
// ONE persistent cooperative kernel integrates every species over [0, T]: species are independent
// and run in lock step, each with its own program counter (step size, stage count,
// stage index).  One grid-wide barrier separates the ghost-internal-value phase (projection
// expansions of the internal nodes the ghost stencils read) from the stage phase, and one ends the
// stage phase; the step controller (accept/reject, next h and s, "one scalar product per
// time step") runs redundantly in every block on the same block-partial error sums in the same order,
// so all blocks take identical decisions with no host round trip and no extra barrier.
//
// Stage program of one step with s stages (n = s - 4 recurrence stages + 4 finishing stages):
//   g_0 = x;  g_{k+1} = mu_k hA g_k + nu_k g_k + kappa_k g_{k-1}            (k < n)
//   finishing with the POWER basis p_q = (hA)^q y, y = g_n:  x_{n+1} = y + sum_q sigma_q p_q and
//   the embedded error e = sigma_4 p_4 from the same 4 matvecs (Horner + separate error chain would
//   cost 8; P:962-994 evaluates w by Horner).
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "mr.cuh"
#ifndef RD_ROCK4_TABLE
#define RD_ROCK4_TABLE "rock4_coeffs.inc"
#endif
#include RD_ROCK4_TABLE

namespace cg = cooperative_groups;

namespace rdmr {
namespace {

constexpr int kR4Threads = 256;
constexpr int kNsteps = RD_ROCK4_SMAX - 4;
__constant__ double c_ell[kNsteps];
__constant__ double c_sig[kNsteps][4];
__constant__ int c_off[kNsteps + 1];
double* g_rec = nullptr;  // device copy of kRock4Rec
bool g_tables = false;

rd_status tables() {
  if (g_tables) return RD_OK;
  RD_CUDA_TRY(cudaMemcpyToSymbol(c_ell, kRock4Ell, sizeof(kRock4Ell)));
  RD_CUDA_TRY(cudaMemcpyToSymbol(c_sig, kRock4Sig, sizeof(kRock4Sig)));
  RD_CUDA_TRY(cudaMemcpyToSymbol(c_off, kRock4Off, sizeof(kRock4Off)));
  RD_CUDA_TRY(cudaMalloc(&g_rec, sizeof(kRock4Rec)));
  RD_CUDA_TRY(cudaMemcpy(g_rec, kRock4Rec, sizeof(kRock4Rec), cudaMemcpyHostToDevice));
  g_tables = true;
  return RD_OK;
}

struct R4Spec {
  double* buf[5];  // stage vectors, each [N + n_need]: V = [leaf values | needed internal values];
                   // 0: state, 1..3: recurrence, 4: spare state / x_acc
  double* u;       // the species' leaf values in the grid (or the forced-step input)
  double* gh;      // ghost values [n_if * 4] of the current stage (ghost phase)
  double eps;
};

struct R4Params {
  GridDev G;
  int nsp;
  R4Spec sp[kMaxSpecies];
  double T, rtol, atol, rho1;
  int smax;
  const double* rec;
  double* part;       // [nsp][n_chunks]: error square sums per chunk of rows
  long long* stats;   // [nsp][6]: steps, rejects, matvecs, s_min, s_max, failed; then [1]: rounds
  unsigned int* tick; // [4] chunk tickets (round-robin slots)
  int ticket_chunks;  // chunks per ticket (~6 tickets per block per round)
  int forced;         // 1: one step with (forced_s, forced_h), outputs to out/err
  int forced_s;
  double forced_h;
  double* out;
  double* err;
};

enum : int { OP_REC = 0, OP_P1 = 1, OP_P2 = 2, OP_P3 = 3, OP_P4 = 4, OP_DONE = 5 };

struct Ctl {
  double t, h, he;
  int s, k, op, last, rejprev, xcur;
  int in, prev, out, xacc;
  double c0, c1, c2;  // mu, nu, kappa (REC) / sigma_q (P1..P4)
  long long steps, rejects, matvecs;
  int smin, smaxs, failed;
};

__device__ void start_step(Ctl& c, const R4Params& P, double rho) {
  c.last = 0;
  const double ellmax = c_ell[P.smax - 5];
  if (P.forced) {
    c.h = P.forced_h;
    c.s = P.forced_s;
    c.last = 1;
  } else {
    if (c.h * rho > ellmax) c.h = ellmax / rho;
    if (c.t + c.h >= P.T) { c.h = P.T - c.t; c.last = 1; }
    int s = 5;  // K3: s = min{s >= 5 : ell_s >= h rho}
    while (s < P.smax && c_ell[s - 5] < c.h * rho) ++s;
    c.s = s;
  }
  c.smin = c.smin ? min(c.smin, c.s) : c.s;
  c.smaxs = max(c.smaxs, c.s);
  c.k = 0;
  c.op = OP_REC;
}

// Buffer assignment and coefficients of the current op (Ctl.op, Ctl.k).
__device__ void set_op(Ctl& c, const R4Params& P) {
  const int n = c.s - 4;
  const int R[3] = {1, 2, 3};
  if (c.op == OP_REC) {
    const int k = c.k;
    c.in = k == 0 ? c.xcur : R[(k - 1) % 3];
    c.prev = k <= 1 ? c.xcur : R[(k - 2) % 3];
    c.out = R[k % 3];
    const double* r = P.rec + 3 * (c_off[c.s - 5] + k);
    c.c0 = r[0]; c.c1 = r[1]; c.c2 = r[2];
  } else {
    const int y = R[(n - 1) % 3];
    const int f1 = y == 1 ? 2 : 1, f2 = (y == 3) ? 2 : 3;
    c.xacc = c.xcur == 0 ? 4 : 0;
    if (c.op == OP_P1) { c.in = y; c.out = f1; }
    else if (c.op == OP_P2) { c.in = f1; c.out = f2; }
    else if (c.op == OP_P3) { c.in = f2; c.out = f1; }
    else { c.in = f1; c.out = -1; }
    c.prev = y;
    c.c0 = c_sig[c.s - 5][c.op - 1];
  }
}


#ifndef RD_R4_MINB2
#define RD_R4_MINB2 2
#endif
#ifndef RD_R4_MINB3
#define RD_R4_MINB3 2
#endif
#ifndef RD_R4_TIMING
#define RD_R4_TIMING 0
#endif
#if RD_R4_TIMING
#define R4T(slot) do { if (tid == 0) { const long long c_ = clock64(); tacc[slot] += c_ - tlast; tlast = c_; } } while (0)
#else
#define R4T(slot) do { } while (0)
#endif
#ifndef RD_R4_INLINE_PROJ
#define RD_R4_INLINE_PROJ 0
#endif
// 1: internal stencil values are projected inline in the stage phase (one grid barrier per round);
// 0: a separate projection phase fills the V tails (two barriers per round).
constexpr bool kInlineProj = RD_R4_INLINE_PROJ != 0;

// Ghost values in a separate phase (computed once per coarse face, one more grid barrier per round) vs
// predicted per row inside the stage phase: measured better for 3-D (27-point stencils, 4 fine leaves
// per face: ~100 vs ~130 us per round on cfg 4), worse for 2-D (~23.5 vs ~20.8 us on cfg 3).
template <int D>
constexpr bool kGhostPhase = (D == 3);

// Ghost phase for record rec and a group of S active species (their current op inputs).
template <int D, int S>
__device__ __forceinline__ void ghost_group(const R4Params& P, const Ctl* ctl, const int* act, int g0, int64_t rec) {
  const double* V[S];
  double* gh[S];
#pragma unroll
  for (int s = 0; s < S; ++s) {
    V[s] = P.sp[act[g0 + s]].buf[ctl[act[g0 + s]].in];
    gh[s] = P.sp[act[g0 + s]].gh;
  }
  ghost_record<D, S>(P.G, V, gh, rec);
}

// One row r for a group of S active species (act[g0 .. g0+S)): matvec with shared topology, then
// each species' stage combination.  P4 error partials go to red[warp][species].
template <int D, int S>
__device__ __forceinline__ void stage_group(const R4Params& P, const Ctl* ctl, const int* act, int g0, int64_t r,
                                            double (*red)[kMaxSpecies]) {
  const GridDev& G = P.G;
  const double* V[S];
  const double* gh[S];
#pragma unroll
  for (int s = 0; s < S; ++s) {
    V[s] = P.sp[act[g0 + s]].buf[ctl[act[g0 + s]].in];
    gh[s] = P.sp[act[g0 + s]].gh;
  }
  double a[S];
  const bool live = r < G.N;
  if (live) {
    if constexpr (kGhostPhase<D>) fv_row_ghosts<D, S>(G, V, gh, r, a);
    else fv_row_multi<D, S>(G, V, r, a, kInlineProj);
  }
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int i = act[g0 + s];
    const Ctl& c = ctl[i];
    double part = 0.0;
    if (live) {
      const double ah = c.he * a[s];
      if (c.op == OP_REC) {
        P.sp[i].buf[c.out][r] = c.c0 * ah + c.c1 * V[s][r] + c.c2 * P.sp[i].buf[c.prev][r];
      } else if (c.op != OP_P4) {
        double* xacc = P.sp[i].buf[c.xacc];
        P.sp[i].buf[c.out][r] = ah;
        xacc[r] = (c.op == OP_P1 ? P.sp[i].buf[c.prev][r] : xacc[r]) + c.c0 * ah;
      } else {
        double* xacc = P.sp[i].buf[c.xacc];
        const double e = c.c0 * ah;
        const double xn = xacc[r] + e;
        xacc[r] = xn;
        const double sc = P.atol + P.rtol * fmax(fabs(P.sp[i].buf[c.xcur][r]), fabs(xn));
        const double q = e / sc;
        part = q * q;
        if (P.forced) { P.out[r] = xn; P.err[r] = e; }
      }
    }
    if (c.op == OP_P4) {  // block-uniform branch
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
      if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5][i] = part;
    }
  }
}

template <int D>
__global__ void __launch_bounds__(kR4Threads, D == 2 ? RD_R4_MINB2 : RD_R4_MINB3) k_rock4(R4Params P) {
  cg::grid_group grid = cg::this_grid();
  __shared__ Ctl ctl[kMaxSpecies];
  __shared__ double red[kR4Threads / 32];
  __shared__ double redsp[kR4Threads / 32][kMaxSpecies];
  __shared__ int s_act[kMaxSpecies];
  __shared__ int s_nact, s_anyp4;
  __shared__ int s_active;
  __shared__ double errsq[kMaxSpecies];
  __shared__ unsigned int s_ticket;
  __shared__ int s_round;
  const int tid = threadIdx.x;
  const int64_t gtid = blockIdx.x * int64_t(blockDim.x) + tid;
  const int64_t gstride = int64_t(gridDim.x) * blockDim.x;
  const GridDev& G = P.G;
  const int64_t nch = (G.N + kR4Threads - 1) / kR4Threads;
  const int kTicketChunks = P.ticket_chunks;  // chunks of kR4Threads rows per ticket
  const int64_t ntk = (nch + kTicketChunks - 1) / kTicketChunks;

  if (tid < P.nsp) {
    Ctl c{};
    c.t = 0.0;
    c.h = P.T;
    c.xcur = 0;
    start_step(c, P, P.sp[tid].eps * P.rho1);
    c.he = c.h * P.sp[tid].eps;
    set_op(c, P);
    ctl[tid] = c;
  }
  if (tid == 0) s_round = 0;
#if RD_R4_TIMING
  long long tacc[6] = {0, 0, 0, 0, 0, 0};  // A, barA, B, barB, ctl, ghost phase + barrier
  long long tlast = clock64();
#endif
  __syncthreads();
  if (tid == 0) {
    int n = 0, p4 = 0;
    for (int i = 0; i < P.nsp; ++i)
      if (ctl[i].op != OP_DONE) { s_act[n++] = i; p4 |= ctl[i].op == OP_P4; }
    s_nact = n;
    s_anyp4 = p4;
  }
  // state -> slack buffer 0
  for (int i = 0; i < P.nsp; ++i)
    for (int64_t r = gtid; r < G.N; r += gstride) P.sp[i].buf[0][r] = P.sp[i].u[r];
  __syncthreads();
  grid.sync();

  while (true) {
    // ---- phase A: projections of the needed internal nodes of each op's input vector (V tail)
    if (!kInlineProj && G.n_need > 0) {
      for (int i = 0; i < P.nsp; ++i) {
        const Ctl& c = ctl[i];
        if (c.op == OP_DONE) continue;
        double* V = P.sp[i].buf[c.in];
        for (int64_t q = gtid; q < G.n_need; q += gstride) {
          double acc = 0.0;
          const int32_t e1 = G.exp_start[q + 1];
          for (int32_t e = G.exp_start[q]; e < e1; ++e) acc += G.exp_w[e] * V[G.exp_leaf[e]];
          V[G.N + q] = acc;
        }
      }
      R4T(0);
      grid.sync();
      R4T(1);
    }
    // ---- phase G: ghost values (predicted children of coarse leaves at their finer faces), once per
    //      face record for all active species
    if (kGhostPhase<D> && G.n_if > 0) {
      const int nact = s_nact;
      for (int64_t rec = gtid; rec < G.n_if; rec += gstride) {
        if (G.if_type[rec] != 2) continue;
        int g0 = 0;
        for (; g0 + 3 <= nact; g0 += 3) ghost_group<D, 3>(P, ctl, s_act, g0, rec);
        if (nact - g0 == 2) ghost_group<D, 2>(P, ctl, s_act, g0, rec);
        else if (nact - g0 == 1) ghost_group<D, 1>(P, ctl, s_act, g0, rec);
      }
      grid.sync();
    }
    R4T(5);
    // ---- phase B: one stage (matvec + combination) for every active species.  A thread evaluates a
    //      row for all species at once (the topology is loaded once per row).  Rows are handed out by
    //      an atomic ticket (P.ticket_chunks chunks of kR4Threads rows; the next ticket is prefetched)
    //      so blocks that draw interface-heavy chunks (they cluster in Morton order) do not hold the
    //      barrier back.  Each chunk's error partial has its own slot -> fixed reduction order.
    {
      const int slot = s_round & 3;
      if (blockIdx.x == 0 && tid == 0) P.tick[(s_round + 2) & 3] = 0u;  // last used 2 rounds ago
      const int nact = s_nact, anyp4 = s_anyp4;
      unsigned int next = 0;
      if (tid == 0) next = atomicAdd(P.tick + slot, 1u);
      while (true) {
        if (tid == 0) s_ticket = next;
        __syncthreads();
        const int64_t t = s_ticket;
        __syncthreads();
        if (t >= ntk) break;
        if (tid == 0) next = atomicAdd(P.tick + slot, 1u);  // prefetch the next ticket
        const int64_t ch0 = t * kTicketChunks;
        for (int64_t chunk = ch0; chunk < ch0 + kTicketChunks && chunk < nch; ++chunk) {
          const int64_t r = chunk * kR4Threads + tid;
          int g0 = 0;
          for (; g0 + 3 <= nact; g0 += 3) stage_group<D, 3>(P, ctl, s_act, g0, r, redsp);
          if (nact - g0 == 2) stage_group<D, 2>(P, ctl, s_act, g0, r, redsp);
          else if (nact - g0 == 1) stage_group<D, 1>(P, ctl, s_act, g0, r, redsp);
          if (anyp4) {
            __syncthreads();
            if (tid < P.nsp && ctl[tid].op == OP_P4) {
              double sm = 0.0;
              for (int w = 0; w < kR4Threads / 32; ++w) sm += redsp[w][tid];
              P.part[int64_t(tid) * nch + chunk] = sm;
            }
            __syncthreads();
          }
        }
      }
    }
    R4T(2);
    grid.sync();
    R4T(3);
    // ---- error norms of the species that just finished a step: the whole block sums the chunk
    //      partials (fixed thread -> chunk assignment, fixed shuffle/smem tree: identical in every
    //      block).  s_act / ctl[].op are stable here: the controller only runs after the final sync.
    for (int a = 0; a < s_nact; ++a) {
      const int i = s_act[a];
      if (ctl[i].op != OP_P4) continue;
      double acc = 0.0;
      for (int64_t b = tid; b < nch; b += kR4Threads) acc += P.part[int64_t(i) * nch + b];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if ((tid & 31) == 0) red[tid >> 5] = acc;
      __syncthreads();
      if (tid == 0) {
        double t2 = 0.0;
        for (int w = 0; w < kR4Threads / 32; ++w) t2 += red[w];
        errsq[i] = t2;
      }
      __syncthreads();
    }
    __syncthreads();
    // ---- step control, redundantly in every block (identical inputs => identical decisions)
    if (tid < P.nsp) {
      Ctl c = ctl[tid];
      if (c.op != OP_DONE) {
        c.matvecs++;
        if (c.op == OP_REC) {
          if (++c.k >= c.s - 4) c.op = OP_P1;
        } else if (c.op < OP_P4) {
          c.op++;
        } else {
          const double err = sqrt(errsq[tid] / double(G.N > 0 ? G.N : 1));
          const double fac = err > 0.0 ? fmin(5.0, fmax(0.1, 0.8 / sqrt(sqrt(err)))) : 5.0;
          if (P.forced) {
            c.op = OP_DONE;
            c.steps++;
          } else if (err <= 1.0) {  // K5 accept
            c.steps++;
            c.xcur = c.xacc;
            if (c.last) {
              c.op = OP_DONE;
            } else {
              c.t += c.h;
              double hn = c.h * fac;
              if (c.rejprev) hn = fmin(hn, c.h);
              c.rejprev = 0;
              c.h = hn;
            }
          } else {
            c.rejects++;
            c.rejprev = 1;
            c.h = c.h * fac;
            if (c.rejects > 100000) { c.failed = 1; c.op = OP_DONE; }
          }
          if (c.op != OP_DONE) {
            start_step(c, P, P.sp[tid].eps * P.rho1);
            c.he = c.h * P.sp[tid].eps;
          }
        }
        if (c.op != OP_DONE) set_op(c, P);
      }
      ctl[tid] = c;
    }
    __syncthreads();
    if (tid == 0) {
      int n = 0, p4 = 0;
      for (int i = 0; i < P.nsp; ++i)
        if (ctl[i].op != OP_DONE) { s_act[n++] = i; p4 |= ctl[i].op == OP_P4; }
      s_nact = n;
      s_anyp4 = p4;
      s_active = n > 0;
    }
    if (tid == 0) ++s_round;
    __syncthreads();
    R4T(4);
    if (!s_active) break;
  }
  // final state back into the grid's leaf array
  for (int i = 0; i < P.nsp; ++i) {
    if (P.forced) continue;
    const double* src = P.sp[i].buf[ctl[i].xcur];
    double* dst = P.sp[i].u;
    for (int64_t r = gtid; r < G.N; r += gstride) dst[r] = src[r];
  }
  if (blockIdx.x == 0 && tid == 0) P.stats[6 * P.nsp] = s_round;
#if RD_R4_TIMING
  if (blockIdx.x == 0 && tid == 0)
    for (int q = 0; q < 6; ++q) P.stats[6 * P.nsp + 1 + q] = tacc[q];
#endif
  if (blockIdx.x == 0 && tid < P.nsp) {
    const Ctl& c = ctl[tid];
    long long* s = P.stats + 6 * tid;
    s[0] = c.steps; s[1] = c.rejects; s[2] = c.matvecs; s[3] = c.smin; s[4] = c.smaxs; s[5] = c.failed;
  }
}

rd_status run_rock4(mr_grid* g, const std::vector<int>& species, const std::vector<double>& eps, double T,
                    const rd_rock4_opts& o, int forced, int fs, double fh, const double* fx, double* out,
                    double* err, rd_stats* stats, cudaStream_t st) {
  RD_TRY(tables());
  GridDev& G = g->d;
  const int nsp = int(species.size());
  if (nsp == 0 || G.N == 0) return RD_OK;
  // workspace: 5 stage vectors of [N + n_need] per species (V = [leaves | needed internal nodes])
  const int64_t vl = G.N + G.n_need + 1;
  const int64_t gl = 4 * G.n_if + 4;
  const int64_t per = 5 * vl + gl;
  const int64_t need = per * nsp;
  if (need > g->r4_cap) {
    if (g->r4_work) cudaFree(g->r4_work);
    g->r4_work = nullptr;
    const int64_t c = need + need / 4;
    RD_CUDA_TRY(cudaMalloc(&g->r4_work, size_t(c) * 8));
    g->r4_cap = c;
  }
  int dev = 0, nsm = 0, occ = 0;
  RD_CUDA_TRY(cudaGetDevice(&dev));
  RD_CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  void* fn = G.dim == 2 ? (void*)k_rock4<2> : (void*)k_rock4<3>;
  RD_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kR4Threads, 0));
  if (occ < 1) return RD_ECUDA;
  int bps = 2;
  if (const char* e = getenv("RDMR_R4_BPS")) bps = std::max(1, atoi(e));
  int64_t blocks = std::min<int64_t>(int64_t(nsm) * std::min(occ, bps),
                                     std::max<int64_t>(1, (G.N + kR4Threads - 1) / kR4Threads));
  const int64_t nch = (G.N + kR4Threads - 1) / kR4Threads;
  const int64_t npart = int64_t(nsp) * nch;
  if (npart + 6 * kMaxSpecies + 64 > g->r4_part_cap) {
    if (g->r4_part) cudaFree(g->r4_part);
    g->r4_part = nullptr;
    RD_CUDA_TRY(cudaMalloc(&g->r4_part, size_t(npart + 6 * kMaxSpecies + 64) * 8));
    g->r4_part_cap = npart + 6 * kMaxSpecies + 64;
  }
  R4Params P;
  P.G = G;
  P.nsp = nsp;
  for (int q = 0; q < nsp; ++q) {
    const int i = species[q];
    double* w = g->r4_work + per * q;
    for (int b = 0; b < 5; ++b) P.sp[q].buf[b] = w + b * vl;
    P.sp[q].gh = w + 5 * vl;
    P.sp[q].u = forced ? const_cast<double*>(fx) : G.u + int64_t(i) * G.N;
    P.sp[q].eps = eps[q];
  }
  P.T = T; P.rtol = o.rtol; P.atol = o.atol; P.rho1 = g->rho1;
  P.smax = std::min(o.s_max, RD_ROCK4_SMAX);
  P.rec = g_rec;
  P.part = g->r4_part;
  P.stats = reinterpret_cast<long long*>(g->r4_part + npart);
  P.tick = reinterpret_cast<unsigned int*>(P.stats + 6 * kMaxSpecies + 8);
  RD_CUDA_TRY(cudaMemsetAsync(P.tick, 0, 4 * sizeof(unsigned int), st));
  P.ticket_chunks = int(std::max<int64_t>(1, std::min<int64_t>(8, nch / (blocks * 4))));
  if (const char* e = getenv("RDMR_R4_TC")) P.ticket_chunks = std::max(1, atoi(e));
  P.forced = forced; P.forced_s = fs; P.forced_h = fh; P.out = out; P.err = err;
  void* args[] = {&P};
  RD_CUDA_TRY(cudaLaunchCooperativeKernel(fn, dim3(unsigned(blocks)), dim3(kR4Threads), args, 0, st));
  RD_COUNT_LAUNCH(1);
  long long hs[6 * kMaxSpecies + 8];
  RD_CUDA_TRY(cudaMemcpyAsync(hs, P.stats, sizeof(long long) * (6 * nsp + 7), cudaMemcpyDeviceToHost, st));
  RD_CUDA_TRY(cudaStreamSynchronize(st));
  bool failed = false;
  for (int q = 0; q < nsp; ++q) {
    const long long* s = hs + 6 * q;
    failed = failed || s[5];
    if (stats) {
      stats->rock4_steps += s[0];
      stats->rock4_rejects += s[1];
      stats->rock4_matvecs += s[2];
      stats->rock4_s_min = stats->rock4_s_min ? std::min<int64_t>(stats->rock4_s_min, s[3]) : s[3];
      stats->rock4_s_max = std::max<int64_t>(stats->rock4_s_max, s[4]);
    }
  }
  if (stats) {
    stats->rho1 = g->rho1;
    stats->rock4_rounds += hs[6 * nsp];
  }
#if RD_R4_TIMING
  std::fprintf(stderr, "[rock4 timing block0, cycles] phaseA %lld barA %lld ghosts+bar %lld phaseB %lld barB %lld ctl %lld rounds %lld\n",
               hs[6 * nsp + 1], hs[6 * nsp + 2], hs[6 * nsp + 6], hs[6 * nsp + 3], hs[6 * nsp + 4], hs[6 * nsp + 5], hs[6 * nsp]);
#endif
  return failed ? RD_ESTIFF : RD_OK;
}

}  // namespace

rd_status diffusion_rock4(mr_grid* g, const double* eps_diff, double T, const rd_rock4_opts* opts, rd_stats* stats,
                          cudaStream_t st) {
  rd_rock4_opts o{1e-8, 1e-8, 200};
  if (opts) o = *opts;
  if (!g || !eps_diff || !(T > 0) || !(o.rtol > 0) || !(o.atol > 0) || o.s_max < 5) return RD_EINVAL;
  std::vector<int> sp;
  std::vector<double> ep;
  for (int i = 0; i < g->d.m; ++i) {
    if (!(eps_diff[i] >= 0)) return RD_EINVAL;
    if (eps_diff[i] > 0) { sp.push_back(i); ep.push_back(eps_diff[i]); }  // eps = 0: D is the identity
  }
  return run_rock4(g, sp, ep, T, o, 0, 0, 0.0, nullptr, nullptr, nullptr, stats, st);
}

}  // namespace rdmr

using namespace rdmr;

extern "C" rd_status rd_diffusion_rock4(mr_grid* g, const double* eps_diff, double T, const rd_rock4_opts* opts,
                                        rd_stats* stats, void* stream) {
  return diffusion_rock4(g, eps_diff, T, opts, stats, static_cast<cudaStream_t>(stream));
}

extern "C" rd_status rd_rock4_forced_step(mr_grid* g, const double* x, double eps, double h, int s, double* out,
                                          double* err, void* stream) {
  if (!g || !x || !out || s < 5 || s > RD_ROCK4_SMAX || !(h > 0) || !(eps > 0)) return RD_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double* e = err;
  if (!e) RD_CUDA_TRY(cudaMallocAsync(&e, size_t(std::max<int64_t>(g->d.N, 1)) * 8, st));
  rd_rock4_opts o{1e-8, 1e-8, RD_ROCK4_SMAX};
  rd_status rc = run_rock4(g, {0}, {eps}, h, o, 1, s, h, x, out, e, nullptr, st);
  if (!err) cudaFreeAsync(e, st);
  return rc;
}

extern "C" int rd_rock4_smax(void) { return RD_ROCK4_SMAX; }

extern "C" rd_status rd_rock4_coeffs(int s, double* ell, double* sigma4, double* mu, double* nu, double* kappa) {
  if (s < 5 || s > RD_ROCK4_SMAX) return RD_EINVAL;
  const int i = s - 5;
  if (ell) *ell = kRock4Ell[i];
  for (int q = 0; q < 4 && sigma4; ++q) sigma4[q] = kRock4Sig[i][q];
  for (int k = 0; k < s - 4; ++k) {
    const double* r = kRock4Rec[kRock4Off[i] + k];
    if (mu) mu[k] = r[0];
    if (nu) nu[k] = r[1];
    if (kappa) kappa[k] = r[2];
  }
  return RD_OK;
}
