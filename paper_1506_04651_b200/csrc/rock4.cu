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
#include <mutex>
#include <string>
#include <vector>

#include "mr.cuh"
#ifndef RD_ROCK4_TABLE
#define RD_ROCK4_TABLE "rock4_coeffs.inc"
#endif
#include RD_ROCK4_TABLE

namespace cg = cooperative_groups;

namespace rdmr {
namespace {

constexpr int kR4Threads = kR4Chunk;
constexpr int kNsteps = RD_ROCK4_SMAX - 4;
__constant__ double c_ell[kNsteps];
__constant__ double c_sig[kNsteps][4];
__constant__ int c_off[kNsteps + 1];
// recurrence coefficients of the stage counts s <= kConstRecS in the constant bank (the controller reads
// them every round; s = 5..9 on the BJ configurations): 666 triples, 16 KB
constexpr int kConstRecS = 40;
constexpr int kConstRecN = 666;  // kRock4Off[kConstRecS - 4]
__constant__ double c_rec[kConstRecN][3];
// The coefficient tables live per device: __constant__ symbols exist once per device context, and the
// recurrence table is a device allocation.  Uploaded on the first Rock4 call on each device.
constexpr int kMaxDevices = 64;
double* g_rec[kMaxDevices] = {};  // device copy of kRock4Rec, per device
std::mutex g_tables_mu;

rd_status tables(const double** rec) {
  int dev = 0;
  RD_CUDA_TRY(cudaGetDevice(&dev));
  if (dev < 0 || dev >= kMaxDevices) return RD_ENOTSUP;
  std::lock_guard<std::mutex> lk(g_tables_mu);
  if (!g_rec[dev]) {
    RD_CUDA_TRY(cudaMemcpyToSymbol(c_ell, kRock4Ell, sizeof(kRock4Ell)));
    RD_CUDA_TRY(cudaMemcpyToSymbol(c_sig, kRock4Sig, sizeof(kRock4Sig)));
    RD_CUDA_TRY(cudaMemcpyToSymbol(c_off, kRock4Off, sizeof(kRock4Off)));
    static_assert(kConstRecN <= 19306, "rec table");
    RD_CUDA_TRY(cudaMemcpyToSymbol(c_rec, kRock4Rec, sizeof(double) * 3 * kConstRecN));
    double* r = nullptr;
    RD_CUDA_TRY(cudaMalloc(&r, sizeof(kRock4Rec)));
    RD_CUDA_TRY(cudaMemcpy(r, kRock4Rec, sizeof(kRock4Rec), cudaMemcpyHostToDevice));
    g_rec[dev] = r;
  }
  *rec = g_rec[dev];
  return RD_OK;
}

struct R4Spec {
  double* buf[5];  // stage vectors, each [N + n_need]: V = [leaf values | needed internal values];
                   // 0: state, 1..3: recurrence, 4: spare state / x_acc
  double* u;       // the species' leaf values in the grid (or the forced-step input)
  double* gh;      // ghost values [n_if * 4] of the current stage (ghost phase)
  double eps;
  int id;          // species index in the grid (hprop slot)
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
  unsigned int* tick; // [4] chunk tickets (round-robin slots); [3]: assembled kernel's last-block counter;
                      // [4]: matrix-free kernel's last-block counter
  double* errfin;     // [kMaxSpecies]: assembled kernel, error square sums reduced by the last block
  double* hprop;      // [kMaxSpecies] per grid species: the step size the controller proposed for the next
                      // step when the previous D call ended (0: none yet), read as h0 (reading R-K5b)
  int forced;         // 1: one step with (forced_s, forced_h), outputs to out/err
  int forced_s;
  double forced_h;
  double* out;
  double* err;
};

#ifndef RD_R4_SG
#define RD_R4_SG 1  // species per stage-row group (1, 2, 3: measured 2.46 / 2.47 / 2.49 ms per cfg-4 call)
#endif
enum : int { OP_REC = 0, OP_P1 = 1, OP_P2 = 2, OP_P3 = 3, OP_P4 = 4, OP_DONE = 5 };

struct Ctl {
  double t, h, he, hwant;  // hwant: h before the end-of-interval clip
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
    c.hwant = c.h;
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

// Buffer assignment and coefficients of the current op (Ctl.op, Ctl.k).  The recurrence uses two
// ping-pong buffers B0 = 1, B1 = 2: g_{k+1} = mu hA g_k + nu g_k + kappa g_{k-1} overwrites g_{k-1} in
// place (prev and out are the same own-row entries, read before written by the same thread; only `in`
// is gathered across rows), so a round touches two stage vectors per species instead of three and the
// 3-D working set stays closer to L2.  Finishing: P1 reads y = g_{s-4} and writes into the other
// buffer (it held g_{s-5}, last gathered one round earlier); P2..P4 alternate.
__device__ void set_op(Ctl& c, const R4Params& P) {
  const int n = c.s - 4;
  if (c.op == OP_REC) {
    const int k = c.k;
    c.in = k == 0 ? c.xcur : 1 + ((k - 1) & 1);
    c.prev = k <= 1 ? c.xcur : 1 + (k & 1);
    c.out = 1 + (k & 1);
    const int e = c_off[c.s - 5] + k;
    if (c.s <= kConstRecS) {
      c.c0 = c_rec[e][0]; c.c1 = c_rec[e][1]; c.c2 = c_rec[e][2];
    } else {
      const double* r = P.rec + 3 * e;
      c.c0 = r[0]; c.c1 = r[1]; c.c2 = r[2];
    }
  } else {
    const int y = 1 + ((n - 1) & 1);  // g_{s-4}, the last recurrence output
    const int o = 3 - y;              // the other ping-pong buffer
    c.xacc = c.xcur == 0 ? 4 : 0;
    if (c.op == OP_P1) { c.in = y; c.out = o; }
    else if (c.op == OP_P2) { c.in = o; c.out = y; }
    else if (c.op == OP_P3) { c.in = y; c.out = o; }
    else { c.in = o; c.out = -1; }
    c.prev = y;
    c.c0 = c_sig[c.s - 5][c.op - 1];
  }
}


#ifndef RD_R4_MINB2
#define RD_R4_MINB2 2
#endif
#ifndef RD_R4_MINB3
#define RD_R4_MINB3 5  // 3-D: 5 x 256 threads (48 registers): 3, 4, 5, 6 blocks measured 2.69, 2.45, 2.40, 2.76 ms per cfg-4 call
                        // (round 1, one block of 3 species per row: 4 x 256 beat 2 x 256, 112.7 -> 94 us/round)
#endif
#ifndef RD_R4_TIMING
#define RD_R4_TIMING 0
#endif
#if RD_R4_TIMING
#define R4T(slot) do { if (tid == 0) { const long long c_ = clock64(); tacc[slot] += c_ - tlast; tlast = c_; } } while (0)
#else
#define R4T(slot) do { } while (0)
#endif
// Internal stencil values are filled by a separate projection phase (inline projection in the stage
// phase, one barrier fewer, was measured slower and removed).
constexpr bool kInlineProj = false;

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

// End of a round (after the grid barrier), run by warp 0 of every block on identical data: error
// norms of the species that just finished a step (the warp sums the npart partials with a fixed lane
// -> partial assignment and a fixed butterfly, so every block gets the same bits), then the step
// control (K5) and the next op of every species.  One block barrier publishes the result.
// Per-round op of one active species, resolved once per round from its Ctl (the stage code then reads
// only broadcast shared-memory words): out = c0 ah + c1 in + c2 p2 (REC); out = ah, xacc = (P1 ? p2 :
// xacc) + c0 ah (P1..P3); xacc += c0 ah with the error term against p1 = x_n (P4); ah = he (A in)_r.
struct SpOp {
  const double* in;
  const double* p1;  // REC: in, P4: x_n (xcur), else unused
  const double* p2;  // REC, P1: prev (y); P2..P4: xacc
  double* out;       // REC..P3
  double* xacc;
  double c0, c1, c2, he;
  int op, sp;
};

// B: the species' 5 stage buffers (a shared-memory copy of P.sp[i].buf: a dynamically indexed
// parameter load would go through the constant cache every round)
__device__ __forceinline__ void make_spop(double* const* B, const Ctl& c, int i, SpOp& o) {
  o.in = B[c.in];
  o.p1 = c.op == OP_REC ? B[c.in] : B[c.xcur];
  o.p2 = (c.op == OP_REC || c.op == OP_P1) ? B[c.prev] : B[c.xacc];
  o.out = c.op == OP_REC ? B[c.out] : (c.op == OP_P4 ? nullptr : B[c.out]);
  o.xacc = B[c.xacc];
  o.c0 = c.c0; o.c1 = c.c1; o.c2 = c.c2; o.he = c.he;
  o.op = c.op;
  o.sp = i;
}

// One row r of the matrix-free stage for the S active species so[g0 ..] (per-round descriptors in
// shared memory, built by the controller lanes): matvec with shared topology, then each species'
// stage combination.  P4 error partials go to red[warp][species].
template <int D, int S>
__device__ __forceinline__ void stage_group_op(const R4Params& P, const SpOp* so, int g0, int64_t r,
                                               double (*red)[kMaxSpecies]) {
  const GridDev& G = P.G;
  const double* V[S];
  const double* gh[S];
#pragma unroll
  for (int s = 0; s < S; ++s) {
    V[s] = so[g0 + s].in;
    gh[s] = P.sp[so[g0 + s].sp].gh;
  }
  double a[S];
  const bool live = r < G.N;
  // the combination operands (own row, coalesced) are loaded before the mat-vec so their latency
  // overlaps the neighbour gathers
  double o2v[S], o1v[S];
#pragma unroll
  for (int s = 0; s < S; ++s) {
    o2v[s] = live ? so[g0 + s].p2[r] : 0.0;  // REC, P1: prev; P2..P4: x_acc
    o1v[s] = (live && so[g0 + s].op == OP_P4) ? so[g0 + s].p1[r] : 0.0;  // P4: x_n
  }
  if (live) {
    if constexpr (kGhostPhase<D>) fv_row_ghosts<D, S>(G, V, gh, r, a);
    else fv_row_multi<D, S>(G, V, r, a, kInlineProj);
  }
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const SpOp& o = so[g0 + s];
    double part = 0.0;
    if (live) {
      const double ah = o.he * a[s];
      const double o2 = o2v[s];
      if (o.op == OP_REC) {
        o.out[r] = o.c0 * ah + o.c1 * V[s][r] + o.c2 * o2;
      } else if (o.op != OP_P4) {
        o.out[r] = ah;
        o.xacc[r] = o2 + o.c0 * ah;
      } else {
        const double e = o.c0 * ah;
        const double xn = o2 + e;
        o.xacc[r] = xn;
        const double sc = P.atol + P.rtol * fmax(fabs(o1v[s]), fabs(xn));
        const double q = e / sc;
        part = q * q;
        if (P.forced) { P.out[r] = xn; P.err[r] = e; }
      }
    }
    if (o.op == OP_P4) {  // block-uniform branch
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) part += __shfl_xor_sync(0xffffffffu, part, off);
      if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5][o.sp] = part;
    }
  }
}

// 3-D stage: projections of chunk c's simple nodes (GridDev::proj_*) in the buffers its rows were just
// written to (the next round's inputs: out, or x_acc in a P4 round), by the block that ran the chunk,
// after the chunk's block barrier (the rows are this block's own writes).  Expansion list order.
__device__ __forceinline__ void project_chunk(const R4Params& P, const SpOp* so, int nact, int c) {
  const GridDev& G = P.G;
  const int32_t b = G.proj_cstart[c], n = G.proj_cstart[c + 1] - b;
  for (int i = threadIdx.x; i < n * nact; i += blockDim.x) {
    const int2 ql = G.proj_cnode[b + i / nact];  // (node, first child's leaf index); weights 2^-3
    const SpOp& o = so[i % nact];
    double* t = o.op == OP_P4 ? o.xacc : o.out;
    double v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = t[ql.y + k];
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) acc += 0.125 * v[k];
    t[G.N + ql.x] = acc;
  }
}

// s_op: NULL, or the active species' per-round descriptors to build for the next round (assembled
// kernel: the controller lanes write them straight from their registers, so the next round starts
// without another block barrier).
__device__ void round_end(const R4Params& P, Ctl* ctl, double* errsq, int* s_act, int& s_nact, int& s_anyp4,
                          int& s_active, int& s_round, int64_t npart, int64_t N, SpOp* s_op = nullptr,
                          double* const (*s_buf)[5] = nullptr, const double* errfin = nullptr) {
  const int tid = threadIdx.x;
#if RD_R4_TIMING
  __shared__ long long s_rt[4];
  long long t0 = clock64();
  if (s_round == 0 && tid < 4) s_rt[tid] = 0;
#define RT(q) do { if (tid == 0) { const long long t1 = clock64(); s_rt[q] += t1 - t0; t0 = t1; } } while (0)
#else
#define RT(q) do { } while (0)
#endif
  if (tid < 32) {
    if (errfin) {  // reduced before the barrier by the last block (assembled kernel)
      if (tid < P.nsp && ctl[tid].op == OP_P4) errsq[tid] = __ldcg(errfin + tid);
    }
    for (int a = 0; a < (errfin ? 0 : s_nact); ++a) {
      const int i = s_act[a];
      if (ctl[i].op != OP_P4) continue;
      double acc = 0.0;
      const double* pp = P.part + int64_t(i) * npart;
      for (int64_t b0 = 0; b0 < npart; b0 += 32 * 16) {  // 16 independent loads per lane in flight
        double v[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const int64_t b = b0 + tid + 32 * k;
          v[k] = b < npart ? pp[b] : 0.0;
        }
#pragma unroll
        for (int k = 0; k < 16; ++k) acc += v[k];
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (tid == 0) errsq[i] = acc;
    }
    __syncwarp();
    RT(0);
    Ctl c;
    bool act = false, p4 = false;
    if (tid < P.nsp) {  // step control (identical inputs in every block => identical decisions)
      c = ctl[tid];
      if (c.op != OP_DONE) {
        c.matvecs++;
        if (c.op == OP_REC) {
          if (++c.k >= c.s - 4) c.op = OP_P1;
        } else if (c.op < OP_P4) {
          c.op++;
        } else {
          const double err = sqrt(errsq[tid] / double(N > 0 ? N : 1));
          const double fac = err > 0.0 ? fmin(5.0, fmax(0.1, 0.8 / sqrt(sqrt(err)))) : 5.0;
          if (!P.forced && !isfinite(err)) {  // a non-finite stage value: fail now, never retry
            c.failed = 1;
            c.op = OP_DONE;
          } else if (P.forced) {
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
      act = c.op != OP_DONE;
      p4 = c.op == OP_P4;
    }
    __syncwarp();
    RT(1);
    // active list in species order by warp vote (lane i = species i)
    const unsigned am = __ballot_sync(0xffffffffu, act);
    const bool anyp4 = __any_sync(0xffffffffu, p4);
    if (act) {
      const int pos = __popc(am & ((1u << tid) - 1u));
      s_act[pos] = tid;
      if (s_op) make_spop(s_buf[tid], c, tid, s_op[pos]);
    }
    if (tid == 0) {
      s_nact = __popc(am);
      s_anyp4 = anyp4;
      s_active = am != 0u;
      ++s_round;
    }
    __syncwarp();
    RT(2);
  }
  __syncthreads();
  RT(3);
#if RD_R4_TIMING
  if (tid == 0 && blockIdx.x == 0 && s_active == 0)
    printf("[round_end block0 cycles] errsq %lld ctl %lld act+spop %lld syncthreads %lld (rounds %d)\n", s_rt[0], s_rt[1],
           s_rt[2], s_rt[3], s_round);
#endif
#undef RT
}

template <int D>
__global__ void __launch_bounds__(kR4Threads, D == 2 ? RD_R4_MINB2 : RD_R4_MINB3) k_rock4(R4Params P) {
  cg::grid_group grid = cg::this_grid();
  __shared__ Ctl ctl[kMaxSpecies];
  __shared__ double redsp[kR4Threads / 32][kMaxSpecies];
  __shared__ int s_act[kMaxSpecies];
  __shared__ int s_nact, s_anyp4;
  __shared__ int s_active;
  __shared__ double errsq[kMaxSpecies];
  __shared__ int s_tk[2];
  __shared__ int s_nif2;
  __shared__ int s_nns;  // 3-D: needed internal nodes the stage does not project (operator build)
  __shared__ double redsp2[2][kR4Threads / 32][kMaxSpecies];
  __shared__ int s_round;
  __shared__ int s_last;
  __shared__ SpOp s_op[kMaxSpecies];
  __shared__ double* s_buf[kMaxSpecies][5];
  const int tid = threadIdx.x;
  const int64_t gtid = blockIdx.x * int64_t(blockDim.x) + tid;
  const int64_t gstride = int64_t(gridDim.x) * blockDim.x;
  const GridDev& G = P.G;
  const int64_t nch = (G.N + kR4Threads - 1) / kR4Threads;

  if (tid < P.nsp)
    for (int b = 0; b < 5; ++b) s_buf[tid][b] = P.sp[tid].buf[b];
  if (tid < P.nsp) {
    Ctl c{};
    c.t = 0.0;
    c.h = P.T;
    if (!P.forced && P.hprop) {  // the previous D call's proposal (R-K5b)
      const double hp = P.hprop[P.sp[tid].id];
      if (hp > 0.0 && hp < P.T) c.h = hp;
    }
    c.xcur = 0;
    start_step(c, P, P.sp[tid].eps * P.rho1);
    c.he = c.h * P.sp[tid].eps;
    set_op(c, P);
    ctl[tid] = c;
  }
  if (tid == 0) {
    s_round = 0;
    s_nif2 = (kGhostPhase<D> && G.n_if > 0) ? *G.if2_count : 0;
    s_nns = kGhostPhase<D> ? *G.proj_ns_count : 0;
  }
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
  __syncthreads();
  if (tid < s_nact) make_spop(s_buf[s_act[tid]], ctl[s_act[tid]], s_act[tid], s_op[tid]);
  // state -> slack buffer 0
  for (int i = 0; i < P.nsp; ++i)
    for (int64_t r = gtid; r < G.N; r += gstride) P.sp[i].buf[0][r] = P.sp[i].u[r];
  __syncthreads();
  grid.sync();

  while (true) {
    // ---- phase A: projections of the needed internal nodes of each op's input vector (V tail).  3-D:
    //      after round 0 only the non-simple nodes (GridDev::proj_*); the simple ones were projected by
    //      the previous round's stage, chunk by chunk, when it wrote this round's input
    const bool fullA = !kGhostPhase<D> || s_round == 0;
    const int64_t nA = fullA ? G.n_need : int64_t(s_nns);
    if (!kInlineProj && nA > 0) {
      // 8 lanes per needed node (4 nodes per warp): lane l sums entries l, l + 8, ... of the node's
      // expansion (leaf, weight) list in batches of 4 (all loads of a batch in flight together), then
      // the 8 partial sums are combined by a fixed xor butterfly; the list is read once for up to three
      // active species at a time.  A long expansion (an internal node several levels above its leaves)
      // costs len / 32 memory round trips instead of len / 4.
      const int nact = s_nact;
      const int lane = tid & 31, l8 = lane & 7;
      const int64_t nq4 = (nA + 3) / 4;
      for (int64_t qb = gtid >> 5; qb < nq4; qb += gstride >> 5) {
        const int64_t qi = qb * 4 + (lane >> 3);
        const bool on = qi < nA;
        const int64_t q = (fullA || !on) ? qi : int64_t(G.proj_ns[qi]);
        const int32_t e0 = on ? G.exp_start[q] : 0, e1 = on ? G.exp_start[q + 1] : 0;
        for (int a0 = 0; a0 < nact; a0 += 3) {
          const int na = min(3, nact - a0);
          double* V[3];
#pragma unroll
          for (int s = 0; s < 3; ++s) V[s] = P.sp[s_act[a0 + (s < na ? s : 0)]].buf[ctl[s_act[a0 + (s < na ? s : 0)]].in];
          double acc[3] = {0.0, 0.0, 0.0};
          for (int32_t eb = e0 + l8; eb < e1; eb += 32) {
            double w[4];
            int32_t l[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const bool in = eb + 8 * u < e1;
              w[u] = in ? G.exp_w[eb + 8 * u] : 0.0;
              l[u] = in ? G.exp_leaf[eb + 8 * u] : G.exp_leaf[eb];
            }
            double v[3][4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
              for (int s = 0; s < 3; ++s) v[s][u] = s < na ? V[s][l[u]] : 0.0;
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
              for (int s = 0; s < 3; ++s) acc[s] += w[u] * v[s][u];
          }
#pragma unroll
          for (int o = 4; o > 0; o >>= 1)
#pragma unroll
            for (int s = 0; s < 3; ++s) acc[s] += __shfl_xor_sync(0xffffffffu, acc[s], o);
          if (on && l8 == 0)
#pragma unroll
            for (int s = 0; s < 3; ++s)
              if (s < na) V[s][G.N + q] = acc[s];
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
      // one (type-2 record, species) pair per thread over the compact list of the records with finer
      // leaves: the record's 27 stencil indices are loaded by each of its species' threads (L1 hits after
      // the first), each thread holds one species' 27 values
      const int64_t npair = int64_t(s_nif2) * nact;
      for (int64_t q = gtid; q < npair; q += gstride) {
        const int64_t k = q / nact;
        ghost_group<D, 1>(P, ctl, s_act, int(q - k * nact), G.if2_list[k]);
      }
      grid.sync();
    }
    R4T(5);
    // ---- phase B: one stage (matvec + combination) for every active species.  A thread evaluates its
    //      row for RD_R4_SG species at a time (1 by default: fewer registers, more resident warps; the
    //      row's topology is then re-read from L1 per species).  Chunks of kR4Threads rows
    //      are handed out by an atomic ticket (the next one is fetched while the current chunk runs) so
    //      blocks that draw interface-heavy chunks (they cluster in Morton order) do not hold the
    //      barrier back.  One block barrier per chunk: the ticket and the warps' P4 partials are
    //      double-buffered by chunk parity, and a chunk's partial (its own slot -> fixed reduction
    //      order) is summed during the next chunk.
    {
      const int slot = s_round & 3;
      if (blockIdx.x == 0 && tid == 0) P.tick[(s_round + 2) & 3] = 0u;  // last used 2 rounds ago
      const int nact = s_nact, anyp4 = s_anyp4;
      // s_tk holds the next chunk (ticket t -> chunk_order[t], resolved by thread 0 while the current
      // chunk runs); longest-first order: chunks with the most interface faces first (sorted at operator
      // build), so the round ends on light chunks
      if (tid == 0) {
        const unsigned t0 = atomicAdd(P.tick + slot, 1u);
        s_tk[0] = t0 < nch ? G.chunk_order[t0] : -1;
      }
      __syncthreads();
      int64_t prev = -1;
      for (int k = 0;; ++k) {
        const int64_t chunk = s_tk[k & 1];
        if (anyp4 && prev >= 0 && tid < P.nsp && ctl[tid].op == OP_P4) {
          double sm = 0.0;
          for (int w = 0; w < kR4Threads / 32; ++w) sm += redsp2[(k + 1) & 1][w][tid];
          P.part[int64_t(tid) * nch + prev] = sm;
        }
        if (kGhostPhase<D> && prev >= 0) project_chunk(P, s_op, nact, int(prev));
        if (chunk < 0) break;
        if (tid == 0) {
          const unsigned t1 = atomicAdd(P.tick + slot, 1u);
          s_tk[(k + 1) & 1] = t1 < nch ? G.chunk_order[t1] : -1;
        }
        const int64_t r = chunk * kR4Threads + tid;
        double (*red)[kMaxSpecies] = redsp2[k & 1];
        int g0 = 0;
        if (RD_R4_SG >= 3)
          for (; g0 + 3 <= nact; g0 += 3) stage_group_op<D, 3>(P, s_op, g0, r, red);
        if (RD_R4_SG >= 2)
          for (; g0 + 2 <= nact; g0 += 2) stage_group_op<D, 2>(P, s_op, g0, r, red);
        for (; g0 < nact; ++g0) stage_group_op<D, 1>(P, s_op, g0, r, red);
        __syncthreads();
        prev = chunk;
      }
    }
    // the last block to finish a P4 stage sums the chunk partials (fixed order) before the barrier, so
    // that after it every block reads one value per species instead of all nch partials
    if (s_anyp4) {
      __threadfence();
      __syncthreads();
      if (tid == 0) s_last = (atomicAdd(P.tick + 4, 1u) + 1u) % gridDim.x == 0u;
      __syncthreads();
      if (s_last) {
        for (int i = 0; i < P.nsp; ++i) {
          if (ctl[i].op != OP_P4) continue;
          double acc = 0.0;
          for (int64_t b = tid; b < nch; b += kR4Threads) acc += __ldcg(P.part + int64_t(i) * nch + b);
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
          if ((tid & 31) == 0) redsp[tid >> 5][i] = acc;
          __syncthreads();
          if (tid == 0) {
            double sm = 0.0;
            for (int w = 0; w < kR4Threads / 32; ++w) sm += redsp[w][i];
            P.errfin[i] = sm;
          }
          __syncthreads();
        }
      }
    }
    R4T(2);
    grid.sync();
    R4T(3);
    round_end(P, ctl, errsq, s_act, s_nact, s_anyp4, s_active, s_round, nch, G.N, s_op, s_buf, P.errfin);
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
    if (!P.forced && P.hprop && !c.failed) P.hprop[P.sp[tid].id] = c.hwant;
  }
}

// ---------------------------------------------------------------------------------------------
constexpr int kR4MatThreads = 32 * kMatWarps;
#ifndef RD_R4_MAT_UNROLL
#define RD_R4_MAT_UNROLL 4
#endif
constexpr int kMatUnroll = RD_R4_MAT_UNROLL;
#ifndef RD_MAT_THREADS_SM
#define RD_MAT_THREADS_SM 1024
#endif
constexpr int kR4MatBps = RD_MAT_THREADS_SM / kR4MatThreads;     // resident blocks per SM
constexpr int kR4MatSmemCap = 200 * 1024 / kR4MatBps;            // dynamic shared memory per block
#ifndef RD_MAT_GROUP
#define RD_MAT_GROUP 3
#endif
constexpr int kMatGroup = RD_MAT_GROUP;  // species per stage pass (3: shared matrix loads; 1: fewer registers)


// Stage vectors are written by other blocks in earlier rounds of this launch, so their loads are
// coherent L2 loads (__ldcg, ld.global.cg): the non-coherent read-only path (__ldg) is not ordered by
// the grid barrier in the CUDA memory model.  Only the operator arrays (constant for the launch) use
// __ldg.
// One stage of S species (descriptors so[g0 ..]) on the row group of this lane (row r, G = 2^lg lanes
// per row, `lead` = the first of them).  The combination operands are loaded before the mat-vec so
// their latency overlaps the value gathers; col / wt point at this lane's slot column (stride 32).
// WK (mat_wk): 0 FP32 weights, 1 FP64 weights, 2 compact two-point links (column | type << 30, the
// coefficient rebuilt from the row level j: sum_t w_t (x_col - x_row)).
template <int S, int WK>
__device__ __forceinline__ void stage_mat_group(const R4Params& P, const SpOp* so, int g0, int32_t r, int j,
                                                const int32_t* col, const void* wt, int wdt, int lg, bool lead,
                                                double (*red)[kMaxSpecies]) {
  const bool live = r >= 0;
  const bool upd = live && lead;
  double o1[S], o2[S], a[S], xr[S];
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const SpOp& o = so[g0 + s];
    o1[s] = (upd && (o.op == OP_REC || o.op == OP_P4)) ? __ldcg(o.p1 + r) : 0.0;
    o2[s] = upd ? __ldcg(o.p2 + r) : 0.0;
    xr[s] = (WK == 2 && live) ? __ldcg(o.in + r) : 0.0;
    a[s] = 0.0;
  }
  if (live) {
    double tw[3] = {0.0, 0.0, 0.0};
    if (WK == 2)
#pragma unroll
      for (int t = 0; t < 3; ++t) tw[t] = tp_coef(t, P.G.dim, j);
#pragma unroll kMatUnroll
    for (int e = 0; e < wdt; ++e) {
      int32_t c = col[32 * e];
      double w;
      if (WK == 0) w = double(static_cast<const float*>(wt)[32 * e]);
      else if (WK == 1) w = static_cast<const double*>(wt)[32 * e];
      else {
        const int t = int(uint32_t(c) >> 30);
        w = t == 0 ? tw[0] : (t == 1 ? tw[1] : tw[2]);
        c &= 0x3fffffff;
      }
#pragma unroll
      for (int s = 0; s < S; ++s) a[s] = fma(w, WK == 2 ? __ldcg(so[g0 + s].in + c) - xr[s] : __ldcg(so[g0 + s].in + c), a[s]);
    }
  }
  for (int o = 1; o < (1 << lg); o <<= 1)  // warp-uniform: join the G lanes of each row
#pragma unroll
    for (int s = 0; s < S; ++s) a[s] += __shfl_xor_sync(0xffffffffu, a[s], o);
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const SpOp& o = so[g0 + s];
    double part = 0.0;
    if (upd) {
      const double ah = o.he * a[s];
      if (o.op == OP_REC) {
        o.out[r] = o.c0 * ah + o.c1 * o1[s] + o.c2 * o2[s];
      } else if (o.op != OP_P4) {
        o.out[r] = ah;
        o.xacc[r] = o2[s] + o.c0 * ah;
      } else {
        const double e = o.c0 * ah;
        const double xn = o2[s] + e;
        o.xacc[r] = xn;
        const double sc = P.atol + P.rtol * fmax(fabs(o1[s]), fabs(xn));
        const double q = e / sc;
        part = q * q;
        if (P.forced) { P.out[r] = xn; P.err[r] = e; }
      }
    }
    if (o.op == OP_P4) {  // block-uniform branch; each warp accumulates into its own slot
#pragma unroll
      for (int q = 16; q > 0; q >>= 1) part += __shfl_xor_sync(0xffffffffu, part, q);
      if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5][o.sp] += part;
    }
  }
}

// Rock4 on the assembled operator (fvmat.cu, 2-D): a round is ONE sparse mat-vec stage of every active
// species, then the grid barrier and the controller.  Warp gw of the grid owns slices gw, gw + nw,
// ... (static, so the per-block error partials have a fixed summation order).  CACHE: the operator
// is constant for the whole call, so each warp copies its slices (metadata, rows, columns, FP32
// weights) into shared memory once; a stage then reads only the value vectors from L2, one memory
// latency deep.  Shared layout of a warp: [2 nsl meta words | 32 nsl rows | per slice: 32 w columns,
// 32 w weights].
template <bool CACHE, int WK>
__global__ void __launch_bounds__(kR4MatThreads, kR4MatBps) k_rock4_mat(R4Params P) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ int4 dsm4[];
  __shared__ Ctl ctl[kMaxSpecies];

  __shared__ double redsp[kMatWarps][kMaxSpecies];
  __shared__ int s_act[kMaxSpecies];
  __shared__ int s_nact, s_anyp4, s_active, s_round;
  __shared__ double errsq[kMaxSpecies];
  __shared__ int s_words[kMatWarps];
  __shared__ int s_last;
  __shared__ SpOp s_op[kMaxSpecies];
  __shared__ double* s_buf[kMaxSpecies][5];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t gtid = blockIdx.x * int64_t(blockDim.x) + tid;
  const int64_t gstride = int64_t(gridDim.x) * blockDim.x;
  const GridDev& G = P.G;
  const int64_t gw = gtid >> 5, nw = gstride >> 5;
  const int nsl = gw < G.n_slice ? int((G.n_slice - gw + nw - 1) / nw) : 0;
  int* wsm = reinterpret_cast<int*>(dsm4);

  if (tid < P.nsp)
    for (int b = 0; b < 5; ++b) s_buf[tid][b] = P.sp[tid].buf[b];
  if (tid < P.nsp) {
    Ctl c{};
    c.t = 0.0;
    c.h = P.T;
    if (!P.forced && P.hprop) {  // the previous D call's proposal (R-K5b)
      const double hp = P.hprop[P.sp[tid].id];
      if (hp > 0.0 && hp < P.T) c.h = hp;
    }
    c.xcur = 0;
    start_step(c, P, P.sp[tid].eps * P.rho1);
    c.he = c.h * P.sp[tid].eps;
    set_op(c, P);
    ctl[tid] = c;
  }
  if (tid == 0) s_round = 0;
  if (CACHE) {  // this warp's shared region
    int words = 0;
    for (int k = 0; k < nsl; ++k) words += 34 + 32 * mat_slot_words(WK) * (G.m_slc[gw + k * nw].z & 0xff);
    if (lane == 0) s_words[wid] = words;
    __syncthreads();
    int off = 0;
    for (int w = 0; w < wid; ++w) off += s_words[w];
    wsm += off;
    int* meta = wsm;
    int* rows = wsm + 2 * nsl;
    int coff = 34 * nsl;
    for (int k = 0; k < nsl; ++k) {
      const int4 md = G.m_slc[gw + k * nw];
      const int wdt = md.z & 0xff, nrows = (md.z >> 8) & 0xff;
      if (lane == 0) { meta[2 * k] = coff; meta[2 * k + 1] = md.z; }
      int rw = lane < nrows ? G.m_row[md.x + lane] : -1;
      if (WK == 2 && rw >= 0) rw |= int(G.keys[rw] >> kLevelShift) << 27;  // level in the high bits
      rows[32 * k + lane] = rw;
      for (int i = lane; i < 32 * wdt; i += 32) {
        wsm[coff + i] = G.m_col[md.y + i];
        if (WK == 0) wsm[coff + 32 * wdt + i] = __float_as_int(G.m_w[md.y + i]);
        if (WK == 1) reinterpret_cast<double*>(wsm + coff + 32 * wdt)[i] = G.m_wd[md.y + i];
      }
      coff += 32 * mat_slot_words(WK) * wdt;
    }
  }
#if RD_R4_TIMING
  long long tacc[6] = {0, 0, 0, 0, 0, 0};  // stage phase, partials, barrier, round end
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
  __syncthreads();
  if (tid < s_nact) make_spop(s_buf[s_act[tid]], ctl[s_act[tid]], s_act[tid], s_op[tid]);
  for (int i = 0; i < P.nsp; ++i)
    for (int64_t r = gtid; r < G.N; r += gstride) P.sp[i].buf[0][r] = P.sp[i].u[r];
  __syncthreads();
  grid.sync();

  while (true) {
    const int nact = s_nact, anyp4 = s_anyp4;
    if (anyp4) redsp[wid][lane] = 0.0;  // this warp's own row (read after the stage's block barrier)
    __syncwarp();
    for (int k = 0; k < nsl; ++k) {
      int z, j = 0;
      int32_t r;
      const int32_t* col;
      const void* wt;
      if (CACHE) {
        z = wsm[2 * k + 1];
        const int lg = z >> 16, q = lane >> lg;
        r = wsm[2 * nsl + 32 * k + q];
        if (WK == 2 && r >= 0) { j = r >> 27; r &= (1 << 27) - 1; }
        col = wsm + wsm[2 * k] + lane;
        if (WK == 0) wt = col + 32 * (z & 0xff);
        else wt = reinterpret_cast<const double*>(wsm + wsm[2 * k] + 32 * (z & 0xff)) + lane;
      } else {
        const int4 md = G.m_slc[gw + k * nw];
        z = md.z;
        const int lg = z >> 16, q = lane >> lg;
        r = q < ((z >> 8) & 0xff) ? G.m_row[md.x + q] : -1;
        if (WK == 2 && r >= 0) j = int(G.keys[r] >> kLevelShift);
        col = G.m_col + md.y + lane;
        if (WK == 0) wt = G.m_w + md.y + lane;
        else wt = G.m_wd + md.y + lane;
      }
      const int wdt = z & 0xff, lg = z >> 16;
      const bool lead = (lane & ((1 << lg) - 1)) == 0;
      int g0 = 0;
      if (kMatGroup == 3) {
        for (; g0 + 3 <= nact; g0 += 3) stage_mat_group<3, WK>(P, s_op, g0, r, j, col, wt, wdt, lg, lead, redsp);
        if (nact - g0 == 2) {
          stage_mat_group<2, WK>(P, s_op, g0, r, j, col, wt, wdt, lg, lead, redsp);
          g0 += 2;
        }
      }
      for (; g0 < nact; ++g0) stage_mat_group<1, WK>(P, s_op, g0, r, j, col, wt, wdt, lg, lead, redsp);
    }
    R4T(0);
    if (anyp4) {  // per-block partial of every species in P4, fixed warp order
      __syncthreads();
      if (tid < P.nsp && ctl[tid].op == OP_P4) {
        double sm = 0.0;
        for (int w = 0; w < kMatWarps; ++w) sm += redsp[w][tid];
        P.part[int64_t(tid) * gridDim.x + blockIdx.x] = sm;
        __threadfence();
      }
      __syncthreads();
      // the last block to arrive sums the partials (fixed order) before the barrier, so that after it
      // every block reads one value instead of all gridDim.x partials
      if (tid == 0) s_last = (atomicAdd(P.tick + 3, 1u) + 1u) % gridDim.x == 0u;
      __syncthreads();
      if (s_last) {  // warp w reduces species w, w + kMatWarps, ... (all species in parallel)
        for (int i = wid; i < P.nsp; i += kMatWarps) {
          if (ctl[i].op != OP_P4) continue;
          double acc = 0.0;
          for (int b = lane; b < int(gridDim.x); b += 32) acc += __ldcg(P.part + int64_t(i) * gridDim.x + b);
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
          if (lane == 0) P.errfin[i] = acc;
        }
      }
    }
    R4T(1);
#if RD_R4_TIMING
    __syncthreads();  // timing build only: separates the wait for this block's warps from the grid barrier
    R4T(4);
#endif
    grid.sync();
    R4T(2);
    round_end(P, ctl, errsq, s_act, s_nact, s_anyp4, s_active, s_round, gridDim.x, G.N, s_op, s_buf, P.errfin);
    R4T(3);
    if (!s_active) break;
  }
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
    if (!P.forced && P.hprop && !c.failed) P.hprop[P.sp[tid].id] = c.hwant;
  }
}

}  // namespace

// Reads the controller results of a finished launch into stats; RD_ESTIFF if a species failed.
rd_status rock4_finish(R4Pending& pd, rd_stats* stats) {
  if (!pd.armed) return RD_OK;
  pd.armed = false;
  const long long* hs = pd.hs;
  const int nsp = pd.nsp;
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
  if (pd.ev[0]) {
    float kms = 0.0f;
    if (stats && cudaEventElapsedTime(&kms, pd.ev[0], pd.ev[1]) == cudaSuccess) stats->rock4_kernel_ms += kms;
    cudaEventDestroy(pd.ev[0]);
    cudaEventDestroy(pd.ev[1]);
    pd.ev[0] = pd.ev[1] = nullptr;
  }
  if (stats) {
    stats->rho1 = pd.rho1;
    stats->rock4_rounds += hs[6 * nsp];
    stats->rock4_mat_slots = pd.mat_slots;
  }
#if RD_R4_TIMING
  std::fprintf(stderr, "[rock4 timing block0, cycles] %lld %lld %lld %lld %lld %lld rounds %lld\n", hs[6 * nsp + 1],
               hs[6 * nsp + 2], hs[6 * nsp + 3], hs[6 * nsp + 4], hs[6 * nsp + 5], hs[6 * nsp + 6], hs[6 * nsp]);
#endif
  return failed ? RD_ESTIFF : RD_OK;
}

// Stage-vector workspace of nsp species on the grid's current leaf set (5 stage vectors of
// [N + n_need] and the ghost values per species), grown with 25 % slack.  mr_grid_build reserves it for
// all m species, so the first diffusion substep of a fresh grid does not allocate ~200 MB from the
// stream-ordered pool inside the step (1-3 ms of host time on BJ configs[3], sporadically 12-25 ms).
rd_status rock4_reserve(mr_grid* g, int nsp, cudaStream_t st) {
  const GridDev& G = g->d;
  const int64_t need = (5 * (G.N + G.n_need + 1) + 4 * G.n_if + 4) * int64_t(nsp);
  if (need > g->r4_cap) {
    if (g->r4_work) rd_free(g->r4_work, st);
    g->r4_work = nullptr;
    g->r4_cap = 0;
    const int64_t c = need + need / 4;
    RD_CUDA_TRY(rd_malloc(&g->r4_work, size_t(c) * 8, st));
    g->r4_cap = c;
  }
  return RD_OK;
}

namespace {
// pend == NULL: the results are read back (synchronises) and returned.  pend != NULL (rd_strang_step):
// they are copied asynchronously into pend->hs (pinned, owned by the caller) and rock4_finish reads
// them after the caller's single synchronisation of the step.
rd_status run_rock4(mr_grid* g, const std::vector<int>& species, const std::vector<double>& eps, double T,
                    const rd_rock4_opts& o, int forced, int fs, double fh, const double* fx, double* out,
                    double* err, rd_stats* stats, cudaStream_t st, R4Pending* pend = nullptr) {
  const double* rec_table = nullptr;
  RD_TRY(tables(&rec_table));
  GridDev& G = g->d;
  const int nsp = int(species.size());
  if (nsp == 0 || G.N == 0) return RD_OK;
  // workspace: 5 stage vectors of [N + n_need] per species (V = [leaves | needed internal nodes])
  const int64_t vl = G.N + G.n_need + 1;
  const int64_t gl = 4 * G.n_if + 4;
  const int64_t per = 5 * vl + gl;
  RD_TRY(rock4_reserve(g, nsp, st));
  // operator form: the assembled sparse matrix (2-D default; fvmat.cu) or the matrix-free stencil
  int dev = 0, nsm = 0, occ = 0;
  RD_CUDA_TRY(cudaGetDevice(&dev));
  RD_CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  bool use_mat = use_assembled_operator(g);
  const int nb_mat = kR4MatBps * nsm;
  if (use_mat) {
    RD_TRY(grid_assemble_matrix(g, nb_mat, st));
    use_mat = g->mat_state == 1;
    if (!use_mat && G.op_mode != RD_OP_PREDICTION) return RD_ENOTSUP;  // two-point forms exist only assembled
  }
  const int wk = mat_wk(G.op_mode);
  void* fn = G.dim == 2 ? (void*)k_rock4<2> : (void*)k_rock4<3>;
  int nthr = kR4Threads;
  size_t dyn = 0;
  int64_t blocks = 0;
  if (use_mat) {
    nthr = kR4MatThreads;
    dyn = size_t(g->mat_smem_words) * 4;
    bool cache = dyn <= size_t(kR4MatSmemCap);
    if (const char* e = getenv("RDMR_R4_CACHE")) cache = cache && atoi(e) != 0;
    void* fc = wk == 0 ? (void*)k_rock4_mat<true, 0> : (wk == 1 ? (void*)k_rock4_mat<true, 1> : (void*)k_rock4_mat<true, 2>);
    void* fu = wk == 0 ? (void*)k_rock4_mat<false, 0> : (wk == 1 ? (void*)k_rock4_mat<false, 1> : (void*)k_rock4_mat<false, 2>);
    if (cache) {
      fn = fc;
      RD_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kR4MatSmemCap));
      RD_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, nthr, dyn));
      cache = occ >= kR4MatBps;
    }
    if (!cache) {
      fn = fu;
      dyn = 0;
      RD_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, nthr, 0));
      if (occ < 1) return RD_ECUDA;
      blocks = int64_t(nsm) * std::min(occ, kR4MatBps);
    } else {
      blocks = nb_mat;
    }
  } else {
    RD_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, nthr, 0));
    if (occ < 1) return RD_ECUDA;
    int bps = G.dim == 3 ? RD_R4_MINB3 : RD_R4_MINB2;
    if (const char* e = getenv("RDMR_R4_BPS"))
      if (atoi(e) > 0) bps = atoi(e);
    blocks = std::min<int64_t>(int64_t(nsm) * std::min(occ, bps), std::max<int64_t>(1, (G.N + nthr - 1) / nthr));
  }
  const int64_t nch = (G.N + kR4Threads - 1) / kR4Threads;
  const int64_t npart = int64_t(nsp) * std::max<int64_t>(nch, blocks);
  if (npart + 6 * kMaxSpecies + 64 > g->r4_part_cap) {
    if (g->r4_part) rd_free(g->r4_part, st);
    g->r4_part = nullptr;
    RD_CUDA_TRY(rd_malloc(&g->r4_part, size_t(npart + 6 * kMaxSpecies + 64) * 8, st));
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
    P.sp[q].id = species[q];
  }
  P.T = T; P.rtol = o.rtol; P.atol = o.atol; P.rho1 = g->rho1;
  P.smax = std::min(o.s_max, RD_ROCK4_SMAX);
  P.rec = rec_table;
  P.part = g->r4_part;
  P.stats = reinterpret_cast<long long*>(g->r4_part + npart);
  P.tick = reinterpret_cast<unsigned int*>(P.stats + 6 * kMaxSpecies + 8);
  P.errfin = reinterpret_cast<double*>(P.stats + 6 * kMaxSpecies + 16);  // inside the 64-slot tail
  if (!g->r4_ctl) {  // per-species step-size proposals, zero until the first call ends
    RD_CUDA_TRY(rd_malloc(&g->r4_ctl, sizeof(double) * kMaxSpecies, st));
    RD_CUDA_TRY(cudaMemsetAsync(g->r4_ctl, 0, sizeof(double) * kMaxSpecies, st));
  }
  P.hprop = static_cast<double*>(g->r4_ctl);
  RD_CUDA_TRY(cudaMemsetAsync(P.tick, 0, 8 * sizeof(unsigned int), st));
  P.forced = forced; P.forced_s = fs; P.forced_h = fh; P.out = out; P.err = err;
  void* args[] = {&P};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  if (stats) {
    RD_CUDA_TRY(cudaEventCreate(&ev[0]));
    RD_CUDA_TRY(cudaEventCreate(&ev[1]));
    RD_CUDA_TRY(cudaEventRecord(ev[0], st));
  }
#ifdef RD_TRACE
  const auto t0_ = std::chrono::steady_clock::now();
#endif
  RD_CUDA_TRY(cudaLaunchCooperativeKernel(fn, dim3(unsigned(blocks)), dim3(nthr), args, dyn, st));
#ifdef RD_TRACE
  {
    const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0_).count();
    if (us > 200.0) std::fprintf(stderr, "[trace] cudaLaunchCooperativeKernel took %.0f us\n", us);
  }
#endif
  if (stats) RD_CUDA_TRY(cudaEventRecord(ev[1], st));
  RD_COUNT_LAUNCH(1);
  R4Pending local;
  R4Pending& pd = pend ? *pend : local;
  long long hs_local[6 * kMaxSpecies + 8];
  if (!pend) pd.hs = hs_local;
  pd.nsp = nsp;
  pd.ev[0] = ev[0];
  pd.ev[1] = ev[1];
  pd.rho1 = g->rho1;
  pd.mat_slots = use_mat ? g->mat_slots : 0;
  pd.armed = true;
  RD_CUDA_TRY(cudaMemcpyAsync(pd.hs, P.stats, sizeof(long long) * (6 * nsp + 7), cudaMemcpyDeviceToHost, st));
  if (pend) return RD_OK;
  RD_CUDA_TRY(cudaStreamSynchronize(st));
  return rock4_finish(pd, stats);
}

}  // namespace

bool use_assembled_operator(const mr_grid* g) {
  if (g->d.op_mode != RD_OP_PREDICTION) return true;  // the two-point forms are assembled only
  bool use_mat = g->d.dim == 2;
  if (const char* e = getenv("RDMR_R4_MODE")) use_mat = std::string(e) == "mat" ? true : (std::string(e) == "free" ? false : use_mat);
  return use_mat;
}

int assembled_launch_blocks() {
  int dev = 0, nsm = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    return 0;
  return kR4MatBps * nsm;
}

rd_status diffusion_rock4(mr_grid* g, const double* eps_diff, double T, const rd_rock4_opts* opts, rd_stats* stats,
                          cudaStream_t st, R4Pending* pend) {
  rd_rock4_opts o{1e-8, 1e-8, 200};
  if (opts) o = *opts;
  if (!g || !eps_diff || !(T > 0) || !(o.rtol > 0) || !(o.atol > 0) || o.s_max < 5) return RD_EINVAL;
  NvtxRange nvtx("rd_diffusion_rock4");
  SpanTimer span(stats, &rd_stats::diffusion_ms, st);
  std::vector<int> sp;
  std::vector<double> ep;
  for (int i = 0; i < g->d.m; ++i) {
    if (!(eps_diff[i] >= 0)) return RD_EINVAL;
    if (eps_diff[i] > 0) { sp.push_back(i); ep.push_back(eps_diff[i]); }  // eps = 0: D is the identity
  }
  return run_rock4(g, sp, ep, T, o, 0, 0, 0.0, nullptr, nullptr, nullptr, stats, st, pend);
}

}  // namespace rdmr

using namespace rdmr;

extern "C" rd_status rd_diffusion_rock4(mr_grid* g, const double* eps_diff, double T, const rd_rock4_opts* opts,
                                        rd_stats* stats, void* stream) {
  return diffusion_rock4(g, eps_diff, T, opts, stats, static_cast<cudaStream_t>(stream), nullptr);
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
