// Strang splitting step (§2.1): RDR  U_{n+1} = R_{dt/2} D_dt R_{dt/2} U_n  (the paper's
// choice: it ends with the stiffest substep) or DRD  D_{dt/2} R_dt D_{dt/2}.
// R = per-leaf Radau5 on the grid's leaf array, D = Rock4 persistent kernel.
//
// Scheduling: every reaction substep takes its cells longest-first (LPT) by the cost proxy of the state
// it starts from (k_cost_proxy), so the costly cells near the fronts start early instead of forming the
// kernel's tail, and the lanes of a warp hold cells of similar cost.  The arithmetic per cell is unchanged.
#include <cub/cub.cuh>

#include <cmath>

#include "mr.cuh"

namespace rdmr {
rd_status diffusion_rock4(mr_grid* g, const double* eps_diff, double T, const rd_rock4_opts* opts, rd_stats* stats,
                          cudaStream_t st, R4Pending* pend);
rd_status reaction_rk4(int64_t n, int m, double* u, const rd_model* model, double T, int nsteps, cudaStream_t st);
rd_status reaction_cost_keys(int64_t n, int m, const double* u, const rd_model* model, const rd_radau5_opts* opts,
                             int32_t* key, cudaStream_t st, int64_t ld = -1, bool sched = false);
rd_status reaction_radau5(int64_t n, int m, double* u, const rd_model* model, double T, const rd_radau5_opts* opts,
                          rd_stats* stats, int32_t* cell_counters, const int32_t* order, cudaStream_t st,
                          int64_t ld = -1, unsigned long long* acc = nullptr);
void add_radau5_totals(rd_stats* stats, const unsigned long long* tot);

namespace {
constexpr int64_t kLptMinCells = 65536;
__global__ void k_iota(int32_t* v, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    v[i] = int32_t(i);
}

// Scratch for the LPT order: cost keys [N] (lpt_cnt), sort keys/values.
rd_status lpt_scratch(mr_grid* g, int64_t n, cudaStream_t st) {
  if (n <= g->cap_lpt) return RD_OK;
  rd_free(g->lpt_cnt, st);
  rd_free(g->lpt_keys, st);
  rd_free(g->lpt_iota, st);
  rd_free(g->lpt_order, st);
  rd_free(g->lpt_tmp, st);
  g->lpt_cnt = g->lpt_keys = g->lpt_iota = g->lpt_order = nullptr;
  g->lpt_tmp = nullptr;
  const int64_t c = n + n / 4 + 1024;
  RD_CUDA_TRY(rd_malloc(&g->lpt_cnt, size_t(c) * 4, st));
  RD_CUDA_TRY(rd_malloc(&g->lpt_keys, size_t(c) * 4, st));
  RD_CUDA_TRY(rd_malloc(&g->lpt_iota, size_t(c) * 4, st));
  RD_CUDA_TRY(rd_malloc(&g->lpt_order, size_t(c) * 4, st));
  size_t bytes = 0;
  RD_CUDA_TRY(cub::DeviceRadixSort::SortPairsDescending(nullptr, bytes, g->lpt_cnt, g->lpt_keys, g->lpt_iota,
                                                         g->lpt_order, c));
  RD_CUDA_TRY(rd_malloc(&g->lpt_tmp, bytes, st));
  g->lpt_tmp_bytes = bytes;
  g->cap_lpt = c;
  return RD_OK;
}

// Once-per-step status buffers (device Radau5 accumulator, pinned host copies).
rd_status status_buffers(mr_grid* g) {
  if (!g->r5_acc) RD_CUDA_TRY(cudaMalloc(&g->r5_acc, 16 * sizeof(unsigned long long)));
  if (!g->r5_host) RD_CUDA_TRY(cudaMallocHost(&g->r5_host, 16 * sizeof(unsigned long long)));
  if (!g->r4_host) RD_CUDA_TRY(cudaMallocHost(&g->r4_host, 2 * kR4HostWords * sizeof(long long)));
  return RD_OK;
}

}  // namespace

// Workspaces of a Strang step on the grid's current leaf set, allocated ahead of the first step
// (mr_grid_build): the Rock4 stage vectors of all species, the longest-first order scratch, the
// once-per-step status buffers.
rd_status rock4_reserve(mr_grid* g, int nsp, cudaStream_t st);
rd_status grid_reserve_step_workspace(mr_grid* g, cudaStream_t st) {
  RD_TRY(rock4_reserve(g, g->d.m, st));
  if (g->d.N >= kLptMinCells) RD_TRY(lpt_scratch(g, g->d.N, st));
  return status_buffers(g);
}

namespace {
// order = cells sorted by descending cost key (lpt_cnt; stable for ties).
rd_status lpt_order(mr_grid* g, int64_t n, cudaStream_t st, int bits) {
  k_iota<<<unsigned((n + 255) / 256), 256, 0, st>>>(g->lpt_iota, n);
  RD_COUNT_LAUNCH(1);
  size_t bytes = g->lpt_tmp_bytes;
  RD_CUDA_TRY(cub::DeviceRadixSort::SortPairsDescending(g->lpt_tmp, bytes, g->lpt_cnt, g->lpt_keys, g->lpt_iota,
                                                         g->lpt_order, n, 0, bits, st));
  RD_COUNT_LAUNCH(2 + (bits + 7) / 8);  // onesweep histogram, scan + one pass per 8 key bits
  return RD_OK;
}
}  // namespace
}  // namespace rdmr

using namespace rdmr;

extern "C" rd_status rd_strang_step(mr_grid* g, const rd_model* model, const double* eps_diff, double dt, int scheme,
                                    const rd_radau5_opts* ropts, const rd_rock4_opts* kopts, rd_stats* stats,
                                    void* stream) {
  const bool rk4 = (scheme & RD_STRANG_RK4) != 0;
  scheme &= ~RD_STRANG_RK4;
  if (!g || !model || !eps_diff || !(dt > 0) || (scheme != RD_STRANG_RDR && scheme != RD_STRANG_DRD)) return RD_EINVAL;
  if (model->m != g->d.m) return RD_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  NvtxRange nvtx("rd_strang_step");
  const int64_t n = g->d.N;
  double* u = g->d.u;
  const int m = g->d.m;
  rd_status rc[3];
  if (rk4) {  // explicit reaction substeps (non-stiff models): h_max = ropts->h0 (reading R-K4)
    const double hmax = ropts ? ropts->h0 : 0.0;
    auto nsub = [&](double T) { return hmax > 0.0 ? int(std::ceil(T / hmax)) : 1; };
    auto react = [&](double T) -> rd_status {
      SpanTimer span(stats, &rd_stats::reaction_ms, st);
      return reaction_rk4(n, m, u, model, T, nsub(T), st);
    };
    if (scheme == RD_STRANG_RDR) {
      RD_TRY(react(0.5 * dt));
      rc[1] = diffusion_rock4(g, eps_diff, dt, kopts, stats, st, nullptr);
      if (rc[1] != RD_OK && rc[1] != RD_ESTIFF) return rc[1];
      RD_TRY(react(0.5 * dt));
    } else {
      rc[1] = diffusion_rock4(g, eps_diff, 0.5 * dt, kopts, stats, st, nullptr);
      if (rc[1] != RD_OK && rc[1] != RD_ESTIFF) return rc[1];
      RD_TRY(react(dt));
      const rd_status r3 = diffusion_rock4(g, eps_diff, 0.5 * dt, kopts, stats, st, nullptr);
      if (r3 != RD_OK) return r3;
    }
    return rc[1];
  }
  // Radau5 totals accumulate on the device and the Rock4 results are copied asynchronously: the step
  // synchronises once, at its end, to report failures (RD_ESTIFF) and fill stats.
  SpanDefer defer;  // phase timers of the substeps are read after the step's single synchronisation
  RD_TRY(status_buffers(g));
  unsigned long long* acc = g->r5_acc;
  RD_CUDA_TRY(cudaMemsetAsync(acc, 0, 16 * sizeof(unsigned long long), st));
  R4Pending pd[2];
  pd[0].hs = g->r4_host;
  pd[1].hs = g->r4_host + kR4HostWords;
  rd_status rc0 = RD_OK;
  // Longest-first order of a reaction substep from the cost proxy of the state it starts from (the
  // attempt counts of the first half step do not predict the second's: after the diffusion substep
  // their correlation on cfg 4 is 0.26 / -0.09, tools/r5_halves.py).  NULL: natural order.
  RD_TRY(lpt_scratch(g, n, st));
  // (with at most one cell per resident lane every cell starts at once: the order cannot pay for its sort)
  const bool use_lpt = n >= kLptMinCells && getenv("RDMR_NO_PROXY_LPT") == nullptr;
  const bool sched_key = getenv("RDMR_LPT_KEY16") == nullptr;  // 31-bit scheduling key (radau5.cu k_cost_proxy)
  auto proxy_order = [&](const int32_t** order) -> rd_status {
    *order = nullptr;
    if (!use_lpt || reaction_cost_keys(n, m, u, model, ropts, g->lpt_cnt, st, -1, sched_key) != RD_OK) return RD_OK;
    RD_TRY(lpt_order(g, n, st, sched_key ? 31 : 16));
    *order = g->lpt_order;
    return RD_OK;
  };
  const int32_t* order = nullptr;
  if (scheme == RD_STRANG_RDR) {
    RD_TRY(proxy_order(&order));
    RD_TRY(reaction_radau5(n, m, u, model, 0.5 * dt, ropts, stats, nullptr, order, st, -1, acc));
    rc0 = diffusion_rock4(g, eps_diff, dt, kopts, stats, st, &pd[0]);
    if (rc0 == RD_OK) {
      RD_TRY(proxy_order(&order));
      rc0 = reaction_radau5(n, m, u, model, 0.5 * dt, ropts, stats, nullptr, order, st, -1, acc);
    }
  } else {
    rc0 = diffusion_rock4(g, eps_diff, 0.5 * dt, kopts, stats, st, &pd[0]);
    if (rc0 == RD_OK) {
      RD_TRY(proxy_order(&order));
      rc0 = reaction_radau5(n, m, u, model, dt, ropts, stats, nullptr, order, st, -1, acc);
    }
    if (rc0 == RD_OK) rc0 = diffusion_rock4(g, eps_diff, 0.5 * dt, kopts, stats, st, &pd[1]);
  }
  RD_CUDA_TRY(cudaMemcpyAsync(g->r5_host, acc + 1, 9 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
  RD_CUDA_TRY(cudaStreamSynchronize(st));
  SpanDefer::resolve();
  add_radau5_totals(stats, g->r5_host);
  const rd_status r4a = rock4_finish(pd[0], stats), r4b = rock4_finish(pd[1], stats);
  if (rc0 != RD_OK) return rc0;
  if (g->r5_host[7] || r4a == RD_ESTIFF || r4b == RD_ESTIFF) return RD_ESTIFF;
  return RD_OK;
}
