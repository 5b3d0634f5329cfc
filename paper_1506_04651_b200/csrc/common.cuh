// Internal header of the B200 library (product side; shares nothing with oracle/).
#pragma once
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>

#include <vector>

#include <nvtx3/nvToolsExt.h>
#include <stdint.h>

#include <cstdio>

#include "../../include/rdmr.h"

#define RD_CUDA_TRY(expr)                                                       \
  do {                                                                          \
    cudaError_t e_ = (expr);                                                    \
    if (e_ != cudaSuccess) {                                                    \
      std::fprintf(stderr, "rdmr: %s failed: %s (%s:%d)\n", #expr,             \
                   cudaGetErrorString(e_), __FILE__, __LINE__);                 \
      return e_ == cudaErrorMemoryAllocation ? RD_ENOMEM : RD_ECUDA;            \
    }                                                                           \
  } while (0)

#define RD_TRY(expr)              \
  do {                            \
    rd_status s_ = (expr);        \
    if (s_ != RD_OK) return s_;   \
  } while (0)

namespace rdmr {

// Device memory of the library comes from the device's default stream-ordered pool with an unbounded
// release threshold: buffers that grids grow, free and regrow (every adaptation, every fresh grid)
// are recycled inside the pool instead of going back to the driver (cudaMalloc / cudaFree stall the
// device).  Allocation and release are ordered on the call's stream.
cudaError_t pool_init();
inline cudaError_t rd_malloc(void** p, size_t bytes, cudaStream_t st) {
  cudaError_t e = pool_init();
  if (e != cudaSuccess) return e;
#ifdef RD_TRACE
  const auto t0 = std::chrono::steady_clock::now();
  e = cudaMallocAsync(p, bytes, st);
  const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
  if (us > 200.0) std::fprintf(stderr, "[trace] cudaMallocAsync %zu bytes took %.0f us\n", bytes, us);
  return e;
#else
  return cudaMallocAsync(p, bytes, st);
#endif
}
template <class T>
inline cudaError_t rd_malloc(T** p, size_t bytes, cudaStream_t st) {
  return rd_malloc(reinterpret_cast<void**>(p), bytes, st);
}
inline void rd_free(void* p, cudaStream_t st) {
  if (p) cudaFreeAsync(p, st);
}

// Device time of a span of stream work, reported into an rd_stats field when stats are requested (the
// calls that fill stats synchronise anyway).
// NVTX range over a host-side call (header-only NVTX v3: free unless a profiler is attached); lets
// nsys / ncu --nvtx attribute kernels to the R / D / A phases of a Strang step.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// Inside a SpanDefer scope (rd_strang_step) the end event is only recorded; the elapsed times are
// read after the scope's own synchronisation (SpanDefer::resolve), so requesting stats adds no host
// synchronisation to a Strang step.
struct SpanPending {
  cudaEvent_t e0, e1;
  double* out;
};
extern thread_local int g_span_defer;
extern thread_local std::vector<SpanPending> g_span_pending;
struct SpanTimer {
  cudaEvent_t e[2] = {nullptr, nullptr};
  cudaStream_t st;
  double* out;
  SpanTimer(rd_stats* s, double rd_stats::*field, cudaStream_t stream) : st(stream), out(s ? &(s->*field) : nullptr) {
    if (out && cudaEventCreate(&e[0]) == cudaSuccess && cudaEventCreate(&e[1]) == cudaSuccess) cudaEventRecord(e[0], st);
    else out = nullptr;
  }
  ~SpanTimer() {
    if (!out) return;
    cudaEventRecord(e[1], st);
    if (g_span_defer > 0) {
      g_span_pending.push_back({e[0], e[1], out});
      return;
    }
    float ms = 0.0f;
    if (cudaEventSynchronize(e[1]) == cudaSuccess && cudaEventElapsedTime(&ms, e[0], e[1]) == cudaSuccess) *out += ms;
    cudaEventDestroy(e[0]);
    cudaEventDestroy(e[1]);
  }
};
struct SpanDefer {
  SpanDefer() { ++g_span_defer; }
  ~SpanDefer() {  // (an early error return: release the events without reading them)
    if (--g_span_defer == 0) resolve(false);
  }
  // call after the stream has been synchronised
  static void resolve(bool read = true) {
    for (const SpanPending& p : g_span_pending) {
      float ms = 0.0f;
      if (read && cudaEventElapsedTime(&ms, p.e0, p.e1) == cudaSuccess) *p.out += ms;
      cudaEventDestroy(p.e0);
      cudaEventDestroy(p.e1);
    }
    g_span_pending.clear();
  }
};

// host-side count of kernel launches issued by the library (rd_kernel_launches())
extern long long g_launches;
#define RD_COUNT_LAUNCH(n) (::rdmr::g_launches += (n))

constexpr int kMaxReac = 256;
constexpr int kMaxSpecies = 32;  // warp-per-cell Radau5: one lane per species row

// Model as a by-value kernel parameter (lives in the constant bank): P:271-275 (Oregonator,
// with 1/mu and 1/eps_b pre-inverted), BJ configs[4] (mass action).
struct DevModel {
  int kind, m, n_reac;
  double q, f_c, inv_eps_b, inv_mu;
  double k_nag;  // NAGUMO (kind 3)
  int8_t reac[kMaxReac][2];
  int8_t prod[kMaxReac][2];
  double rate[kMaxReac];
  // species incidence lists for the warp kernel: f_i = sum_{e in [inc_start[i], inc_start[i+1])}
  // inc_c[e] * v_{inc_r[e]}  (stoichiometric coefficient of species i in reaction inc_r[e])
  int16_t inc_start[kMaxSpecies + 1];
  uint8_t inc_r[4 * kMaxReac];
  int8_t inc_c[4 * kMaxReac];
  // packed incidence entries (staged into shared memory by the warp kernel): rate, and
  // i0 | i1 << 8 | (coef + 8) << 16 with i = 32 for an absent reactant (a slot holding 1.0)
  int n_inc;
  double inc_rate[4 * kMaxReac];
  uint32_t inc_pack[4 * kMaxReac];
  // per reaction: i0 | i1 << 8 (32 = absent reactant slot holding 1.0); per incidence entry: the
  // reaction index and the stoichiometric coefficient as a double
  uint16_t rx_pack[kMaxReac];
  double inc_coef[4 * kMaxReac];
};

rd_status make_dev_model(const rd_model* in, DevModel* out);

// ------------------------------------------------------------------ Morton
// Within each d-bit digit group coordinate 1 (x) is the most significant bit (reading C10).
__host__ __device__ inline uint64_t spread2(uint64_t v) {  // bit b -> bit 2b
  v &= 0xffffffffull;
  v = (v | (v << 16)) & 0x0000ffff0000ffffull;
  v = (v | (v << 8)) & 0x00ff00ff00ff00ffull;
  v = (v | (v << 4)) & 0x0f0f0f0f0f0f0f0full;
  v = (v | (v << 2)) & 0x3333333333333333ull;
  v = (v | (v << 1)) & 0x5555555555555555ull;
  return v;
}
__host__ __device__ inline uint64_t squash2(uint64_t v) {
  v &= 0x5555555555555555ull;
  v = (v | (v >> 1)) & 0x3333333333333333ull;
  v = (v | (v >> 2)) & 0x0f0f0f0f0f0f0f0full;
  v = (v | (v >> 4)) & 0x00ff00ff00ff00ffull;
  v = (v | (v >> 8)) & 0x0000ffff0000ffffull;
  v = (v | (v >> 16)) & 0x00000000ffffffffull;
  return v;
}
__host__ __device__ inline uint64_t spread3(uint64_t v) {  // bit b -> bit 3b (21 bits)
  v &= 0x1fffffull;
  v = (v | (v << 32)) & 0x1f00000000ffffull;
  v = (v | (v << 16)) & 0x1f0000ff0000ffull;
  v = (v | (v << 8)) & 0x100f00f00f00f00full;
  v = (v | (v << 4)) & 0x10c30c30c30c30c3ull;
  v = (v | (v << 2)) & 0x1249249249249249ull;
  return v;
}
__host__ __device__ inline uint64_t squash3(uint64_t v) {
  v &= 0x1249249249249249ull;
  v = (v | (v >> 2)) & 0x10c30c30c30c30c3ull;
  v = (v | (v >> 4)) & 0x100f00f00f00f00full;
  v = (v | (v >> 8)) & 0x1f0000ff0000ffull;
  v = (v | (v >> 16)) & 0x1f00000000ffffull;
  v = (v | (v >> 32)) & 0x1fffffull;
  return v;
}
template <int D>
__host__ __device__ inline uint64_t morton_enc(const int* k) {
  if (D == 2) return (spread2(uint64_t(k[0])) << 1) | spread2(uint64_t(k[1]));
  return (spread3(uint64_t(k[0])) << 2) | (spread3(uint64_t(k[1])) << 1) | spread3(uint64_t(k[2]));
}
template <int D>
__host__ __device__ inline void morton_dec(uint64_t s, int* k) {
  if (D == 2) {
    k[0] = int(squash2(s >> 1));
    k[1] = int(squash2(s));
  } else {
    k[0] = int(squash3(s >> 2));
    k[1] = int(squash3(s >> 1));
    k[2] = int(squash3(s));
  }
}
constexpr int kLevelShift = 58;

}  // namespace rdmr
