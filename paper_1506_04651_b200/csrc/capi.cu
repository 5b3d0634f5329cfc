// C-ABI entry points that are not tied to one kernel family: status strings, key helpers
// (reading C10/C11).
#include "common.cuh"

namespace rdmr {
long long g_launches = 0;
thread_local int g_span_defer = 0;
thread_local std::vector<SpanPending> g_span_pending;

cudaError_t pool_init() {
  static int done_dev = -1;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess || done_dev == dev) return e;
  cudaMemPool_t pool;
  e = cudaDeviceGetDefaultMemPool(&pool, dev);
  if (e != cudaSuccess) return e;
  uint64_t thr = ~0ull;
  e = cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  if (e == cudaSuccess) done_dev = dev;
  return e;
}
}

using namespace rdmr;

extern "C" int64_t rd_kernel_launches(void) { return g_launches; }

extern "C" const char* rd_status_string(rd_status s) {
  switch (s) {
    case RD_OK: return "ok";
    case RD_EINVAL: return "invalid argument";
    case RD_ENOMEM: return "out of device memory";
    case RD_ECUDA: return "CUDA error";
    case RD_ESTIFF: return "Radau5 failed on at least one cell";
    case RD_ESTRUCT: return "grid structure invariant violated";
    case RD_ENOTSUP: return "not supported";
    default: return "unknown status";
  }
}

extern "C" uint64_t mr_key_encode(int dim, int level, const int32_t* k) {
  if ((dim != 2 && dim != 3) || level < 0 || !k) return ~0ull;
  int kk[3] = {k[0], k[1], dim == 3 ? k[2] : 0};
  const uint64_t s = dim == 2 ? morton_enc<2>(kk) : morton_enc<3>(kk);
  return (uint64_t(level) << kLevelShift) | s;
}

extern "C" void mr_key_decode(int dim, uint64_t key, int* level, int32_t* k) {
  if ((dim != 2 && dim != 3) || !level || !k) return;
  *level = int(key >> kLevelShift);
  const uint64_t s = key & ((1ull << kLevelShift) - 1);
  int kk[3] = {0, 0, 0};
  if (dim == 2) morton_dec<2>(s, kk);
  else morton_dec<3>(s, kk);
  for (int a = 0; a < dim; ++a) k[a] = kk[a];
}
