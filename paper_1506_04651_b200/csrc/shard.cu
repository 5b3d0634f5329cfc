// Cost-balanced partition of the leaf order for the sharded Strang step: the
// paper splits the leaf set into contiguous intervals of its (Morton-ordered) tree;
// here the intervals are balanced by a per-cell cost (the Radau5 cost proxy or the attempt counts of the
// previous half step) instead of by cell count.
//
// Definition (exact integer arithmetic): w_c = max(cost_c, 0) + 1, S_i = sum_{c < i} w_c, W = S_n;
// bounds[k] = min{ i in [0, n] : p S_i >= k W },  k = 0..p.  bounds[0] = 0, bounds[p] = n, monotone.
#include <cub/cub.cuh>

#include "common.cuh"

namespace rdmr {
namespace {
struct Weight {
  const int32_t* cost;
  __host__ __device__ int64_t operator()(int64_t c) const { return int64_t(cost[c] > 0 ? cost[c] : 0) + 1; }
};

// incl[i] = S_{i+1}; one thread per interior bound, binary search for the first i with p S_i >= k W
__global__ void k_bounds(const int64_t* incl, int64_t n, int p, int64_t* out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x + 1;
  if (k >= p) return;
  const int64_t W = incl[n - 1];
  const int64_t target = int64_t(k) * W;  // compare p S_i >= k W
  int64_t lo = 0, hi = n;                 // S_0 = 0 < target; S_n = W: p W >= k W
  while (lo < hi) {
    const int64_t mid = (lo + hi) / 2;
    const int64_t S = mid == 0 ? 0 : incl[mid - 1];
    if (int64_t(p) * S >= target) hi = mid;
    else lo = mid + 1;
  }
  out[k] = lo;
}
}  // namespace
}  // namespace rdmr

using namespace rdmr;

extern "C" rd_status rd_shard_bounds(int64_t n, const int32_t* cost, int p, int64_t* bounds, void* stream) {
  if (n < 0 || p < 1 || p > (1 << 20) || !bounds) return RD_EINVAL;
  bounds[0] = 0;
  bounds[p] = n;
  if (p == 1) return RD_OK;
  if (!cost || n == 0) {  // uniform weights: bounds[k] = ceil(k n / p)
    for (int k = 1; k < p; ++k) bounds[k] = (int64_t(k) * n + p - 1) / p;
    return RD_OK;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cub::CountingInputIterator<int64_t> it(0);
  cub::TransformInputIterator<int64_t, Weight, cub::CountingInputIterator<int64_t>> w(it, Weight{cost});
  size_t tmp_bytes = 0;
  RD_CUDA_TRY(cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, w, static_cast<int64_t*>(nullptr), n, st));
  void* buf = nullptr;
  const size_t off = (size_t(n) * 8 + size_t(p) * 8 + 255) & ~size_t(255);
  RD_CUDA_TRY(rd_malloc(&buf, off + tmp_bytes, st));
  int64_t* incl = static_cast<int64_t*>(buf);
  int64_t* dev_b = incl + n;
  RD_CUDA_TRY(cub::DeviceScan::InclusiveSum(static_cast<char*>(buf) + off, tmp_bytes, w, incl, n, st));
  RD_COUNT_LAUNCH(2);
  k_bounds<<<unsigned((p + 126) / 128), 128, 0, st>>>(incl, n, p, dev_b);
  RD_COUNT_LAUNCH(1);
  RD_CUDA_TRY(cudaGetLastError());
  RD_CUDA_TRY(cudaMemcpyAsync(bounds + 1, dev_b + 1, size_t(p - 1) * 8, cudaMemcpyDeviceToHost, st));
  rd_free(buf, st);
  RD_CUDA_TRY(cudaStreamSynchronize(st));
  return RD_OK;
}
