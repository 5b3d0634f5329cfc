// Microbenchmark: cost of cooperative_groups grid.sync() on the B200 vs grid size (1000 barriers).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k(int iters, double* sink) {
  cg::grid_group g = cg::this_grid();
  double a = threadIdx.x;
  for (int i = 0; i < iters; ++i) { a = a * 1.0000001 + 1e-9; g.sync(); }
  if (a == 42.0) *sink = a;
}
int main() {
  double* sink; cudaMalloc(&sink, 8);
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  for (int tpb : {128, 256, 512}) for (int bps : {1, 2, 3, 4}) {
    int blocks = nsm * bps, iters = 2000;
    void* args[] = {&iters, &sink};
    cudaLaunchCooperativeKernel((void*)k, blocks, tpb, args, 0, 0);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    cudaLaunchCooperativeKernel((void*)k, blocks, tpb, args, 0, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("tpb=%d blocks=%d  %.3f us per grid.sync  (%s)\n", tpb, blocks, 1000.0 * ms / iters, cudaGetErrorString(cudaGetLastError()));
  }
}
