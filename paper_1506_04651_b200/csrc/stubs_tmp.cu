// TEMPORARY: replaced by mr.cu / rock4.cu / strang.cu
#include "common.cuh"
extern "C" {
rd_status mr_grid_build(const mr_params*, int, const double*, void*, mr_grid**) { return RD_ENOTSUP; }
rd_status mr_adapt(mr_grid*, void*) { return RD_ENOTSUP; }
rd_status mr_grid_leaves(const mr_grid*, int64_t*, const uint64_t**, double**) { return RD_ENOTSUP; }
rd_status mr_grid_info(const mr_grid*, int64_t*, int*, int*, double*, double*) { return RD_ENOTSUP; }
void mr_grid_free(mr_grid*) {}
rd_status mr_rowmajor_to_morton(int, int, int, const double*, double*, void*) { return RD_ENOTSUP; }
rd_status rd_fv_apply(mr_grid*, const double*, double*, void*) { return RD_ENOTSUP; }
rd_status rd_diffusion_rock4(mr_grid*, const double*, double, const rd_rock4_opts*, rd_stats*, void*) { return RD_ENOTSUP; }
rd_status rd_rock4_forced_step(mr_grid*, const double*, double, double, int, double*, double*, void*) { return RD_ENOTSUP; }
rd_status rd_strang_step(mr_grid*, const rd_model*, const double*, double, int, const rd_radau5_opts*, const rd_rock4_opts*, rd_stats*, void*) { return RD_ENOTSUP; }
int rd_rock4_smax(void) { return 0; }
rd_status rd_rock4_coeffs(int, double*, double*, double*, double*, double*) { return RD_ENOTSUP; }
}
