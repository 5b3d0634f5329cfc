// Strang splitting step (§2.1): RDR  U_{n+1} = R_{dt/2} D_dt R_{dt/2} U_n  (the paper's
// choice: it ends with the stiffest substep) or DRD  D_{dt/2} R_dt D_{dt/2}.
// R = per-leaf Radau5 on the grid's leaf array (rd_reaction_radau5), D = Rock4 persistent kernel.
#include "mr.cuh"

namespace rdmr {
rd_status diffusion_rock4(mr_grid* g, const double* eps_diff, double T, const rd_rock4_opts* opts, rd_stats* stats,
                          cudaStream_t st);
}

using namespace rdmr;

extern "C" rd_status rd_strang_step(mr_grid* g, const rd_model* model, const double* eps_diff, double dt, int scheme,
                                    const rd_radau5_opts* ropts, const rd_rock4_opts* kopts, rd_stats* stats,
                                    void* stream) {
  if (!g || !model || !eps_diff || !(dt > 0) || (scheme != RD_STRANG_RDR && scheme != RD_STRANG_DRD)) return RD_EINVAL;
  if (model->m != g->d.m) return RD_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t n = g->d.N;
  double* u = g->d.u;
  rd_status rc[3];
  if (scheme == RD_STRANG_RDR) {
    rc[0] = rd_reaction_radau5(n, g->d.m, u, model, 0.5 * dt, ropts, stats, nullptr, stream);
    if (rc[0] != RD_OK && rc[0] != RD_ESTIFF) return rc[0];
    rc[1] = diffusion_rock4(g, eps_diff, dt, kopts, stats, st);
    if (rc[1] != RD_OK && rc[1] != RD_ESTIFF) return rc[1];
    rc[2] = rd_reaction_radau5(n, g->d.m, u, model, 0.5 * dt, ropts, stats, nullptr, stream);
  } else {
    rc[0] = diffusion_rock4(g, eps_diff, 0.5 * dt, kopts, stats, st);
    if (rc[0] != RD_OK && rc[0] != RD_ESTIFF) return rc[0];
    rc[1] = rd_reaction_radau5(n, g->d.m, u, model, dt, ropts, stats, nullptr, stream);
    if (rc[1] != RD_OK && rc[1] != RD_ESTIFF) return rc[1];
    rc[2] = diffusion_rock4(g, eps_diff, 0.5 * dt, kopts, stats, st);
  }
  for (rd_status r : rc)
    if (r != RD_OK) return r;
  return RD_OK;
}
