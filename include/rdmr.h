/* rdmr.h — C-ABI of the B200-native Strang / Radau5 / Rock4 / multiresolution hot path
 * (Descombes, Duarte, Dumont, Guillet, Louvet, Massot, "Task-based adaptive multiresolution
 * for time-space multi-scale reaction-diffusion systems on multi-core architectures",
 * arXiv 1506.04651).  "P:NNN" cites a line of the paper's LaTeX source;
 * "SURVEY §x" and "DESIGN.md" name the readings this build takes where the paper is silent.
 *
 * The system (Eq. thesystem):  d u_i/dt - div(eps_i grad u_i) = f_i(u),  i = 1..m,
 * on Omega = [0,1]^d (d = 2, 3), homogeneous Neumann boundary conditions, solved by Strang
 * splitting between a per-cell stiff reaction substep (Radau5) and a
 * per-species diffusion substep (Rock4) on the leaves of a finite-volume
 * multiresolution grid adapted by Harten detail thresholding.
 *
 * Conventions (all entry points):
 *  - Device pointers are raw CUDA device addresses (e.g. torch tensor.data_ptr()); "host" says
 *    when a pointer is a host address.  Caller buffers are BORROWED for the duration of the call;
 *    the library never frees them.  Arrays of doubles must be 8-byte aligned.
 *  - stream is a cudaStream_t (NULL = legacy default stream).  Work is stream-ordered; calls that
 *    synchronise say so.
 *  - Every call returns an rd_status; no C++ exception crosses this boundary.  On RD_EINVAL
 *    nothing was enqueued and no output was modified.
 *  - A grid handle is used by one stream at a time (not re-entrant per handle).
 *  - The library never falls back to the CPU: without a CUDA device every compute call returns
 *    RD_ECUDA.
 */
#ifndef RDMR_H
#define RDMR_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------ status */
typedef int rd_status;
enum {
  RD_OK = 0,
  RD_EINVAL = -1,   /* bad argument or level cap exceeded (SURVEY §8(b) validation list)          */
  RD_ENOMEM = -2,   /* device allocation failed                                                   */
  RD_ECUDA = -3,    /* CUDA runtime error or no device                                            */
  RD_ESTIFF = -4,   /* >= 1 Radau5 cell failed (h underflow / max steps / non-finite); failed    */
                    /* cells keep their last accepted state; counted in rd_stats.n_failed         */
  RD_ESTRUCT = -5,  /* grading / tree invariant violated                              */
  RD_ENOTSUP = -6   /* valid request this build does not support                                 */
};
const char* rd_status_string(rd_status s);

/* ------------------------------------------------------------------ MR grid
 * Opaque, device resident.  Node (j, k), k in Z^d, 0 <= k_a < 2^j, is keyed level-major:
 *   key = (uint64(j) << 58) | morton_j(k)
 * where morton_j interleaves the bits of k from the most significant one with coordinate 1 (x)
 * first (§5.1; reading C10/C11).  Leaves are stored in ascending key order
 * (level-wise, Morton-minor), values as structure of arrays u[i*N + r].
 * Level cap of this build: J <= 14 (d = 2), J <= 9 (d = 3) — the per-level node maps are dense
 * (DESIGN.md "Data layout"); larger J returns RD_EINVAL. */
typedef struct mr_grid mr_grid;

typedef struct {
  int dim;        /* 2 or 3                                                                      */
  int level_min;  /* L_min: leaves never coarser than this level (BJ "coarsest level")           */
  int level_max;  /* J: finest level                                                             */
  double eps_mr;  /* Harten threshold eps; eps_j = 2^{(d/2)(j-J)} eps; 0 => uniform J    */
} mr_params;

/* Build the graded tree from level-J cell values (DESIGN.md R-B): full tree, projection
 * to all levels, details + significance, coarsening to a fixed point
 * with no refinement.
 *   u_finest: device, [m][2^{dJ}] doubles, level-J MORTON order (see mr_rowmajor_to_morton).
 * Synchronises (fixed-point termination flags, leaf count).  *out owns all its device memory,
 * including the Strang step's workspaces reserved here for the built leaf set (Rock4 stage vectors of
 * all m species, about 10 m (N + needed nodes) doubles; the reaction scheduling scratch, 16 N bytes), so
 * the first rd_strang_step / rd_diffusion_rock4 on the grid does not allocate.  RD_ENOMEM / RD_ECUDA if
 * that fails (nothing is leaked). */
rd_status mr_grid_build(const mr_params* p, int m, const double* u_finest, void* stream, mr_grid** out);

/* Re-adapt between time steps (DESIGN.md R-A): projection, details and
 * significance on the current leaf values, one-level refinement of significant leaves + graded
 * repair, prediction of new nodes (Eq. inter_1d), coarsening fixed point
 * excluding nodes created in this call, leaf compaction in key order.  Invalidates
 * previously returned leaf pointers.  Synchronises. */
rd_status mr_adapt(mr_grid* g, void* stream);

/* Leaf arrays of the grid (device, owned by the grid, valid until the next mr_adapt/mr_grid_free).
 * keys: [N] ascending; u: [m][N] writable SoA state. */
rd_status mr_grid_leaves(const mr_grid* g, int64_t* n_leaves, const uint64_t** keys, double** u);

/* n_internal: internal nodes at levels >= L_min; level_lo/hi: coarsest/finest leaf level;
 * cr = 1 - N / 2^{dJ} (compression ratio); rho1 = Gershgorin bound of the eps=1
 * FV operator (DESIGN.md R-K2).  Any output pointer may be NULL. */
rd_status mr_grid_info(const mr_grid* g, int64_t* n_internal, int* level_lo, int* level_hi, double* cr,
                       double* rho1);
void mr_grid_free(mr_grid* g);

/* Operator / storage statistics (host): out[0..n) of (N leaves, interface terms, needed internal
 * nodes, projection-expansion entries, dense map size, dim, J, L_min).  For profiling. */
rd_status mr_grid_stats(const mr_grid* g, int64_t* out, int n);

/* Key helpers (host): P:749-753.  k has dim entries. */
uint64_t mr_key_encode(int dim, int level, const int32_t* k);
void mr_key_decode(int dim, uint64_t key, int* level, int32_t* k);

/* Diffusion operator at level jumps (readings C3, R-T):
 *   RD_OP_PREDICTION (default): ghost values by the MR prediction operator (north_star);
 *   RD_OP_TWO_POINT: two-point fluxes between leaf centres (the setting of App. A, where a
 *     coefficient follows from the link type and the level), stored with explicit FP64 weights;
 *   RD_OP_TWO_POINT_COMPACT: the same operator in App. A's compact storage: per link only the column
 *     and its type (same level / to coarser / to finer), the coefficient rebuilt from the level.
 * Two-point forms always use the assembled leaf operator (d = 2 and 3).  Recompiles the operator (the
 * choice persists through mr_adapt).  RD_EINVAL for an unknown mode. */
enum { RD_OP_PREDICTION = 0, RD_OP_TWO_POINT = 1, RD_OP_TWO_POINT_COMPACT = 2 };
rd_status mr_set_operator(mr_grid* g, int mode, void* stream);

/* Layout helper: src device [m][2^{dJ}] row-major (x fastest) -> dst device [m][2^{dJ}] in
 * level-J Morton order.  Pure permutation (no arithmetic).  Stream ordered. */
rd_status mr_rowmajor_to_morton(int dim, int level, int m, const double* src, double* dst, void* stream);

/* FV diffusion operator with eps = 1 on the leaves (Eq. discretise; DESIGN.md R-F):
 * y = A x, x,y device [N].  Same-level faces: (x_N - x_C)/h_j^2; faces toward a coarser leaf use
 * the ghost value predicted by Eq. inter_1d from the coarse neighbourhood, faces toward
 * finer leaves the conservative mirror; boundary faces contribute 0 (Neumann).  Stream ordered.
 * Evaluated in the operator form rd_diffusion_rock4 uses: for d = 2 the leaf matrix assembled after each
 * build / adapt (ghost predictions and internal projections folded into the row weights; the first call
 * after an adaptation assembles it and synchronises), for d = 3 the stencils; the environment variable
 * RDMR_R4_MODE = mat | free overrides (test hook). */
rd_status rd_fv_apply(mr_grid* g, const double* x, double* y, void* stream);

/* ------------------------------------------------------------------ models
 * kind 1 Oregonator (BJ configs[0] with q as a parameter):
 *   f_a = (-q a - a b + f_c c)/mu,  f_b = (q a - a b + b(1-b))/eps_b,  f_c = b - c;  m = 3.
 * kind 2 mass action (BJ configs[4]): f = S v, v_r = rate_r prod_{reactants} u,
 *   reactants/products: host [n_reac][2] species indices, -1 = none; rate: host [n_reac].
 * kind 3 NAGUMO: m = 1, f = k_nag u^2 (1 - u) (paper: k = 10).
 * Host arrays are copied at the call. */
enum { RD_MODEL_OREGONATOR = 1, RD_MODEL_MASS_ACTION = 2, RD_MODEL_NAGUMO = 3 };
typedef struct {
  int kind;
  int m;
  double q, f_c, eps_b, mu;
  int n_reac;                 /* <= 256 */
  const int32_t* reactants;   /* host */
  const int32_t* products;    /* host */
  const double* rate;         /* host */
  double k_nag;               /* NAGUMO rate constant k (kind 3) */
} rd_model;

/* Radau5 options (DESIGN.md R-R).  rtol/atol used as given (reading C4). */
typedef struct {
  double rtol, atol;
  double h0;          /* initial step; 0 => the whole substep (reading S2) */
  int nit;            /* max simplified-Newton iterations (default 7; 1..16)             */
  int64_t max_steps;  /* attempts per cell before failure                               */
} rd_radau5_opts;

/* Rock4 options (DESIGN.md R-K): error-controlled, rtol/atol on the RMS error norm. */
typedef struct {
  double rtol, atol;
  int s_max;          /* max stage count, 5..200 */
} rd_rock4_opts;

typedef struct {
  int64_t n_cells, n_attempts, n_accept, n_reject, n_f, n_jac, n_lu, n_newton, n_failed;
  int64_t rock4_steps, rock4_rejects, rock4_matvecs;
  int64_t rock4_s_min, rock4_s_max;
  int64_t rock4_rounds;   /* lock-step stage rounds of the persistent Rock4 kernel (grid barriers/phase) */
  int64_t rock4_mat_slots; /* sliced-ELL slots of the assembled leaf operator the last Rock4 call used  */
                           /* (nonzeros + padding; 0 = matrix-free stencil form)                        */
  double rho1;
  double rock4_kernel_ms;  /* device time of the Rock4 integration kernels alone (CUDA events on the    */
                           /* call's stream; operator assembly excluded), summed over calls             */
  double reaction_ms;      /* device time of the reaction substeps (CUDA events around the Radau5        */
                           /* launch), summed over calls                                                */
  double diffusion_ms;     /* device time of the diffusion substeps (operator assembly + Rock4), summed  */
} rd_stats;

/* Reaction substep: every cell r in [0,n) independently integrates
 * y' = f(y), y = (u[0*n+r], .., u[(m-1)*n+r]), over [0, T] with Radau5 (3-stage Radau IIA,
 * simplified Newton on the transformed system with one real and one complex m x m LU,
 * embedded error estimate, step-size control).  u: device [m][n], in place.
 * cell_counters: NULL or device int32 [8][n] = (attempts, accepted, rejected, f evals,
 * Jacobians, LU pairs, Newton iterations, status) per cell ("complexity" = f evals;
 * status 0 ok, 1 max_steps, 2 step underflow 0.1 h <= t eps_mach, 3 non-finite state).
 * stats: NULL or host; the call ADDS its totals.  The call always synchronises its stream at the end
 * (to report failures) and returns RD_ESTIFF if any cell failed.  Its work counter and totals live
 * in a per-call stream-ordered scratch: concurrent calls on different streams are independent.
 * Thread safety: different grids / buffers may be used from different host threads. */
rd_status rd_reaction_radau5(int64_t n, int m, double* u, const rd_model* model, double T,
                             const rd_radau5_opts* opts, rd_stats* stats, int32_t* cell_counters,
                             void* stream);

/* Reaction on a subset of cells (the sharded Strang step: each rank integrates
 * its own interval of the leaf order).  Same method, options, statistics and status as
 * rd_reaction_radau5, for the n cells c_k = order ? order[k] : k (k < n) of a field whose species rows
 * have stride ld: species i of cell c is u[i*ld + c] (device; ld >= n and every c < ld).  A contiguous
 * interval [a, b) of a [m][N] field is (n = b - a, ld = N, u + a, order = NULL).  order: NULL or device
 * int32 [n] (distinct cells; the order only schedules, the per-cell arithmetic is unchanged).
 * cell_counters: NULL or device int32 [8][ld] with the same stride.  RD_EINVAL if ld < n. */
rd_status rd_reaction_radau5_cells(int64_t n, int64_t ld, int m, double* u, const rd_model* model, double T,
                                   const rd_radau5_opts* opts, const int32_t* order, rd_stats* stats,
                                   int32_t* cell_counters, void* stream);

/* Per-cell reaction cost proxy (the key every reaction substep of >= 65536 cells is scheduled by,
 * longest first: rd_strang_step's substeps and rd_reaction_radau5 / _cells without an order): key_c =
 * clamp(64 (log2 sum_i |f_i(u_c)| / (atol + rtol |u_ic|) + 256), 0, 65535), FP32.  u: device, stride
 * ld as above; key: device int32 [n].  m <= 4 (RD_ENOTSUP above).  Stream ordered. */
rd_status rd_reaction_cost(int64_t n, int64_t ld, int m, const double* u, const rd_model* model,
                           const rd_radau5_opts* opts, int32_t* key, void* stream);

/* Cost-balanced contiguous partition of [0, n) into p intervals (sharded Strang step):
 * with w_c = max(cost_c, 0) + 1, S_i = sum_{c<i} w_c, W = S_n:  bounds[k] = min{ i : p S_i >= k W },
 * so bounds[0] = 0, bounds[p] = n, nondecreasing, and every interval's weight is within max_c w_c of
 * W / p.  cost: device int32 [n] or NULL (w_c = 1: bounds[k] = ceil(k n / p)).  bounds: host int64
 * [p + 1].  Exact integer arithmetic (identical on every rank for identical inputs).  Synchronises
 * the stream.  RD_EINVAL for n < 0, p < 1 or bounds NULL. */
rd_status rd_shard_bounds(int64_t n, const int32_t* cost, int p, int64_t* bounds, void* stream);

/* Explicit reaction substep for non-stiff models ("any explicit Runge-Kutta method such as
 * the well-known and simple RK4", reading R-K4): every cell r in [0,n) advances
 * y' = f(y) over [0, T] by nsteps equal classical RK4 steps (nsteps < 1 is taken as 1).  u: device
 * [m][n], in place; m <= 4 (one cell per thread; RD_ENOTSUP above).  No error control and no failure
 * status: the caller keeps h |f'| inside RK4's stability interval (NAGUMO: |f'| <= 3k).
 * Stream ordered, no synchronisation. */
rd_status rd_reaction_rk4(int64_t n, int m, double* u, const rd_model* model, double T, int nsteps,
                          void* stream);

/* Diffusion substep: for each species i with eps_diff[i] > 0, integrate
 * dV/dt = eps_i A V over [0, T] on the grid's leaves with Rock4 (stage count from the Gershgorin
 * bound, orthogonal-polynomial recurrence stages + degree-4 finishing polynomial, embedded error
 * estimate, step control).  eps_diff: host [m].  Runs as one persistent cooperative kernel with a
 * device-side step controller.  Each species' first step size is the one its controller proposed when
 * the previous diffusion substep on this grid ended (T on a fresh grid; reading R-K5b); the
 * proposal is kept in the grid (device memory) and survives mr_adapt.  stats: NULL or host
 * (synchronises, adds). */
rd_status rd_diffusion_rock4(mr_grid* g, const double* eps_diff, double T, const rd_rock4_opts* opts,
                             rd_stats* stats, void* stream);

/* One forced Rock4 step (no control; pins): out = R_s(h eps A) x, err = sigma_4 (h eps A)^4 x
 * for species vector x (device [N]).  err may be NULL. */
rd_status rd_rock4_forced_step(mr_grid* g, const double* x, double eps, double h, int s, double* out,
                               double* err, void* stream);

/* Strang step: RD_STRANG_RDR: R_{dt/2} D_dt R_{dt/2} (the paper's choice, P:360-363,
 * default); RD_STRANG_DRD: D_{dt/2} R_dt D_{dt/2}.  Advances the grid's leaf values in
 * place; does not adapt (call mr_adapt after).  eps_diff: host [m].  The substeps run
 * stream-ordered; the step synchronises its stream ONCE, at its end, to read the reaction totals and
 * the Rock4 controller results (RD_ESTIFF if a cell or a species failed); stats (NULL or host) are
 * filled after that synchronisation, so requesting them adds none.  One grid: one stream at a time. */
enum { RD_STRANG_RDR = 0, RD_STRANG_DRD = 1 };
/* scheme flag: the reaction substeps use classical RK4 (rd_reaction_rk4, non-stiff models such as
 * NAGUMO) with h_max = ropts->h0 (0: one step per substep) instead of Radau5 */
enum { RD_STRANG_RK4 = 0x100 };
rd_status rd_strang_step(mr_grid* g, const rd_model* model, const double* eps_diff, double dt, int scheme,
                         const rd_radau5_opts* ropts, const rd_rock4_opts* kopts, rd_stats* stats,
                         void* stream);

/* Rock4 coefficient table compiled into the library (generated offline by
 * paper_1506_04651_b200/tools/gen_rock4.cpp): ell_s, sigma_1..4 and the n = s-4 recurrence
 * coefficients.  Host outputs, mu/nu/kappa sized s-4.  RD_EINVAL outside 5..rd_rock4_smax(). */
int rd_rock4_smax(void);

/* Cumulative number of CUDA kernel launches this library has issued in this process (host-side
 * counter; CUB scans count their kernels).  For launch accounting in benchmarks. */
int64_t rd_kernel_launches(void);
rd_status rd_rock4_coeffs(int s, double* ell, double* sigma4, double* mu, double* nu, double* kappa);

#ifdef __cplusplus
}
#endif
#endif /* RDMR_H */
