/*
 * sfb.h — C ABI of the B200-native batched Safety-Filter (SF) solver.
 *
 * The reference has no FFI: its SF is the Python call
 *   swarmplan.solver.solve_batch(init, sys, mode, cfg=None, cache=None)
 *   (/root/reference/pkg/src/swarmplan/solver.py:286-355)
 * with the factorization object KktCache (solver.py:64-91). These entry points
 * are what a binding of that call needs (INTEGRATION.md shows the ctypes stub
 * the Python drop-in `paper_2510_09204_b200.solver` uses):
 *
 *   sfb_plan_create   replaces KktCache.__init__ (solver.py:68-86): builds the
 *                     Kronecker-compressed KKT inverse blocks on the host in FP64,
 *                     checks cond(M) > 1e14 -> SFB_ESETUP, uploads constants.
 *   sfb_solve         replaces the solve_batch loop (solver.py:297-355) for a batch
 *                     of members (instance x sample): stream-ordered, no host sync.
 *   sfb_plan_destroy  frees the plan.
 *   sfb_last_error    thread-local message of the last failing call.
 *
 * Layouts (all row-major, FP64 unless noted, DEVICE pointers in sfb_batch /
 * sfb_out): member-contiguous coefficients [B][n_d][n][n_basis] — the reference's
 * (n_d, n*n_basis, B) with the batch axis moved first. All buffers are owned by
 * the caller; the plan is immutable after creation and may be shared by
 * concurrent sfb_solve calls on different streams.
 */
#ifndef SFB_H
#define SFB_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SFB_ABI_VERSION 1

/* status codes (return values) */
#define SFB_OK        0
#define SFB_EINVAL    1   /* bad argument / unsupported shape  (reference: ShapeError/UsageError) */
#define SFB_ESETUP    2   /* KKT singular or near-singular     (reference: SetupError, solver.py:82-83) */
#define SFB_ECUDA     3   /* CUDA runtime error                 */
#define SFB_ENOMEM    4

/* objective kinds (reference ObjectiveMode.kind, solver.py:44-61) */
#define SFB_MODE_PROJECTION 0
#define SFB_MODE_SMOOTHNESS 1

/* per-member solve status (reference SolverResult.status, solver.py:112) */
#define SFB_STATUS_MAX_ITERS        0
#define SFB_STATUS_CONVERGED_PRIMAL 1
#define SFB_STATUS_CONVERGED_FP     2

typedef struct sfb_dims {
  int32_t n;          /* robots                                  (SystemDims.n)        */
  int32_t n_d;        /* workspace axes, 2 or 3                  (SystemDims.n_d)      */
  int32_t n_basis;    /* Bernstein coefficients per axis         (SystemDims.n_basis)  */
  int32_t num_steps;  /* grid points K+1                         (SystemDims.num_steps)*/
  int32_t n_obs;      /* obstacles                               (SystemDims.n_obs)    */
  int32_t n_bnd;      /* boundary rows per robot: 6 rest-to-rest, 2 otherwise (a_rows/n) */
} sfb_dims;

typedef struct sfb_plan sfb_plan;

/* Host inputs (FP64, row-major):
 *   W    [num_steps][n_basis]  position basis (BasisMatrices.W)
 *   Wdd  [num_steps][n_basis]  acceleration basis (smoothness mode), may be NULL in projection mode
 *   E    [n_bnd][n_basis]      per-robot boundary rows, A = I_n (x) E (constraints.py:111-115)
 * rho > 0 (SolverConfig.rho). Must be called with the target device current. */
int sfb_plan_create(sfb_plan** out, const sfb_dims* dims, const double* W, const double* Wdd,
                    const double* E, double rho, int32_t mode);
void sfb_plan_destroy(sfb_plan* plan);
/* cond(M) of the full KKT matrix, as np.linalg.cond would report it */
double sfb_plan_cond(const sfb_plan* plan);

/* sfb_batch.flags */
#define SFB_BATCH_STATIC_OBSTACLES 1  /* caller guarantees obs_pos is constant over the steps */

typedef struct sfb_batch {
  int32_t n_members;               /* B                                                   */
  int32_t n_instances;             /* I (distinct constraint systems)                     */
  const int32_t* member_instance;  /* [B] instance of each member                         */
  const double* xi0;               /* [B][n_d][n][n_basis] warm start                     */
  const double* lam0;              /* [B][n_d][n][n_basis]                                */
  const double* target;            /* [B][n_d][n][n_basis]; NULL in smoothness mode       */
  const double* bvals;             /* [I][n_d][n][n_bnd]  = ConstraintSystem.b per axis   */
  const double* box;               /* [I][2][n_d]  (p_min, p_max) from ConstraintSystem.h */
  const double* obs_pos;           /* [I][n_d][n_obs][num_steps] ConstraintSystem.obs_pos */
  const double* obs_axes;          /* [I][n_obs][3]  ConstraintSystem.obs_axes            */
  const double* pair_axes;         /* [I][3]         ConstraintSystem.pair_axes           */
  int32_t flags;                   /* SFB_BATCH_* hints                                   */
} sfb_batch;

typedef struct sfb_config {
  double rho;          /* must equal the plan's rho */
  double primal_tol;
  double fp_tol;
  double d_max;        /* ConstraintSystem.d_max */
  int32_t max_iters;
  int32_t early_exit;  /* 1: reference convergence tests; 0: exactly max_iters+1 map evaluations */
  int32_t cluster;     /* CTAs per member (1..8, a thread-block cluster splitting the time
                          axis); 0 = auto: small batches spread over more SMs for latency.
                          Results are bitwise reproducible for a fixed cluster size and agree
                          across sizes to rounding (~1e-15). */
} sfb_config;

typedef struct sfb_out {
  double* xi;          /* [B][n_d][n][n_basis] */
  double* lam;         /* [B][n_d][n][n_basis] */
  double* primal;      /* [B]  trace[-1, 0]    */
  double* eq_max;      /* [B]  eq_violation_max */
  int32_t* iterations; /* [B]  len(trace) - 1  */
  int32_t* status;     /* [B]  SFB_STATUS_*    */
  double* trace;       /* [B][max_iters+1][2] (primal, fixed-point residual) or NULL */
  uint64_t* counters;  /* [B][4] or NULL: exact rows evaluated, active rows, rows screened, map evaluations */
} sfb_out;

/* Stream-ordered solve (stream = cudaStream_t, NULL = legacy default). */
int sfb_solve(const sfb_plan* plan, const sfb_batch* batch, const sfb_config* cfg,
              const sfb_out* out, void* stream);

/* Post-solve epilogue of the reference's time scaling (basis.py:119-142): per member, the
 * largest speed and acceleration norm over robots and the dense grid rows of Wd / Wdd
 * ([k_dense][n_basis], FP64). coeffs [B][n_d][n][n_basis]; all pointers on the device. */
int sfb_kinematic_peaks(const double* coeffs, int32_t n_members, int32_t n_d, int32_t n,
                        int32_t n_basis, const double* Wd, const double* Wdd, int32_t k_dense,
                        double* vmax, double* amax, void* stream);

/* Post-solve trajectory metrics of the reference (replaces metrics.py:48-87, compute_metrics),
 * per member: out[b][5] = smoothness, arc_length, min_pairwise_clearance,
 * avg_pairwise_distance, min_obstacle_clearance (inf where the reference reports inf).
 * coeffs [B][n_d][n][n_basis]; Wdd [k_grid][n_basis] on the basis grid; W_dense
 * [k_dense][n_basis] and t_dense [k_dense] on the dense grid (dense_basis, metrics.py:40-44);
 * obs [n_obs][3][n_d] = center, velocity, radii[:n_d] per obstacle, member b reading
 * obs + b * obs_member_stride (0 = shared by all members); work holds
 * sfb_trajectory_metrics_work(...) doubles. All pointers on the device; bitwise reproducible. */
int sfb_trajectory_metrics(const double* coeffs, int32_t n_members, int32_t n_d, int32_t n,
                           int32_t n_basis, const double* Wdd, int32_t k_grid,
                           const double* W_dense, const double* t_dense, int32_t k_dense,
                           const double* obs, int32_t n_obs, int64_t obs_member_stride,
                           double* work, double* out, void* stream);
/* Scratch size (doubles) of sfb_trajectory_metrics, -1 if the shape is unsupported. */
int64_t sfb_trajectory_metrics_work(int32_t n_members, int32_t n_d, int32_t n, int32_t n_basis,
                                    int32_t k_dense, int32_t n_obs);

/* Analysis intermediates of one map evaluation's INPUT coefficients, as the reference's
 * fixed_point_step returns them (solver.py:246-256 -> _analyze, solver.py:158-169): the
 * spherical variables of every separation row (extract_spherical, constraints.py:195-213,
 * the reference's atan2 / sin / cos closed forms) and the workspace slack
 * s = max(0, h - G xi) (solver.py:166-167). coeffs [B][n_d][n][n_basis]; member b reads
 * instance member_instance[b] of pair_axes [I][3], obs_axes [I][n_obs][3],
 * obs_pos [I][n_d][n_obs][num_steps] and box [I][2][n_d]; W [num_steps][n_basis].
 * Outputs in the reference's layouts (batch axis last): alpha, beta, d [n_pairs][num_steps][B]
 * (pairs i < j, lexicographic), alpha_o, beta_o, d_o [n][n_obs][num_steps][B],
 * s [n_d][2 n num_steps][B]. All pointers on the device; stream-ordered. */
int sfb_analysis_vars(const double* coeffs, int32_t n_members, const int32_t* member_instance,
                      int32_t n_d, int32_t n, int32_t n_basis, int32_t num_steps, int32_t n_obs,
                      const double* W, const double* pair_axes, const double* obs_axes,
                      const double* obs_pos, const double* box, double d_max, double* alpha,
                      double* beta, double* d, double* alpha_o, double* beta_o, double* d_o,
                      double* s, void* stream);

/* Dynamic shared memory one member needs (0 if the shape is unsupported). */
int64_t sfb_smem_bytes(const sfb_plan* plan);

/* Launch shape sfb_solve would use for n_members members with sfb_config.cluster = cluster and
 * sfb_batch.flags = flags: the cluster size (auto-resolved when cluster <= 0), the dynamic shared
 * memory per CTA and how many such CTAs one SM holds (capacity planning; no launch). */
int sfb_launch_info(const sfb_plan* plan, int32_t n_members, int32_t cluster, int32_t flags,
                    int32_t* cluster_out, int32_t* smem_out, int32_t* ctas_per_sm);

const char* sfb_last_error(void);
int32_t sfb_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SFB_H */
