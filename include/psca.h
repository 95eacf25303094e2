/*
 * psca.h -- C ABI of the B200-native PSCA activity-detection hot path.
 *
 * The reference (arXiv 2503.15259, /root/reference/pkg/src/actdet) is a pure
 * Python package; its "operator API" for this path is the set of Python
 * solver functions listed below.  Each entry point here replaces one of them
 * (reference file:line in the comment) and is what a ctypes / cffi binding in
 * the reference package would call.
 *
 * Conventions
 *   - every pointer is a DEVICE pointer (cudaMalloc'd or a torch CUDA tensor's
 *     data_ptr) unless the comment says otherwise; complex128 arrays are
 *     interleaved (re, im) doubles, C order, exactly numpy's complex128 layout,
 *     and must be 16-byte aligned (the kernels load them as 16-byte vectors;
 *     a misaligned complex array or workspace is rejected with PSCA_E_ARG);
 *   - batched arrays carry a leading instance dimension B;
 *   - `stream` is a cudaStream_t passed as void* (0 = legacy default stream);
 *     every call is stream-ordered and re-entrant per stream, allocates
 *     nothing, and uses only the caller's workspace;
 *   - return value: PSCA_OK or a negative PSCA_E* code (argument / launch
 *     errors).  Numerical failures never fail the call: they are reported per
 *     instance in `status` (mirroring psca_run's trace.meta["abort"]).
 */
#ifndef PSCA_H
#define PSCA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PSCA_OK 0
#define PSCA_E_ARG (-1)       /* bad shape / kind / pointer                  */
#define PSCA_E_CUDA (-2)      /* kernel launch or CUDA runtime failure       */
#define PSCA_E_WORKSPACE (-3) /* workspace smaller than *_workspace_bytes()  */
#define PSCA_E_UNSUPPORTED (-4)

/* problem kinds: estimators.py:27 KINDS */
#define PSCA_ML_K 0
#define PSCA_MAP_K 1
#define PSCA_ML_UD 2
#define PSCA_MAP_UR 3

/* per-instance status (estimators.py:263-271, 285-286) */
#define PSCA_RUNNING 0     /* ran to max_iter                                 */
#define PSCA_CHOL_FAIL 1   /* Sigma not numerically PD (ConditioningError)    */
#define PSCA_QFLOOR 2      /* min q < 0.5 L / ||Sigma||_F                      */
#define PSCA_CONVERGED 3   /* update_norm < tol                               */

/* Smoothed effective-pathloss prior, plain scalars (priors.py:173-281).
 * phi(d) = p_lin * (k d)^-eta; area2 = d_outer^2 - d_inner^2;
 * cv, cw = density value / slope targets of the Hermite bridge at g_low. */
typedef struct {
    double eps, g_low, g_high, dead_zone_grad;
    double p_lin, k, eta, area2, cv, cw;
} psca_eff_prior;

/* Arguments of psca_solve (estimators.py:239-289 psca_run, batched;
 * unroll.py:69-73 forward is the same call with explicit steps and tol=0). */
typedef struct {
    int kind;               /* PSCA_ML_K .. PSCA_MAP_UR                         */
    int B, N, L;            /* instances, devices, pilot length                 */
    int n_antennas;         /* M (MAP prior scale 1/M)                          */
    int max_iter;           /* T                                               */
    double tol;             /* early stop on update_norm < tol (0 = never)     */
    int record_objective;   /* estimators.py:279-280                           */
    int n_chunks;           /* column chunks per instance; 0 = automatic       */
    const double* pilots;   /* [B][L][N] complex128                            */
    const double* gains;    /* [B][N]   (known-pathloss kinds; else may be 0)  */
    const double* emp_cov;  /* [B][L][L] complex128                            */
    const double* noise;    /* [B] sigma^2 > 0                                 */
    const double* steps;    /* [max_iter] rho_k in (0,1]                       */
    const double* prior_lin;/* map-k: [N] = -log(p/(1-p))/M  (priors.py:154-158) */
    const double* prior_p;  /* map-ur: [N] activation probabilities p_n      */
    psca_eff_prior eff;     /* map-ur prior scalars                            */
    /* map-k with a pairwise MVB prior (priors.py:56-151, group activity): the
     * gradient term is -(c1 + c2 x)/M at every iterate (priors.py:154-159)
     * instead of the constant prior_lin.  c2 is the symmetric N x N
     * interaction matrix in CSR form (zero diagonal).  All four null for the
     * independent prior. */
    const double* prior_c1;       /* [N]                                      */
    const int* prior_c2_indptr;   /* [N+1]                                    */
    const int* prior_c2_indices;  /* [nnz]                                    */
    const double* prior_c2_data;  /* [nnz]                                    */
    double* x_out;          /* [B][N]  final estimate (trace.final)            */
    double* update_norm;    /* [B][max_iter]                                    */
    double* objective;      /* [B][max_iter] or 0                              */
    double* iterates;       /* [B][max_iter+1][N] or 0                         */
    int* status;            /* [B]                                             */
    int* n_iter;            /* [B] completed iterations                        */
    double* cond_est;       /* [B] condition estimate at a Cholesky abort       */
    /* Fault injection (test seam; the device-side counterpart of the
     * reference test that monkeypatches CovState.build to raise,
     * test_estimators.py:268-279): 0 = off; k >= 1 makes the factorisation
     * that opens iteration k-1 report PSCA_CHOL_FAIL for every instance still
     * running (cond_est = +inf), exactly as a non-positive pivot would. */
    int fault_iter;
    /* Per-instance step schedules: 0 = every instance uses steps[0..max_iter);
     * otherwise instance b uses steps[b*steps_stride + k] (steps_stride >=
     * max_iter).  Lets one batched forward evaluate several candidate PSCA-Net
     * step vectors at once (unroll.py:131-172 evaluates them one by one). */
    int steps_stride;
} psca_solve_args;

/* Workspace (device bytes) psca_solve needs for these arguments. */
size_t psca_solve_workspace_bytes(const psca_solve_args* a);

/* The PSCA iteration for a batch of independent instances
 * (replaces estimators.psca_run, estimators.py:239-289, and
 *  unroll.forward, unroll.py:69-73). */
int psca_solve(const psca_solve_args* a, void* workspace, size_t workspace_bytes, void* stream);

/* Sigma_hat = Y Y^H / n_antennas  (sysmodel.py:244-248 empirical_cov), on DMMA.
 * y: [B][L][Mc] complex128 -> out: [B][L][L] complex128. */
int psca_empirical_cov(const double* y, int B, int L, int Mc, int n_antennas, double* out,
                       void* stream);

/* Received signal of a scene batch: Y = S[:, active] diag(sqrt(g[active])) H + Z
 * (sysmodel.py:230-241; the draws stay on the host -- the Philox streams are
 * the scene contract -- and the GEMM runs on DMMA).  pilots [B][L][N],
 * active [B][K] (int32 device indices), gains [B][N], h [B][K][M], z [B][L][M]
 * complex128 -> y [B][L][M]. */
int psca_received(const double* pilots, const int* active, const double* gains, const double* h,
                  const double* z, int B, int L, int N, int K, int M, double* y, void* stream);

/* Sigma = S diag(w) S^H + sigma^2 I  (covlinalg.py:43-57 cov_unknown; cov_known
 * :60-67 passes w = alpha*g).  pilots [B][L][N], w [B][N], noise [B] -> out [B][L][L]. */
size_t psca_cov_workspace_bytes(int B, int N, int L);
int psca_cov_unknown(const double* pilots, const double* w, const double* noise, int B, int N,
                     int L, double* out, void* workspace, size_t workspace_bytes, void* stream);

/* Hermitian PD inverse  (covlinalg.py:91-115 frobenius_inverse).
 * sigma [B][L][L] -> out [B][L][L] exactly Hermitian; status[b] = PSCA_CHOL_FAIL
 * with cond_est[b] when a pivot is not positive; logdet[b] = log|Sigma| (may be 0). */
size_t psca_inverse_workspace_bytes(int B, int L);
int psca_hpd_inverse(const double* sigma, int B, int L, double* out, int* status,
                     double* cond_est, double* logdet, void* workspace,
                     size_t workspace_bytes, void* stream);

/* q_n = s^H P s, r_n = s^H P Sigma_hat P s  (covlinalg.py:134-156 quad_forms).
 * pilots [B][L][N], sigma_inv [B][L][L], emp_cov [B][L][L] -> q, r [B][N]. */
size_t psca_quad_workspace_bytes(int B, int N, int L);
int psca_quad_forms(const double* pilots, const double* sigma_inv, const double* emp_cov, int B,
                    int N, int L, double* q, double* r, void* workspace,
                    size_t workspace_bytes, void* stream);

/* log|Sigma| + Re tr(Sigma^-1 Sigma_hat)  (covlinalg.py:159-172 eval_objective).
 * out [B]; status[b] = PSCA_CHOL_FAIL when Sigma is not PD. */
size_t psca_objective_workspace_bytes(int B, int L);
int psca_eval_objective(const double* sigma, const double* sigma_inv, const double* emp_cov,
                        int B, int L, double* out, int* status, void* workspace,
                        size_t workspace_bytes, void* stream);

/* Prior terms at x (the solver evaluates the same device code at every
 * iterate): gradient of the prior penalty and, optionally, its value and the
 * smoothed density.
 *   map-k, independent prior:  grad = prior_lin = -log(p/(1-p))/M,
 *       value = sum prior_lin x        (priors.py:145-158)
 *   map-k, pairwise MVB prior: grad = -(c1 + c2 x)/M,
 *       value = -(c1.x + x.(c2 x)/2)/M (priors.py:145-159)
 *   map-ur: grad = -(1/M) clip(p'/p, +-dzg) with the dead-zone push,
 *       value = -(1/M) sum log max(p, 1e-300), density = p^eps(x)
 *                                       (priors.py:313-399)
 * Replaces priors.log_prior_grad_known / log_prior_value_known /
 * log_prior_grad_unknown / log_prior_value_unknown / pdf_eff_smooth. */
typedef struct {
    int kind;               /* PSCA_MAP_K or PSCA_MAP_UR                        */
    int B, N, n_antennas;
    const double* x;        /* [B][N]                                          */
    const double* prior_lin;/* map-k independent: [N]                          */
    const double* prior_p;  /* map-ur: [N]                                     */
    psca_eff_prior eff;     /* map-ur                                          */
    const double* prior_c1; /* map-k pairwise: [N] and CSR c2, else all 0      */
    const int* prior_c2_indptr;
    const int* prior_c2_indices;
    const double* prior_c2_data;
    double* grad;           /* [B][N]                                          */
    double* value;          /* [B] or 0                                        */
    double* density;        /* map-ur: [B][N] or 0                             */
} psca_prior_args;

int psca_prior_terms(const psca_prior_args* a, void* stream);

/* One PSCA coordinate step from the quadratic forms at x (the column-kernel
 * epilogue as a standalone call): q-floor guard, gradient, surrogate
 * coefficient, clipped coordinate minimiser and the relaxed update
 *   grad = g (q - r) [known] or (q - r) [unknown], + prior_grad (map kinds)
 *   coef = (g q)^2 [known] or q^2 [unknown]
 *   cand = clip(x - grad / coef, 0, hi)
 *   x_new = (1 - rho) x + rho cand,  update_norm = ||x_new - x||_2
 *   status = PSCA_QFLOOR if min q < 0.5 L / ||Sigma||_F (sigma given), else 0
 * (estimators.py:176-200, 233-236, 267-284).  Every output may be 0. */
typedef struct {
    int kind, B, N, L;
    double rho, hi;         /* step and upper box bound (bounds_for)            */
    const double* x;        /* [B][N]                                          */
    const double* q;        /* [B][N]                                          */
    const double* r;        /* [B][N]                                          */
    const double* gains;    /* [B][N] (known-pathloss kinds)                   */
    const double* prior_grad; /* [B][N] (map kinds) or 0                       */
    const double* sigma;    /* [B][L][L] complex128 (q-floor guard) or 0       */
    double* grad;           /* [B][N]                                          */
    double* coef;           /* [B][N]                                          */
    double* cand;           /* [B][N]                                          */
    double* x_new;          /* [B][N]                                          */
    double* update_norm;    /* [B]                                             */
    int* status;            /* [B]                                             */
} psca_coord_args;

int psca_coord_step(const psca_coord_args* a, void* stream);

/* ---------------------------------------------------------------------------
 * Large pilot length (L <= 256; BASELINE config 4: N = 100,000, L = 256) as a
 * host-driven step loop for ONE instance, whose columns may be sharded over
 * ranks (multi-GPU column sharding):
 *     psca_large_begin                         x = 0, Sigma_0 = sigma^2 I, factor
 *     for k: psca_large_columns(k)             this rank's columns: quad forms,
 *                                              update, Sigma-increment partial
 *            [all-reduce the exchange block: dsig and red[0..1] (one SUM over
 *             dsig_len + 2 contiguous doubles), red[2] (MIN) -- ncclAllReduce
 *             over NVLink when sharded]
 *            psca_large_factor(k)              finalise iteration k (q-floor,
 *                                              update norm, tol), factor k+1
 *            the loop may run on after a stop: every kernel is gated on the
 *            device stop flag, so *flag (device int) needs checking only now
 *            and then (no host synchronisation per iteration)
 * red[0] = sum dx^2, red[1] = this shard's prior penalty (objective only),
 * red[2] = min q.  x after iteration k is x_b for even k, x_a for odd k (x_a
 * holds x_0 = 0).  Replaces the same psca_run loop (estimators.py:259-286)
 * for large L. */
typedef struct {
    int kind, N, L, n_antennas, max_iter, record_objective;
    double tol, noise;
    const double* pilots;   /* [L][N] complex128: this rank's columns         */
    const double* gains;    /* [N]                                             */
    const double* emp_cov;  /* [L][L] complex128                               */
    const double* steps;    /* [max_iter]                                      */
    const double* prior_lin;/* map-k [N]                                       */
    const double* prior_p;  /* map-ur [N]                                      */
    psca_eff_prior eff;
    double* x_a;            /* [N] x for even iterates                         */
    double* x_b;            /* [N] x for odd iterates                          */
    double* update_norm;    /* [max_iter]                                      */
    double* objective;      /* [max_iter] or 0                                 */
    double* iterates;       /* [max_iter+1][N] or 0                            */
    int* status;            /* [1]                                             */
    int* n_iter;            /* [1]                                             */
    double* cond_est;       /* [1] or 0                                        */
    /* map-k with a pairwise MVB prior (priors.py:56-159), as in
     * psca_solve_args: c1 [N] and the CSR interaction matrix c2; all null for
     * the independent prior (prior_lin).  The row sums c2 x need every
     * device's x, so this form takes the whole instance (no column shards). */
    const double* prior_c1;
    const int* prior_c2_indptr;
    const int* prior_c2_indices;
    const double* prior_c2_data;
} psca_large_args;

size_t psca_large_workspace_bytes(const psca_large_args* a);
/* Device addresses (inside the workspace) of the per-iteration exchange
 * block: dsig (dsig_len doubles) immediately followed by red (red == dsig +
 * dsig_len): dsig, red[0] and red[1] are summed over ranks, red[2] is
 * min-reduced. */
int psca_large_exchange(const psca_large_args* a, void* workspace, double** dsig,
                        size_t* dsig_len, double** red);
/* Device address of the stop flag (int, 0 = continue) inside the workspace;
 * written through flag_dev (an int** passed as void*). */
int psca_large_flag(const psca_large_args* a, void* workspace, int* flag_dev);
int psca_large_begin(const psca_large_args* a, void* workspace, size_t workspace_bytes,
                     void* stream);
int psca_large_columns(const psca_large_args* a, int k, void* workspace, size_t workspace_bytes,
                       void* stream);
int psca_large_factor(const psca_large_args* a, int k, void* workspace, size_t workspace_bytes,
                      void* stream);

/* One block-coordinate-descent sweep over all devices of every instance
 * (baselines.py:54-150 bcd_ml / bcd_map_k, the sequential comparison
 * detector): per device the exact coordinate minimiser on the current
 * Sigma^-1, then a Sherman-Morrison rank-1 update of Sigma^-1
 * (covlinalg.py:118-131).  x and sigma_inv carry the state between sweeps;
 * init = 1 starts from x = 0, Sigma^-1 = I / sigma^2.  status[b] = 1 when a
 * rank-1 denominator falls below 1e-14 (the reference's SingularUpdateError).
 * L <= 128 and the per-instance state must fit one SM's shared memory. */
typedef struct {
    int kind;               /* PSCA_ML_K, PSCA_MAP_K or PSCA_ML_UD               */
    int B, N, L, n_antennas;
    int init;
    const double* pilots;   /* [B][L][N] complex128                            */
    const double* gains;    /* [B][N] (known-pathloss kinds)                   */
    const double* emp_cov;  /* [B][L][L] complex128                            */
    const double* noise;    /* [B]                                             */
    const double* prior_lin;/* map-k, independent prior: [N] = -log(p/(1-p))/M */
    const double* prior_c1; /* map-k, pairwise prior (CSR c2), else 0          */
    const int* prior_c2_indptr;
    const int* prior_c2_indices;
    const double* prior_c2_data;
    double* x;              /* [B][N] in / out                                 */
    double* sigma_inv;      /* [B][L][L] complex128 in / out                   */
    int* status;            /* [B] in / out, 0 = running                       */
} psca_bcd_args;

int psca_bcd_sweep(const psca_bcd_args* a, void* stream);

/* Number of kernel launches the last psca_solve on this thread issued
 * (reported as bench.py's gpu_launches). */
int psca_last_launch_count(void);

/* Execution path of the last psca_solve on this thread: 0 = two kernels per
 * iteration (column chunks), 1 = one persistent launch for the whole solve,
 * 2 = two kernels per iteration for each half batch on two internal streams. */
int psca_last_path(void);

/* Device timing of every column / factor kernel launched by this thread
 * between begin and end (CUDA events on the launch stream; bench.py's
 * roofline).  end() synchronises on the recorded events. */
int psca_profile_begin(void);
int psca_profile_end(double* column_ms, int* column_launches, double* factor_ms,
                     int* factor_launches);

/* Experiment builds only (-DPSCA_PROBE=1): copy the clock64 phase probes of
 * the last instrumented launch (n <= 32 values) to host memory `out`. */
int psca_debug_probes(long long* out, int n);

/* on = 1: subsequent psca_solve calls on this thread issue every launch on
 * the caller's stream (no half-batch split over internal streams), so the
 * per-launch profile times are serialised kernel times; 0 restores the
 * default.  Results are identical either way. */
int psca_set_serial(int on);

/* Per-launch device times (ms) and kinds (0 column, 1 factor) of the
 * launches recorded since psca_profile_begin, in launch order (first `cap`
 * entries; synchronises on them).  Returns the number recorded, or a negative
 * PSCA_E* code.  Call before psca_profile_end, which clears the record. */
int psca_profile_launches(double* ms, int* kinds, int cap);

/* Description of the last CUDA error a call on this thread reported. */
const char* psca_last_error(void);

/* Library version string (host pointer). */
const char* psca_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PSCA_H */
