/*
 * pget.h -- C ABI of the B200-native PGET hot path (arXiv 2604.26745).
 *
 * The library (paper_2604_26745_b200/libpget.so) evaluates, on one B200
 * (sm_100a), the attenuated ray-tracing forward model of passive gamma emission
 * tomography, its Jacobian-vector and vector-Jacobian products with respect to
 * the emission lambda and the attenuation mu, and one regularised Gauss-Newton
 * (Levenberg-Marquardt) step solved by conjugate gradients.
 *
 * Model (Sec. 2.1, eq:fwd_model):
 *     F(lam,mu)(s,theta) = int_R lam(s theta_perp + t theta) exp(-B mu(s theta_perp + t theta, theta)) dt,
 *     B mu(x,theta)      = int_0^inf mu(x + tau theta) dtau,
 * discretised as BASELINE.json's ray-sampled quadrature:
 *   - image grid Omega = [-1,1]^2, N x N cell-centred pixels, h = 2/N, row = y, col = x;
 *   - angles theta_a = 2 pi a / n_angles; bank b looks along phi = theta_a + b pi with
 *     omega = (cos phi, sin phi) pointing at the detector, omega_perp = (-sin phi, cos phi);
 *   - detector offsets s_d = (2d - (n_det-1))/(n_det-1) (+ bank1_shift * pitch for bank 1),
 *     J sub-rays at s_d + ((2j+1-J)/(2J)) pitch with normalised Gaussian weights
 *     (sigma = subray_sigma * pitch)  [PAPER.md:33: two banks of 91 detectors];
 *   - samples t_i = -T + (i + 1/2) Delta, Delta = step_px * h, T = Delta ceil((sqrt2 + h)/Delta),
 *     bilinear interpolation of lam, mu at x_i = sigma omega_perp + t_i omega (zero outside);
 *   - A_i = Delta (mu_i / 2 + sum_{k>i} mu_k)  (k > i: nearer the detector),
 *     g_ray = Delta sum_i lam_i exp(-A_i),  y[a][b][d] = sum_j w_j g_ray(a,b,d,j).
 * Derivatives (eq:frechet): D_lam F[dlam] = F(dlam, mu),
 * D_mu F[dmu] = -F(lam B(dmu), mu), with the same quadrature for B; the VJP is the
 * exact transpose of that discrete JVP (the adjoint F'^* used at PAPER.md:231, 277).
 *
 * Layouts (all float32, C-contiguous, CUDA device memory owned by the caller):
 *   images    [batch][n_px][n_px]                     (lam, mu, dlam, dmu, g_lam, g_mu, s_lam, s_mu)
 *   sinograms [batch][n_angles][n_banks][n_det]       (y, dy, w, y_meas), detector fastest
 * Every device pointer must be 16-byte aligned (torch's allocator guarantees it).
 *
 * Ownership: the caller owns every buffer, including the workspace (size from
 * pget_workspace_bytes; any device memory, e.g. a torch uint8 tensor).  The
 * geometry handle owns only its small device tables, allocated in
 * pget_geometry_create and freed in pget_geometry_destroy.  No other call
 * allocates, frees or synchronises; everything is enqueued on `stream`.
 *
 * Errors: arguments are validated synchronously before anything is enqueued; on
 * failure nothing is enqueued and a non-OK status is returned, with a message in
 * pget_last_error_message() (thread-local).  Kernel launch failures return
 * PGET_ERR_CUDA.  No C++ exception crosses this interface; nothing aborts.
 *
 * Tracing: every compute entry point is an NVTX range named after it (Nsight Systems, ncu --nvtx).
 *
 * Threading: a handle is immutable after creation; concurrent calls on
 * different streams are safe when their workspaces and outputs differ.
 */
#ifndef PGET_H
#define PGET_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

struct CUstream_st;
typedef struct CUstream_st* pget_stream_t;   /* == cudaStream_t; NULL = legacy default stream */

typedef struct pget_geometry_s* pget_geometry; /* opaque */

typedef enum {
    PGET_OK = 0,
    PGET_ERR_INVALID_ARGUMENT = 1,
    PGET_ERR_SHAPE = 2,
    PGET_ERR_ALIGNMENT = 3,
    PGET_ERR_WORKSPACE = 4,
    PGET_ERR_OUT_OF_MEMORY = 5,
    PGET_ERR_CUDA = 6,
    PGET_ERR_NOT_FINITE = 7
} pget_status;

/* Geometry descriptor (PAPER.md:33 detector banks; BASELINE.json configs). */
typedef struct {
    int32_t n_px;         /* N >= 2: image N x N on [-1,1]^2                              */
    int32_t n_angles;     /* >= 1: theta_a = 2 pi a / n_angles                             */
    int32_t n_banks;      /* 1 or 2 (opposing bank looks along theta + pi)                 */
    int32_t n_det;        /* >= 2 detectors per bank spanning [-1, 1]                      */
    int32_t n_subrays;    /* J in [1, 64] sub-rays per detector                            */
    double subray_sigma;  /* > 0: Gaussian collimator sigma in detector pitches (0.4)      */
    double step_px;       /* > 0: sample step Delta in pixels (0.5)                        */
    double bank1_shift;   /* bank-1 offset shift in pitches (0 for the configs)            */
    int32_t batch;        /* >= 1 independent image pairs per call                         */
    /* Model variant (eq:d_fwd_model; reading R-N3): the
     * collimator response r_{m,n} and the vertical opening-angle correction c_{m,n} >= 1 as functions of
     * the emission point's distance to the detector, d_i = det_radius - t_i:
     *     y = sum_j sum_i W_j(d_i) Delta lam_i exp(-c_i A_i),   c_i = 1 + c_slope d_i,
     *     W_j(d) = exp(-delta_j^2/(2 sigma(d)^2)) / sum_k exp(-delta_k^2/(2 sigma(d)^2)),
     *     sigma(d) = subray_sigma * pitch * (1 + r_slope d).
     * det_radius <= 0: off (the base model above).  On: det_radius >= T, slopes >= 0 and finite.  The
     * variant runs unpaired, unsegmented and without the GN coefficient cache (its attenuation does not
     * factor along a ray), so it is several times slower than the base model. */
    double det_radius;    /* distance from the rotation centre to the detector face (domain units) */
    double c_slope;       /* c_i = 1 + c_slope d_i                                          */
    double r_slope;       /* sigma(d) = sigma_0 (1 + r_slope d)                              */
    /* Pixel basis (eq:d_fwd_model's d_{m,n,k}, "the distances a ray from m to n
     * covers within pixel k"; reading R-pb): 1 = lam, mu constant on each pixel, a ray
     * crosses pixels k_1..k_M (increasing t) with exact intersection lengths l_q and
     *     A_q = l_q mu_q / 2 + sum_{p>q} l_p mu_p,   g_ray = sum_q r_q lam_q exp(-c_q A_q),
     * r_q = l_q (times W_j(d_q), c_q = 1 + c_slope d_q with the variant above, d_q at the chord
     * midpoint), y = sum_j w_j g_ray (w_j inside r_q with the variant); step_px is unused.
     * 0 = the sampled model above.  Runs unpaired, unsegmented, every angle-bank traced, with the
     * recomputed GN product (sid.cu). */
    int32_t pixel_basis;
    int32_t pad_;
} pget_geometry_desc;

typedef struct {
    int64_t n_rays;             /* batch * n_angles * n_banks * n_det * n_subrays          */
    int64_t n_samples_nominal;  /* batch * sum over rays of (i_hi - i_lo + 1): the unit of
                                   the ray-samples/s metric                                 */
    int64_t image_elems;        /* batch * n_px * n_px                                      */
    int64_t sino_elems;         /* batch * n_angles * n_banks * n_det                       */
    int32_t n_t;                /* unclipped samples per ray = 2 T / Delta                  */
    int32_t n_px, n_angles, n_banks, n_det, n_subrays, batch;
    double h, delta, T;
    int64_t n_samples_traced;   /* line samples the forward / VJP / GN projector evaluates per pass:
                                   n_samples_nominal, or about a quarter of it when angle_banks_merged:
                                   with an even n_angles, 2 banks and bank1_shift = 0 the rays of
                                   (a + n_angles/2, 1 - b) are those of (a, b), and bank 1 of angle a
                                   traces the lines of bank 0 in the opposite direction, so one
                                   traversal serves all four               */
    int32_t angle_banks_merged; /* 1 when that merging is active                                  */
    int32_t pad_;
    int64_t n_samples_traced_jvp; /* the same for the JVP projector (both directions traced:
                                     about half of nominal when merged)                          */
} pget_geometry_info_t;

/* Table ids for pget_geometry_export (bit-exact comparison with the oracle, pin P1). */
enum {
    PGET_TABLE_ANGLES = 0,  /* double [n_angles]                         theta_a              */
    PGET_TABLE_DIRS = 1,    /* double [n_angles][n_banks][2]             (cos phi, sin phi)   */
    PGET_TABLE_OFFSETS = 2, /* double [n_banks][n_det][n_subrays]        sigma_{b,d,j}        */
    PGET_TABLE_WEIGHTS = 3, /* double [n_subrays]                        w_j                  */
    PGET_TABLE_TLAT = 4,    /* double [3]                                (h, Delta, T)        */
    PGET_TABLE_CLIP = 5,    /* int32  [n_angles][n_banks][n_det][n_subrays][2]  (i_lo, i_hi); empty ray = (0,-1) */
    PGET_TABLE_VAR_C = 6,   /* double [n_t]                              c_i (model variant; 0 bytes when off) */
    PGET_TABLE_VAR_W = 7    /* double [n_subrays][n_t]                   W_j(d_i) (model variant)            */
};

/* Operation ids for pget_workspace_bytes. */
enum { PGET_OP_FORWARD = 0, PGET_OP_JVP = 1, PGET_OP_VJP = 2, PGET_OP_GN_CG_STEP = 3, PGET_OP_GN_APPLY = 4,
       PGET_OP_SAFEGUARD = 5, PGET_OP_LM_SOLVE = 6 };

/* Flags for pget_gn_cg_step. */
#define PGET_GN_EVAL_TRIAL 1u   /* also evaluate f(u+s), rho, the accept decision and beta_next */
#define PGET_MAX_CG 256

/* Device-resident statistics of one LM iteration, per batch member (array of `batch`).
 * (SURVEY.md §8(c.2) O7; PAPER.md:160-164 eq:m-function, :248 eq:rho_agreement.) */
typedef struct {
    double f;             /* f(u) = 1/2||F(u)-y||^2 + alpha/2(||L lam||^2 + ||L mu||^2)      */
    double misfit;        /* 1/2 ||F(u) - y||^2                                               */
    double reg;           /* R(u)                                                             */
    double grad_norm;     /* ||b||, b = -grad f(u)                                            */
    double pred;          /* m(0) - m(s) = <b,s> - 1/2(||Js||^2 + alpha ||Ls||^2)             */
    double f_trial;       /* f(u+s)                      (PGET_GN_EVAL_TRIAL)                 */
    double rho;           /* (f(u) - f(u+s)) / pred      (PGET_GN_EVAL_TRIAL)                 */
    double beta_next;     /* x10 on reject (>= beta_min), x0.2 if rho > 0.75 (PGET_GN_EVAL_TRIAL) */
    double beta_min;      /* 1e-3 <b,Hb>/<b,b>                                               */
    double js2;           /* ||Js||^2                                                         */
    double als2;          /* alpha ||Ls||^2                                                   */
    double bs;            /* <b, s>                                                           */
    int32_t accepted;     /* pred > 0 and rho > eta = 0.1 (PGET_GN_EVAL_TRIAL; reading R-accept)  */
    int32_t n_cg_done;    /* CG steps performed                                               */
    int32_t breakdown;    /* 0 none, 1 zeta == 0, 2 <p,Hp> <= 0                              */
    int32_t pad_;
    double cg_res[PGET_MAX_CG + 1]; /* ||z_k||, k = 0..n_cg                                   */
} pget_gn_stats;

/* Parameters of pget_lm_solve (host struct).  (PAPER.md:144-182, 288.) */
#define PGET_LM_BOX 1u   /* project every iterate onto [lam_lo, lam_hi] x [mu_lo, mu_hi] */
#define PGET_LM_SGP 2u   /* with PGET_LM_BOX: solve each step's box-constrained subproblem by scaled gradient
                          * projection (identity scaling, Barzilai-Borwein lengths, exact line
                          * search, n_cg iterations; stats cg_res = ||d_k||, the projected-gradient step)
                          * instead of CG followed by the projection */
typedef struct {
    int32_t n_iter;       /* LM iterations                                                    */
    int32_t n_cg;         /* CG steps per iteration, 0 <= n_cg <= PGET_MAX_CG                  */
    float alpha0;         /* penalty weight of iteration 0                                     */
    float alpha_decay;    /* alpha_k = alpha0 / alpha_decay^min(k, k_freeze) (paper: 5, :288)   */
    int32_t k_freeze;     /* iteration from which alpha stays fixed                            */
    float beta0;          /* initial LM parameter of every member                              */
    float lam_lo, lam_hi, mu_lo, mu_hi;   /* the box (PGET_LM_BOX)                              */
    uint32_t flags;       /* PGET_LM_BOX, PGET_LM_SGP                                          */
    float lam_per_mu;     /* > 0 (with PGET_LM_BOX): also lam <= lam_per_mu * mu in every projection ("low
                           * attenuation but highly emitting materials are not allowed", PAPER.md:148;
                           * reading R-lin); 0 = off                                               */
} pget_lm_params;

/* Device-resident result of the Prop. 1 safeguard check, per batch member (array of `batch`).
 * (Prop. 1 eq:rho_agreement, eq:uk+1_condition;
 * Algorithm 2; m_k of eq:m-function.)
 * m_k(s) = f(u) + <r, J s> + alpha (<L lam, L s_lam> + <L mu, L s_mu>) + 1/2 ||J s||^2
 *          + alpha/2 ||L s||^2   (the stacked F~ = (F, sqrt(alpha) L) of reading Q10). */
typedef struct {
    double f;             /* f(u_k) = m_k(0)                                                  */
    double f_cand;        /* f(u~)                                                            */
    double m_cand;        /* m_k(s~), s~ = u~ - u_k                                           */
    double m_lm;          /* m_k(s_k)                                                         */
    double pred_cand;     /* m_k(0) - m_k(s~)                                                 */
    double pred_lm;       /* m_k(0) - m_k(s_k)                                                */
    double rho_cand;      /* (f(u_k) - f(u~)) / pred_cand; 0 when pred_cand == 0               */
    double kappa;         /* the threshold used                                               */
    int32_t accepted;     /* m_cand <= m_lm and pred_cand > 0 and rho_cand > kappa             */
    int32_t pad_;
} pget_safeguard_stats;

const char* pget_status_string(pget_status s);
const char* pget_last_error_message(void);

/* Build the geometry (host fp64 tables, O1 of SURVEY.md §8(c.2)) and upload its
 * device tables on `device`.  *out receives the handle.  Synchronous.
 * device < 0 creates a host-only handle (info and table export only; every compute
 * call on it returns PGET_ERR_INVALID_ARGUMENT) -- usable without a GPU. */
pget_status pget_geometry_create(const pget_geometry_desc* desc, int device, pget_geometry* out);
pget_status pget_geometry_destroy(pget_geometry g);
pget_status pget_geometry_info(pget_geometry g, pget_geometry_info_t* out);
size_t pget_table_bytes(pget_geometry g, int table_id);                    /* 0 for a bad id */
pget_status pget_geometry_export(pget_geometry g, int table_id, void* host_dst, size_t bytes);

/* Geometry priors P1, P2 of eq:lma_objective (reading R-prior
 * in DESIGN.md): penalties of the emission and attenuation outside the expected rod locations, as
 * diagonal masks,
 *     f(u) += alpha1/2 ||P1 lam||^2 + alpha2/2 ||P2 mu||^2,   P1 = diag(mask_lam), P2 = diag(mask_mu),
 * so the gradient gains (alpha1 mask_lam^2 lam, alpha2 mask_mu^2 mu), H gains that diagonal and m_k
 * the stacked rows sqrt(alpha1) P1 lam, sqrt(alpha2) P2 mu.  pget_lm_solve continues them with alpha
 * (alpha^(k) = (alpha1, alpha2) / 5^k).
 * mask_lam / mask_mu: device fp32 images [batch][N][N] (row = y) or NULL (that term off);
 * alpha1, alpha2: finite and >= 0. */
typedef struct {
    const float* mask_lam;
    const float* mask_mu;
    float alpha1, alpha2;
} pget_prior;

/* Attach the priors to the handle: every later pget_gn_apply, pget_gn_cg_step, pget_lm_solve and
 * pget_safeguard on g includes them until pget_set_prior(g, NULL) clears them.  The handle keeps
 * the two device pointers (the caller keeps the masks alive and unchanged while set); it does not
 * copy them.  Not to be called while calls on g are in flight on another thread.
 * Errors: PGET_ERR_INVALID_ARGUMENT for a NULL/host-only handle or a negative / non-finite weight. */
pget_status pget_set_prior(pget_geometry g, const pget_prior* prior);

/* Workspace bytes needed by `op` (PGET_OP_*); 0 for a bad op. */
size_t pget_workspace_bytes(pget_geometry g, int op);

/* y = F(lam, mu)  (eq:fwd_model). */
pget_status pget_forward(pget_geometry g, const float* lam, const float* mu, float* y,
                         void* ws, size_t ws_bytes, pget_stream_t stream);

/* dy = D_lam F[dlam] + D_mu F[dmu]  (eq:frechet); y = F(lam, mu) too when y != NULL. */
pget_status pget_jvp(pget_geometry g, const float* lam, const float* mu, const float* dlam,
                     const float* dmu, float* y_or_null, float* dy, void* ws, size_t ws_bytes,
                     pget_stream_t stream);

/* (g_lam, g_mu) = F'(lam, mu)^T w  (adjoint of eq:frechet). */
pget_status pget_vjp(pget_geometry g, const float* lam, const float* mu, const float* w,
                     float* g_lam, float* g_mu, void* ws, size_t ws_bytes, pget_stream_t stream);

/* (q_lam, q_mu) = H p = J^T J p + alpha L^T L p + beta p at u = (lam, mu): the GN normal
 * operator of eq:LMA-step with the Laplacian penalty (reading Q10); plus the
 * diagonal of the priors when pget_set_prior attached them. */
pget_status pget_gn_apply(pget_geometry g, const float* lam, const float* mu, const float* p_lam,
                          const float* p_mu, float alpha, float beta, float* q_lam, float* q_mu,
                          void* ws, size_t ws_bytes, pget_stream_t stream);

/* One LM iteration at u = (lam, mu) for measurements y_meas:
 * r = F(u) - y; b = -(J^T r + alpha L^T L u); n_cg CG steps from s = 0 on
 * (J^T J + alpha L^T L + beta I) s = b; pred; with PGET_GN_EVAL_TRIAL also f(u+s),
 * rho, accept (pred > 0 and rho > 0.1, reading R-accept) and beta_next.  Writes s to (s_lam, s_mu) and `batch`
 * pget_gn_stats structs to stats_dev (device memory).  0 <= n_cg <= PGET_MAX_CG. */
pget_status pget_gn_cg_step(pget_geometry g, const float* lam, const float* mu, const float* y_meas,
                            float alpha, float beta, int32_t n_cg, uint32_t flags, float* s_lam,
                            float* s_mu, pget_gn_stats* stats_dev, void* ws, size_t ws_bytes,
                            pget_stream_t stream);

/* Full LM solve (the paper's deterministic LMA iterated; the alpha continuation
 * alpha_k = alpha0 / 5^k frozen later), per batch member, on the device: for
 * k = 0..n_iter-1 one LM iteration at (u_k, alpha_k, beta_k) with PGET_GN_EVAL_TRIAL.  The feasible
 * set (PGET_LM_BOX) is the box [lam_lo, lam_hi] x [mu_lo, mu_hi], intersected with lam <= c mu when
 * lam_per_mu = c > 0 (reading R-lin); P denotes the per-pixel Euclidean projection onto
 * it.  The inner solver is either
 *   - CG (default; reading R-N1): n_cg CG steps on the unconstrained normal equations, then the step
 *     is replaced by the step actually taken, s' = P(u_k + s) - u_k; or
 *   - scaled gradient projection (PGET_LM_SGP, the paper's solver; reading R-SGP):
 *     n_cg projected-gradient iterations on the box-constrained quadratic model, whose iterates stay
 *     feasible, so s' = s.
 * pred, rho and the trial point refer to s' (the trial point u_k + s' is feasible).  Then
 * u_{k+1} = u_k + s' if pred > 0 and rho > 0.1 (accepted, reading R-accept) else u_k, and
 * beta_{k+1} = beta_next (x10 on reject, at least beta_min; x0.2 if rho > 0.75).  With PGET_LM_BOX the
 * initial guess is projected first, so every iterate is feasible.
 * lam, mu: device images, updated in place.  stats_dev: n_iter * batch pget_gn_stats records, iteration-major,
 * receiving every iteration's statistics.  Workspace: pget_workspace_bytes(g, PGET_OP_LM_SOLVE).
 * No host synchronisation; errors as for pget_gn_cg_step. */
pget_status pget_lm_solve(pget_geometry g, float* lam, float* mu, const float* y_meas,
                          const pget_lm_params* params, pget_gn_stats* stats_dev, void* ws,
                          size_t ws_bytes, pget_stream_t stream);

/* Safeguarded acceptance of an externally supplied candidate u~ = (cand_lam, cand_mu) against the
 * LM step s_k = (s_lam, s_mu) at u_k = (lam, mu) (Proposition 1; the check of
 * Algorithm 2):  u_next = u~ if m_k(s~) <= m_k(s_k) and rho_k(s~) > kappa
 * (and m_k(0) - m_k(s~) > 0, reading R-safeguard), else u_k + s_k (fp32 sum), per batch member.
 * Costs two JVP launches (J s~ together with F(u_k), then J s_k) and one forward launch (F(u~)).
 * alpha must be the penalty weight the step s_k was computed with; kappa > 0 (the paper's
 * kappa = eta = 0.1, reading Q11).  All arrays are device memory of the image / sinogram shapes
 * of the other calls; u_next_lam / u_next_mu may alias cand_* but not lam, mu, s_*.  `stats_dev`
 * receives `batch` pget_safeguard_stats.  Errors as for pget_gn_cg_step. */
pget_status pget_safeguard(pget_geometry g, const float* lam, const float* mu, const float* y_meas,
                           const float* s_lam, const float* s_mu, const float* cand_lam,
                           const float* cand_mu, float alpha, float kappa, float* u_next_lam,
                           float* u_next_mu, pget_safeguard_stats* stats_dev, void* ws,
                           size_t ws_bytes, pget_stream_t stream);

/* Diagnostic (tests): where the CG vectors of an LM iteration live inside its workspace.  For op
 * PGET_OP_GN_CG_STEP, region PGET_WS_P_LAM / P_MU is the CG direction p and PGET_WS_Q_LAM / Q_MU the
 * product q = H p of the last CG step, each [batch][N][N] fp32 at ws + *offset.  After a call with
 * n_cg = k >= 1 they hold p_k and q_{k-1} = H p_{k-1} (with n_cg = 0: p_0 = b), so a caller can pin
 * the operator the CG loop applies, step by step.  PGET_OK, or
 * PGET_ERR_INVALID_ARGUMENT for a bad op / region.  Host-side, no device access. */
enum { PGET_WS_P_LAM = 0, PGET_WS_P_MU = 1, PGET_WS_Q_LAM = 2, PGET_WS_Q_MU = 3 };
pget_status pget_workspace_region(pget_geometry g, int op, int region, size_t* offset, size_t* bytes);

/* Diagnostic: checks on the host that the handle's static schedules are consistent (every
 * (member, angle-bank, detector) of the forward/JVP schedules covered once; the adjoint's row
 * segments partition every ray's samples; every unit scheduled once per phase; partial slots hold
 * <= 16 units of one CTA and their row ranges cover the units' rows; every slot reduced once; the
 * coefficient-cache blocks cover every lane; comb lanes >= comb stride apart).  Works on host-only
 * handles (device < 0).  PGET_OK or PGET_ERR_INVALID_ARGUMENT with the violated rule in
 * pget_last_error_message(). */
pget_status pget_schedule_check(pget_geometry g);

/* Failure detection: scans n floats of device array x for NaN / infinity on `stream`,
 * then synchronises it.  PGET_OK if all are finite, PGET_ERR_NOT_FINITE otherwise (for example the
 * output of a call fed non-finite inputs).  flag_dev: one device int32 of scratch (caller-owned).
 * A diagnostic: unlike the compute calls it waits for the stream. */
pget_status pget_check_finite(const float* x, size_t n, int32_t* flag_dev, pget_stream_t stream);

/* Tracing.  Between pget_profile_begin and pget_profile_end every kernel the library
 * launches (on any stream, from any thread) is counted, and each projector launch is
 * bracketed by two CUDA events recorded on the stream it is launched on (up to
 * max_launches projector launches; later ones are counted but not timed).
 * pget_profile_end waits for the recorded events and returns, per projector mode
 * (0 forward, 1 JVP, 2 VJP, 3 GN normal product), the summed device time in ms and
 * the launch count, plus the total number of library kernel launches.  Host-side. */
pget_status pget_profile_begin(int32_t max_launches);
pget_status pget_profile_end(double* ms_per_mode /* [4] */, int64_t* launches_per_mode /* [4] */,
                             int64_t* total_launches);

#ifdef __cplusplus
}
#endif
#endif /* PGET_H */
