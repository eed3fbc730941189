/*
 * pget_oracle.c -- plain, slow, fp64 CPU oracle of the PGET hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no
 * code, header, table or constant generator with the CUDA product path
 * (paper_2604_26745_b200/csrc); it is written directly from the definitions
 * below, with direct loops over rays and samples and no blocking or fusion.
 *
 * Definitions (which restate the paper):
 *   F(lam,mu)(s,th) = int lam(s th_perp + t th) exp(-B mu(s th_perp + t th, th)) dt,
 *   B mu(x,th)      = int_0^inf mu(x + tau th) dtau
 *       -- PAPER.md:48-54, Sec. 2.1, eq:fwd_model (ray-sampled quadrature, readings Q7-Q9)
 *   D_lam F[dlam] = F(dlam, mu);  D_mu F[dmu] = -F(lam B(dmu), mu)
 *       -- PAPER.md:55-59, eq:frechet
 *   adjoint F'^*[w]  -- used at PAPER.md:231, 277 (Thm 10.3, proof of Prop. 1)
 *   f(u) = 1/2 ||F(u)-y||^2 + alpha/2 (||L lam||^2 + ||L mu||^2)
 *       -- PAPER.md:144-148 eq:lma_objective with reading Q10
 *   LM step (J^T J + alpha L^T L + beta I) s = -grad f, m_k, rho_k
 *       -- PAPER.md:160-180 eq:m-function, eq:LMA-step; PAPER.md:248 eq:rho_agreement
 *       -- inner solver: plain CG (reading Q12) instead of the paper's SGP.
 *   LM solve: alpha continuation, beta schedule, box projection -- PAPER.md:144-182, 288 (O9, N1)
 *   SGP inner solver (O11, N1): the box-constrained LM subproblem by gradient projection with
 *       Barzilai-Borwein steps and an exact line search -- PAPER.md:177 (bonettini2008scaled),
 *       identity scaling (reading R-SGP)
 *   geometry priors (O10, N1): f += alpha1/2 ||P1 lam||^2 + alpha2/2 ||P2 mu||^2, P1, P2 diagonal
 *       masks -- PAPER.md:146-148 eq:lma_objective (reading R-prior), continued with alpha
 *       (alpha^(k) = (alpha1, alpha2) / 5^k); set by orc_set_prior, used by every
 *       function below that evaluates f, its gradient, H or m_k (not thread-safe: test use only)
 *   safeguard u_{k+1} = u~ iff m_k(s~) <= m_k(s_k) and rho_k(s~) > kappa
 *       -- PAPER.md:241-258 Prop. 1 eq:uk+1_condition; Algorithm 2 PAPER.md:290-313 (O8, N2)
 *   model variant (O13, N3): the collimator response r_{m,n} and the vertical opening-angle correction
 *       c_{m,n} >= 1 of eq:d_fwd_model, as functions of the emission point's
 *       distance to the detector d = det_radius - t (reading R-N3):
 *         y = sum_j sum_i W_j(d_i) Delta lam_i exp(-c_i A_i),  c_i = 1 + c_slope d_i,
 *         W_j(d) = exp(-delta_j^2 / (2 sigma(d)^2)) / sum_k exp(-delta_k^2 / (2 sigma(d)^2)),
 *         sigma(d) = subray_sigma * pitch * (1 + r_slope d);   on iff det_radius > 0
 *   pixel basis (O14, N3): the exact intersection lengths d_{m,n,k} of eq:d_fwd_model (
 *       reading R-pb): lam, mu constant on each pixel; a ray crosses pixels k_1..k_M (increasing t, the
 *       detector at +t) with lengths l_q; the ray from pixel k_q starts at the midpoint of its chord:
 *         A_q = 1/2 l_q mu_q + sum_{p>q} l_p mu_p,   g_ray = sum_q r_q lam_q exp(-c_q A_q),
 *         r_q = l_q (W_j(d_q) with the O13 variant), d_q = det_radius - t_q at the chord midpoint;
 *       y = sum_j w_j g_ray (base weights) as for the sampled model.  on iff pixel_basis != 0
 *
 * Parity pins: tests/test_oracle.py (P1-P12 of SURVEY.md §8(c.4)); DESIGN.md "Oracle".
 * Compile: gcc -O2 -fopenmp -ffp-contract=off -fPIC -shared (no fast-math).
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
    int n_px, n_angles, n_banks, n_det, n_subrays;
    double subray_sigma, step_px, bank1_shift;
    int batch;
    double det_radius, c_slope, r_slope;   /* O13 model variant (N3); det_radius <= 0: off */
    int pixel_basis;                       /* O14 pixel basis (N3): exact intersection lengths  */
} orc_desc;

/* ------------------------------------------------------------------ O1 geometry */
typedef struct {
    double h, delta, T;
    int n_t;
} orc_lattice;

static orc_lattice o1_lattice(const orc_desc* g)
{
    orc_lattice L;
    L.h = 2.0 / g->n_px;                               /* h = 2/N            */
    L.delta = g->step_px * L.h;                        /* Delta = step_px*h  */
    double m = ceil((sqrt(2.0) + L.h) / L.delta);      /* T = Delta*ceil((sqrt2+h)/Delta) */
    L.T = L.delta * m;
    L.n_t = 2 * (int)m;                                /* n_t = 2T/Delta     */
    return L;
}

static double o1_theta(const orc_desc* g, int a) { return 2.0 * M_PI * a / g->n_angles; }

/* direction of bank b at angle a: phi = theta_a + b*pi; omega = (cos phi, sin phi) */
static void o1_dir(const orc_desc* g, int a, int b, double* c, double* s)
{
    double phi = o1_theta(g, a) + b * M_PI;
    *c = cos(phi);
    *s = sin(phi);
}

/* offset sigma_{b,d,j} = s_d (+ bank1_shift*p for bank 1) + delta_j */
static double o1_offset(const orc_desc* g, int b, int d, int j)
{
    int nd = g->n_det, J = g->n_subrays;
    double p = 2.0 / (nd - 1);
    double s = (double)(2 * d - (nd - 1)) / (double)(nd - 1);
    if (b == 1) s = s + g->bank1_shift * p;
    double dj = (double)(2 * j + 1 - J) / (double)(2 * J) * p;
    return s + dj;
}

static void o1_weights(const orc_desc* g, double* w)
{
    int J = g->n_subrays;
    double p = 2.0 / (g->n_det - 1);
    double sp = g->subray_sigma * p;
    double sum = 0.0;
    for (int j = 0; j < J; ++j) {
        double dj = (double)(2 * j + 1 - J) / (double)(2 * J) * p;
        w[j] = exp(-(dj * dj) / (2.0 * sp * sp));
        sum += w[j];
    }
    for (int j = 0; j < J; ++j) w[j] = w[j] / sum;
}

/* slab clip of x(t) = sigma*omega_perp + t*omega against |x|,|y| <= 1 + h/2 */
static void o1_clip(const orc_desc* g, const orc_lattice* L, double c, double s, double sigma,
                    int* ilo, int* ihi)
{
    double bb = 1.0 + L->h / 2.0;
    double om[2] = {c, s};
    double op[2] = {-s, c};
    double tin = -INFINITY, tout = INFINITY;
    for (int k = 0; k < 2; ++k) {
        double base = sigma * op[k];
        if (om[k] == 0.0) {
            if (fabs(base) > bb) { tin = INFINITY; tout = -INFINITY; }
        } else {
            double t1 = (-bb - base) / om[k];
            double t2 = (bb - base) / om[k];
            double lo = t1 < t2 ? t1 : t2, hi = t1 < t2 ? t2 : t1;
            if (lo > tin) tin = lo;
            if (hi < tout) tout = hi;
        }
    }
    if (!(tin <= tout)) { *ilo = 0; *ihi = -1; return; }
    double lo = ceil((tin + L->T) / L->delta - 0.5);
    double hi = floor((tout + L->T) / L->delta - 0.5);
    if (lo < 0.0) lo = 0.0;
    if (hi > (double)(L->n_t - 1)) hi = (double)(L->n_t - 1);
    if (lo > hi) { *ilo = 0; *ihi = -1; return; }
    *ilo = (int)lo;
    *ihi = (int)hi;
}

int orc_n_t(const orc_desc* g) { return o1_lattice(g).n_t; }

/* Export every O1 table (for the bit-exact comparison with the library, pin P1). */
int orc_tables(const orc_desc* g, double* angles, double* dirs, double* offsets, double* weights,
               double* tlat, int* n_t, int* clip)
{
    orc_lattice L = o1_lattice(g);
    int nA = g->n_angles, nB = g->n_banks, nd = g->n_det, J = g->n_subrays;
    for (int a = 0; a < nA; ++a) angles[a] = o1_theta(g, a);
    for (int a = 0; a < nA; ++a)
        for (int b = 0; b < nB; ++b) o1_dir(g, a, b, &dirs[(a * nB + b) * 2], &dirs[(a * nB + b) * 2 + 1]);
    for (int b = 0; b < nB; ++b)
        for (int d = 0; d < nd; ++d)
            for (int j = 0; j < J; ++j) offsets[(b * nd + d) * J + j] = o1_offset(g, b, d, j);
    o1_weights(g, weights);
    tlat[0] = L.h; tlat[1] = L.delta; tlat[2] = L.T;
    *n_t = L.n_t;
    for (int a = 0; a < nA; ++a)
        for (int b = 0; b < nB; ++b) {
            double c, s;
            o1_dir(g, a, b, &c, &s);
            for (int d = 0; d < nd; ++d)
                for (int j = 0; j < J; ++j) {
                    size_t r = (((size_t)a * nB + b) * nd + d) * J + j;
                    o1_clip(g, &L, c, s, o1_offset(g, b, d, j), &clip[2 * r], &clip[2 * r + 1]);
                }
        }
    return 0;
}

/* ------------------------------------------------------------------ O2 sampling */
/* pixel-index coordinates of sample i: u = (x+1)/h - 1/2, v = (y+1)/h - 1/2 */
static void o2_pos(const orc_lattice* L, double c, double s, double sigma, int i, double* u, double* v)
{
    double t = -L->T + (i + 0.5) * L->delta;
    double x = sigma * (-s) + t * c;
    double y = sigma * c + t * s;
    *u = (x + 1.0) / L->h - 0.5;
    *v = (y + 1.0) / L->h - 0.5;
}

static double o2_pix(const double* img, int N, int j, int i)
{
    if (i < 0 || i >= N || j < 0 || j >= N) return 0.0;
    return img[(size_t)j * N + i];
}

/* bilinear interpolation with zero outside the grid */
static double o2_sample(const double* img, int N, double u, double v)
{
    double fi = floor(u), fj = floor(v);
    int i0 = (int)fi, j0 = (int)fj;
    double fu = u - fi, fv = v - fj;
    return (1.0 - fu) * (1.0 - fv) * o2_pix(img, N, j0, i0) + fu * (1.0 - fv) * o2_pix(img, N, j0, i0 + 1)
         + (1.0 - fu) * fv * o2_pix(img, N, j0 + 1, i0) + fu * fv * o2_pix(img, N, j0 + 1, i0 + 1);
}

/* transpose of o2_sample: scatter val to the 4 neighbours, dropping out-of-grid ones */
static void o2_scatter(double* img, int N, double u, double v, double val)
{
    double fi = floor(u), fj = floor(v);
    int i0 = (int)fi, j0 = (int)fj;
    double fu = u - fi, fv = v - fj;
    double wts[4] = {(1.0 - fu) * (1.0 - fv), fu * (1.0 - fv), (1.0 - fu) * fv, fu * fv};
    int di[4] = {0, 1, 0, 1}, dj[4] = {0, 0, 1, 1};
    for (int k = 0; k < 4; ++k) {
        int ii = i0 + di[k], jj = j0 + dj[k];
        if (ii < 0 || ii >= N || jj < 0 || jj >= N) continue;
        img[(size_t)jj * N + ii] += wts[k] * val;
    }
}

/* ------------------------------------------------------------------ per-ray work */
typedef struct {
    orc_lattice L;
    double w[64];
    int var;          /* O13 variant on */
    double* C;        /* [n_t]    c_i                   */
    double* W;        /* [J][n_t] W_j(d_i)              */
} orc_ctx;

/* O13 tables (variant): distance of lattice sample i to the detector d_i = det_radius - t_i,
 * c_i = 1 + c_slope d_i, W_j(d_i) the normalised Gaussian sub-ray response of width
 * sigma(d_i) = subray_sigma * pitch * (1 + r_slope d_i) */
static void o13_tables(const orc_desc* g, const orc_lattice* L, double* C, double* W)
{
    int J = g->n_subrays;
    double p = 2.0 / (g->n_det - 1);
    for (int i = 0; i < L->n_t; ++i) {
        double t = -L->T + (i + 0.5) * L->delta;
        double d = g->det_radius - t;
        C[i] = 1.0 + g->c_slope * d;
        double sp = g->subray_sigma * p * (1.0 + g->r_slope * d);
        double sum = 0.0;
        for (int j = 0; j < J; ++j) {
            double dj = (double)(2 * j + 1 - J) / (double)(2 * J) * p;
            W[(size_t)j * L->n_t + i] = exp(-(dj * dj) / (2.0 * sp * sp));
            sum += W[(size_t)j * L->n_t + i];
        }
        for (int j = 0; j < J; ++j) W[(size_t)j * L->n_t + i] = W[(size_t)j * L->n_t + i] / sum;
    }
}

static void ctx_free(orc_ctx* cx)
{
    free(cx->C);
    free(cx->W);
    cx->C = cx->W = NULL;
}

static int ctx_init(const orc_desc* g, orc_ctx* cx)
{
    cx->C = cx->W = NULL;
    cx->var = 0;
    if (g->n_subrays > 64 || g->n_subrays < 1 || g->n_det < 2 || g->n_px < 2 || g->n_angles < 1 ||
        g->n_banks < 1 || g->n_banks > 2 || g->step_px <= 0.0)
        return -1;
    cx->L = o1_lattice(g);
    o1_weights(g, cx->w);
    if (g->det_radius > 0.0) {
        if (g->det_radius < cx->L.T || g->c_slope < 0.0 || g->r_slope < 0.0) return -1;
        cx->var = 1;
        cx->C = (double*)malloc(sizeof(double) * cx->L.n_t);
        cx->W = (double*)malloc(sizeof(double) * cx->L.n_t * g->n_subrays);
        if (!cx->C || !cx->W) { ctx_free(cx); return -2; }
        o13_tables(g, &cx->L, cx->C, cx->W);
    }
    return 0;
}

/* Export the O13 tables (pin P18 and the bit-exact comparison with the library). */
int orc_variant_tables(const orc_desc* g, double* C, double* W)
{
    orc_ctx cx;
    if (ctx_init(g, &cx)) return -1;
    if (!cx.var) { ctx_free(&cx); return -3; }
    memcpy(C, cx.C, sizeof(double) * cx.L.n_t);
    memcpy(W, cx.W, sizeof(double) * cx.L.n_t * g->n_subrays);
    ctx_free(&cx);
    return 0;
}

/* O3/O4 for one ray.  Returns g_ray; *dg_ray (if dlam) gets the JVP.
 * A_i = Delta*(1/2 mu_i + sum_{k>i} mu_k);  g = Delta * sum_i lam_i exp(-A_i)
 * dA_i = Delta*(1/2 dmu_i + sum_{k>i} dmu_k); dg = Delta * sum_i (dlam_i - lam_i dA_i) exp(-A_i) */
/* O13 (Cv, Wv non-NULL): g = Delta sum_i W_i lam_i exp(-c_i A_i),
 * dg = Delta sum_i W_i (dlam_i - lam_i c_i dA_i) exp(-c_i A_i)   (eq:d_fwd_model with r, c; eq:frechet) */
static double ray_fwd(const orc_lattice* L, int N, const double* lam, const double* mu,
                      const double* dlam, const double* dmu, double c, double s, double sigma,
                      int ilo, int ihi, double* dg_ray, const double* Cv, const double* Wv)
{
    double g = 0.0, dg = 0.0;
    double sum_mu = 0.0, sum_dmu = 0.0;      /* sum_{k>i} over samples nearer the detector */
    for (int i = ihi; i >= ilo; --i) {
        double u, v;
        o2_pos(L, c, s, sigma, i, &u, &v);
        double li = o2_sample(lam, N, u, v), mi = o2_sample(mu, N, u, v);
        double A = L->delta * (0.5 * mi + sum_mu);
        double ci = Cv ? Cv[i] : 1.0, wi = Wv ? Wv[i] : 1.0;
        double E = Cv ? exp(-ci * A) : exp(-A);
        g += Wv ? wi * li * E : li * E;
        if (dlam) {
            double dli = o2_sample(dlam, N, u, v), dmi = o2_sample(dmu, N, u, v);
            double dA = L->delta * (0.5 * dmi + sum_dmu);
            if (Cv) dg += wi * (dli - li * ci * dA) * E;
            else dg += (dli - li * dA) * E;
            sum_dmu += dmi;
        }
        sum_mu += mi;
    }
    if (dg_ray) *dg_ray = L->delta * dg;
    return L->delta * g;
}

/* Same value as ray_fwd's g, by the O(n^2) double loop written straight from the
 * definition (used only by the brute-force pin on tiny inputs). */
static double ray_fwd_naive(const orc_lattice* L, int N, const double* lam, const double* mu,
                            double c, double s, double sigma, int ilo, int ihi)
{
    double g = 0.0;
    for (int i = ilo; i <= ihi; ++i) {
        double u, v;
        o2_pos(L, c, s, sigma, i, &u, &v);
        double A = 0.5 * o2_sample(mu, N, u, v);
        for (int k = i + 1; k <= ihi; ++k) {
            double uk, vk;
            o2_pos(L, c, s, sigma, k, &uk, &vk);
            A += o2_sample(mu, N, uk, vk);
        }
        g += o2_sample(lam, N, u, v) * exp(-L->delta * A);
    }
    return L->delta * g;
}

/* O5 for one ray with adjoint weight wr:
 * a_lam(i) = wr*Delta*E_i; a_mu(i) = -wr*Delta^2*(sum_{k<i} lam_k E_k + 1/2 lam_i E_i) */
/* O13 (Cv, Wv non-NULL): a_lam(i) = wr Delta W_i E_i, a_mu(i) = -wr Delta^2 (sum_{k<i} W_k lam_k c_k E_k
 * + 1/2 W_i lam_i c_i E_i) with E_i = exp(-c_i A_i) (the transpose of the O13 JVP) */
static void ray_vjp(const orc_lattice* L, int N, const double* lam, const double* mu, double wr,
                    double c, double s, double sigma, int ilo, int ihi, double* glam, double* gmu,
                    double* buf, const double* Cv, const double* Wv)
{
    int n = ihi - ilo + 1;
    if (n <= 0) return;
    double* ls = buf;          /* lam_i */
    double* E = buf + n;       /* E_i   */
    double sum_mu = 0.0;
    for (int i = ihi; i >= ilo; --i) {
        double u, v;
        o2_pos(L, c, s, sigma, i, &u, &v);
        double mi = o2_sample(mu, N, u, v);
        ls[i - ilo] = o2_sample(lam, N, u, v);
        if (Cv) E[i - ilo] = exp(-Cv[i] * (L->delta * (0.5 * mi + sum_mu)));
        else E[i - ilo] = exp(-L->delta * (0.5 * mi + sum_mu));
        sum_mu += mi;
    }
    double prefix = 0.0;       /* sum_{k<i} lam_k E_k (samples farther from the detector) */
    for (int i = ilo; i <= ihi; ++i) {
        double u, v;
        o2_pos(L, c, s, sigma, i, &u, &v);
        double le = Cv ? Wv[i] * ls[i - ilo] * Cv[i] * E[i - ilo] : ls[i - ilo] * E[i - ilo];
        double al = Cv ? wr * L->delta * Wv[i] * E[i - ilo] : wr * L->delta * E[i - ilo];
        double am = -wr * L->delta * L->delta * (prefix + 0.5 * le);
        o2_scatter(glam, N, u, v, al);
        o2_scatter(gmu, N, u, v, am);
        prefix += le;
    }
}

/* ------------------------------------------------------------------ O14 pixel basis */
static int cmp_double(const void* a, const void* b)
{
    double x = *(const double*)a, y = *(const double*)b;
    return x < y ? -1 : (x > y ? 1 : 0);
}

/* The pixels a line x(t) = sigma omega_perp + t omega crosses in the image square [-1,1]^2, in order of
 * increasing t, with the length of the line inside each.  In pixel units (X = (x + 1) N/2, the pixel
 * edges at the integers 0..N): X(t) = X0 + t wX with X0 = (-sigma s + 1) N/2, wX = c N/2 (Y likewise,
 * from sigma c and s); every crossing t = (k - X0) / wX of an edge strictly between the line's entry
 * and exit of the square (slab clipping against [0, N]^2), plus the entry and exit, sorted; each
 * interval of positive length lies in one pixel, found from its midpoint: floor(X0 + t_mid wX).
 * (1/w is formed once per line and multiplied; a line exactly on the square's edge is outside.)
 * pix[q] = row * N + col, len[q] = interval length (domain units: omega is a unit vector),
 * tmid[q] = its midpoint t.  Returns M (<= 2N + 2). */
static int o14_cross(int N, double c, double s, double sigma, int* pix, double* len, double* tmid, double* ts)
{
    double hN = 0.5 * N;
    double X0[2] = {(-sigma * s + 1.0) * hN, (sigma * c + 1.0) * hN};
    double w[2] = {c * hN, s * hN};
    double inv[2] = {0.0, 0.0};
    double tin = -INFINITY, tout = INFINITY;
    for (int k = 0; k < 2; ++k) {
        if (w[k] == 0.0) {
            if (!(X0[k] > 0.0 && X0[k] < (double)N)) return 0;
        } else {
            inv[k] = 1.0 / w[k];
            double t1 = (0.0 - X0[k]) * inv[k], t2 = ((double)N - X0[k]) * inv[k];
            double lo = t1 < t2 ? t1 : t2, hi = t1 < t2 ? t2 : t1;
            if (lo > tin) tin = lo;
            if (hi < tout) tout = hi;
        }
    }
    if (!(tin < tout)) return 0;
    int n = 0;
    ts[n++] = tin;
    ts[n++] = tout;
    for (int k = 0; k < 2; ++k) {
        if (w[k] == 0.0) continue;
        for (int e = 0; e <= N; ++e) {
            double t = ((double)e - X0[k]) * inv[k];
            if (t > tin && t < tout) ts[n++] = t;
        }
    }
    qsort(ts, (size_t)n, sizeof(double), cmp_double);
    int M = 0;
    for (int q = 0; q + 1 < n; ++q) {
        double l = ts[q + 1] - ts[q];
        if (!(l > 0.0)) continue;
        double tm = 0.5 * (ts[q] + ts[q + 1]);
        int col = (int)floor(X0[0] + tm * w[0]);
        int row = (int)floor(X0[1] + tm * w[1]);
        if (col < 0) col = 0;
        if (col > N - 1) col = N - 1;
        if (row < 0) row = 0;
        if (row > N - 1) row = N - 1;
        pix[M] = row * N + col;
        len[M] = l;
        tmid[M] = tm;
        ++M;
    }
    return M;
}

/* O13 response at distance d to the detector, for sub-ray j: c(d) = 1 + c_slope d and the normalised
 * Gaussian W_j(d) of width subray_sigma * pitch * (1 + r_slope d) (the same functions as o13_tables) */
static void o14_resp(const orc_desc* g, double d, int j, double* C, double* W)
{
    int J = g->n_subrays;
    double p = 2.0 / (g->n_det - 1);
    double sp = g->subray_sigma * p * (1.0 + g->r_slope * d);
    double sum = 0.0, wj = 0.0;
    for (int k = 0; k < J; ++k) {
        double dk = (double)(2 * k + 1 - J) / (double)(2 * J) * p;
        double e = exp(-(dk * dk) / (2.0 * sp * sp));
        sum += e;
        if (k == j) wj = e;
    }
    *C = 1.0 + g->c_slope * d;
    *W = wj / sum;
}

/* one ray of the pixel basis: g = sum_q r_q lam_q E_q, E_q = exp(-c_q A_q),
 * A_q = l_q mu_q / 2 + sum_{p>q} l_p mu_p;  JVP dg = sum_q r_q (dlam_q - lam_q c_q dA_q) E_q  (eq:frechet) */
static double ray_fwd_pb(const orc_desc* g, int var, int j, int M, const int* pix, const double* len,
                         const double* tmid, const double* lam, const double* mu, const double* dlam,
                         const double* dmu, double* dg_ray)
{
    double gs = 0.0, dg = 0.0, sum_mu = 0.0, sum_dmu = 0.0;
    for (int q = M - 1; q >= 0; --q) {
        double l = len[q], cq = 1.0, rq = l;
        if (var) {
            double W;
            o14_resp(g, g->det_radius - tmid[q], j, &cq, &W);
            rq = W * l;
        }
        double A = 0.5 * l * mu[pix[q]] + sum_mu;
        double E = exp(-cq * A);
        gs += rq * lam[pix[q]] * E;
        if (dlam) {
            double dA = 0.5 * l * dmu[pix[q]] + sum_dmu;
            dg += rq * (dlam[pix[q]] - lam[pix[q]] * cq * dA) * E;
            sum_dmu += l * dmu[pix[q]];
        }
        sum_mu += l * mu[pix[q]];
    }
    if (dg_ray) *dg_ray = dg;
    return gs;
}

/* its transpose with weight wr: a_lam(q) = wr r_q E_q,
 * a_mu(q) = -wr l_q (sum_{p<q} r_p lam_p c_p E_p + 1/2 r_q lam_q c_q E_q) */
static void ray_vjp_pb(const orc_desc* g, int var, int j, int M, const int* pix, const double* len,
                       const double* tmid, const double* lam, const double* mu, double wr, double* glam,
                       double* gmu, double* buf)
{
    double* E = buf;
    double* R = buf + M;
    double* Cq = buf + 2 * M;
    double sum_mu = 0.0;
    for (int q = M - 1; q >= 0; --q) {
        double l = len[q], cq = 1.0, rq = l;
        if (var) {
            double W;
            o14_resp(g, g->det_radius - tmid[q], j, &cq, &W);
            rq = W * l;
        }
        E[q] = exp(-cq * (0.5 * l * mu[pix[q]] + sum_mu));
        R[q] = rq;
        Cq[q] = cq;
        sum_mu += l * mu[pix[q]];
    }
    double prefix = 0.0;   /* sum_{p<q} r_p lam_p c_p E_p (farther from the detector) */
    for (int q = 0; q < M; ++q) {
        double le = R[q] * lam[pix[q]] * Cq[q] * E[q];
        glam[pix[q]] += wr * R[q] * E[q];
        gmu[pix[q]] += -wr * len[q] * (prefix + 0.5 * le);
        prefix += le;
    }
}

/* Export one ray's crossings (pin P19: traversal against per-pixel clipping). */
int orc_pb_crossings(int N, double c, double s, double sigma, int* pix, double* len, double* tmid)
{
    double* ts = (double*)malloc(sizeof(double) * (2 * (N + 1) + 2));
    if (!ts) return -2;
    int M = o14_cross(N, c, s, sigma, pix, len, tmid, ts);
    free(ts);
    return M;
}

static int num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

int orc_threads(void) { return num_threads(); }

/* ------------------------------------------------------------------ O3 / O4 */
/* lam, mu, dlam, dmu: [B][N][N]; y, dy: [B][n_A][n_banks][n_det].  dlam==NULL -> forward only.
 * naive != 0 selects the O(n^2) quadrature (forward only). */
static int fwd_impl(const orc_desc* g, const double* lam, const double* mu, const double* dlam,
                    const double* dmu, double* y, double* dy, int naive)
{
    orc_ctx cx;
    if (ctx_init(g, &cx)) return -1;
    if (naive && (cx.var || g->pixel_basis)) { ctx_free(&cx); return -1; }
    int N = g->n_px, nA = g->n_angles, nB = g->n_banks, nd = g->n_det, J = g->n_subrays;
    long n_ab = (long)g->batch * nA * nB;
    size_t npx = (size_t)N * N;
#pragma omp parallel for schedule(static)
    for (long q = 0; q < n_ab; ++q) {
        int b = (int)(q % nB), a = (int)((q / nB) % nA);
        long m = q / ((long)nA * nB);
        const double* l = lam + m * npx;
        const double* u = mu + m * npx;
        const double* dl = dlam ? dlam + m * npx : NULL;
        const double* du = dmu ? dmu + m * npx : NULL;
        double c, s;
        o1_dir(g, a, b, &c, &s);
        int* pix = NULL;
        double *len = NULL, *tmid = NULL, *ts = NULL;
        if (g->pixel_basis) {   /* O14 crossing buffers */
            pix = (int*)malloc(sizeof(int) * (2 * N + 4));
            len = (double*)malloc(sizeof(double) * (2 * N + 4) * 3 + sizeof(double) * 2);
            tmid = len + (2 * N + 4);
            ts = tmid + (2 * N + 4);
        }
        for (int d = 0; d < nd; ++d) {
            double acc = 0.0, dacc = 0.0;
            for (int j = 0; j < J; ++j) {
                double sigma = o1_offset(g, b, d, j);
                int ilo, ihi;
                o1_clip(g, &cx.L, c, s, sigma, &ilo, &ihi);
                double gj, dgj = 0.0;
                if (g->pixel_basis) {
                    int M = o14_cross(N, c, s, sigma, pix, len, tmid, ts);
                    gj = ray_fwd_pb(g, cx.var, j, M, pix, len, tmid, l, u, dl, du, dl ? &dgj : NULL);
                } else if (naive)
                    gj = ray_fwd_naive(&cx.L, N, l, u, c, s, sigma, ilo, ihi);
                else
                    gj = ray_fwd(&cx.L, N, l, u, dl, du, c, s, sigma, ilo, ihi, dl ? &dgj : NULL,
                                 cx.var ? cx.C : NULL, cx.var ? cx.W + (size_t)j * cx.L.n_t : NULL);
                if (cx.var) {                        /* O13: the response is inside the ray sum */
                    acc += gj;
                    dacc += dgj;
                } else {
                    acc += cx.w[j] * gj;             /* y = sum_j w_j g_ray */
                    dacc += cx.w[j] * dgj;
                }
            }
            if (y) y[q * nd + d] = acc;
            if (dy) dy[q * nd + d] = dacc;
        }
        free(pix);
        free(len);
    }
    ctx_free(&cx);
    return 0;
}

int orc_forward(const orc_desc* g, const double* lam, const double* mu, double* y)
{
    return fwd_impl(g, lam, mu, NULL, NULL, y, NULL, 0);
}

int orc_forward_naive(const orc_desc* g, const double* lam, const double* mu, double* y)
{
    return fwd_impl(g, lam, mu, NULL, NULL, y, NULL, 1);
}

int orc_jvp(const orc_desc* g, const double* lam, const double* mu, const double* dlam,
            const double* dmu, double* y, double* dy)
{
    return fwd_impl(g, lam, mu, dlam, dmu, y, dy, 0);
}

/* ------------------------------------------------------------------ O5 */
int orc_vjp(const orc_desc* g, const double* lam, const double* mu, const double* w, double* glam,
            double* gmu)
{
    orc_ctx cx;
    if (ctx_init(g, &cx)) return -1;
    int N = g->n_px, nA = g->n_angles, nB = g->n_banks, nd = g->n_det, J = g->n_subrays;
    size_t npx = (size_t)N * N;
    int nth = num_threads();
    memset(glam, 0, sizeof(double) * npx * g->batch);
    memset(gmu, 0, sizeof(double) * npx * g->batch);
    for (int m = 0; m < g->batch; ++m) {
        double* priv = (double*)calloc((size_t)nth * 2 * npx, sizeof(double));
        if (!priv) { ctx_free(&cx); return -2; }
        const double* l = lam + m * npx;
        const double* u = mu + m * npx;
#pragma omp parallel
        {
            int tid = 0;
#ifdef _OPENMP
            tid = omp_get_thread_num();
#endif
            double* gl = priv + (size_t)tid * 2 * npx;
            double* gm = gl + npx;
            double* buf = (double*)malloc(sizeof(double) * 2 * (cx.L.n_t + 1));
            int* pix = (int*)malloc(sizeof(int) * (2 * N + 4));       /* O14 crossing buffers */
            double* len = (double*)malloc(sizeof(double) * (2 * N + 4) * 6 + sizeof(double) * 2);
            double* tmid = len + (2 * N + 4);
            double* pbuf = tmid + (2 * N + 4);
            double* ts = pbuf + 3 * (2 * N + 4);
#pragma omp for schedule(static)
            for (int q = 0; q < nA * nB; ++q) {
                int b = q % nB, a = q / nB;
                double c, s;
                o1_dir(g, a, b, &c, &s);
                for (int d = 0; d < nd; ++d) {
                    double wd = w[((size_t)m * nA * nB + q) * nd + d];
                    for (int j = 0; j < J; ++j) {
                        double sigma = o1_offset(g, b, d, j);
                        int ilo, ihi;
                        o1_clip(g, &cx.L, c, s, sigma, &ilo, &ihi);
                        if (g->pixel_basis) {   /* O14 (with the O13 response W_j inside the ray sum) */
                            int M = o14_cross(N, c, s, sigma, pix, len, tmid, ts);
                            ray_vjp_pb(g, cx.var, j, M, pix, len, tmid, l, u, cx.var ? wd : cx.w[j] * wd, gl, gm, pbuf);
                        } else if (cx.var)   /* O13: the response W_j(d_i) is inside the ray sum */
                            ray_vjp(&cx.L, N, l, u, wd, c, s, sigma, ilo, ihi, gl, gm, buf, cx.C,
                                    cx.W + (size_t)j * cx.L.n_t);
                        else
                            ray_vjp(&cx.L, N, l, u, cx.w[j] * wd, c, s, sigma, ilo, ihi, gl, gm, buf, NULL, NULL);
                    }
                }
            }
            free(buf);
            free(pix);
            free(len);
        }
        for (int t = 0; t < nth; ++t)
            for (size_t k = 0; k < npx; ++k) {
                glam[m * npx + k] += priv[(size_t)t * 2 * npx + k];
                gmu[m * npx + k] += priv[(size_t)t * 2 * npx + npx + k];
            }
        free(priv);
    }
    ctx_free(&cx);
    return 0;
}

/* ------------------------------------------------------------------ O6 regulariser */
/* (Lu)[j][i] = 4u[j][i] - u[j][i-1] - u[j][i+1] - u[j-1][i] - u[j+1][i], zero outside */
void orc_laplacian(int N, int batch, const double* u, double* Lu)
{
    for (int m = 0; m < batch; ++m) {
        const double* x = u + (size_t)m * N * N;
        double* o = Lu + (size_t)m * N * N;
        for (int j = 0; j < N; ++j)
            for (int i = 0; i < N; ++i)
                o[j * N + i] = 4.0 * x[j * N + i] - o2_pix(x, N, j, i - 1) - o2_pix(x, N, j, i + 1)
                             - o2_pix(x, N, j - 1, i) - o2_pix(x, N, j + 1, i);
    }
}

static double dot(const double* a, const double* b, size_t n)
{
    double s = 0.0;
    for (size_t k = 0; k < n; ++k) s += a[k] * b[k];
    return s;
}

/* ------------------------------------------------------------------ O10 geometry priors */
/* P1 = diag(m1), P2 = diag(m2) over [batch][N][N]; a1, a2 the weights at alpha^(0); scale the
 * continuation factor alpha_k / alpha_0 (orc_lm_solve sets it per iteration). */
static struct {
    const double *m1, *m2;
    double a1, a2, scale;
} g_prior = {NULL, NULL, 0.0, 0.0, 1.0};

void orc_set_prior(const double* m1, const double* m2, double a1, double a2)
{
    g_prior.m1 = m1;
    g_prior.m2 = m2;
    g_prior.a1 = m1 ? a1 : 0.0;
    g_prior.a2 = m2 ? a2 : 0.0;
    g_prior.scale = 1.0;
}

/* alpha1/2 ||P1 x_lam||^2 + alpha2/2 ||P2 x_mu||^2 at the current continuation scale */
static double prior_value(const double* xl, const double* xm, size_t npx)
{
    double v = 0.0;
    for (size_t k = 0; k < npx; ++k) {
        if (g_prior.m1) v += 0.5 * g_prior.a1 * g_prior.scale * (g_prior.m1[k] * xl[k]) * (g_prior.m1[k] * xl[k]);
        if (g_prior.m2) v += 0.5 * g_prior.a2 * g_prior.scale * (g_prior.m2[k] * xm[k]) * (g_prior.m2[k] * xm[k]);
    }
    return v;
}

/* out += P^T P x, weighted: out_lam += alpha1 m1^2 x_lam, out_mu += alpha2 m2^2 x_mu (the gradient of
 * prior_value, and its Hessian applied to x) */
static void prior_apply(const double* xl, const double* xm, double* ol, double* om, size_t npx)
{
    for (size_t k = 0; k < npx; ++k) {
        if (g_prior.m1) ol[k] += g_prior.a1 * g_prior.scale * g_prior.m1[k] * g_prior.m1[k] * xl[k];
        if (g_prior.m2) om[k] += g_prior.a2 * g_prior.scale * g_prior.m2[k] * g_prior.m2[k] * xm[k];
    }
}

/* ------------------------------------------------------------------ O7 GN-CG step + LM wrap */
/* Stats layout (double[16 + n_cg + 1]):
 *  0 f(u)   1 1/2||r||^2   2 R(u)   3 ||b||   4 pred = m(0)-m(s)   5 f(u+s)   6 rho
 *  7 accepted   8 beta_next   9 CG steps done   10 breakdown   11 beta_min   12 ||Js||^2
 *  13 alpha||Ls||^2   14 <b,s>   15 (unused)   16.. ||z_k|| for k = 0..n_cg            */
#define ST_CG 16

typedef struct {
    const orc_desc* g;
    const double *lam, *mu;
    double alpha, beta;
    size_t npx;
    double *tmp_y, *tl, *tm;
} hctx;

/* H p = J^T(J p) + alpha L^T L p + beta p  (p, out stacked [lam-part | mu-part]) */
static int apply_H(hctx* H, const double* p, double* out)
{
    size_t n = H->npx;
    if (orc_jvp(H->g, H->lam, H->mu, p, p + n, NULL, H->tmp_y)) return -1;
    if (orc_vjp(H->g, H->lam, H->mu, H->tmp_y, out, out + n)) return -1;
    for (int f = 0; f < 2; ++f) {
        orc_laplacian(H->g->n_px, H->g->batch, p + f * n, H->tl);
        orc_laplacian(H->g->n_px, H->g->batch, H->tl, H->tm);
        for (size_t k = 0; k < n; ++k) out[f * n + k] += H->alpha * H->tm[k] + H->beta * p[f * n + k];
    }
    prior_apply(p, p + n, out, out + n, n);   /* + P^T P p (O10) */
    return 0;
}

static double objective(const orc_desc* g, const double* lam, const double* mu, const double* y,
                        double alpha, double* misfit, double* reg, double* r_out, double* tl)
{
    size_t ns = (size_t)g->batch * g->n_angles * g->n_banks * g->n_det;
    size_t npx = (size_t)g->batch * g->n_px * g->n_px;
    double* r = r_out;
    orc_forward(g, lam, mu, r);
    for (size_t k = 0; k < ns; ++k) r[k] = r[k] - y[k];           /* r = F(u) - y */
    *misfit = 0.5 * dot(r, r, ns);
    orc_laplacian(g->n_px, g->batch, lam, tl);
    double q = dot(tl, tl, npx);
    orc_laplacian(g->n_px, g->batch, mu, tl);
    q += dot(tl, tl, npx);
    *reg = 0.5 * alpha * q;                                       /* R(u) = alpha/2 (||L lam||^2 + ||L mu||^2) */
    *reg += prior_value(lam, mu, npx);                            /* + alpha1/2 ||P1 lam||^2 + alpha2/2 ||P2 mu||^2 */
    return *misfit + *reg;
}

/* One LM iteration; box (NULL or {lam_lo, lam_hi, mu_lo, mu_hi}) replaces the CG step by the step
 * actually taken inside the box, s' = clamp(u + s) - u, before pred and the trial (reading R-N1). */
static int lm_step(const orc_desc* g, const double* lam, const double* mu, const double* y, double alpha,
                   double beta, int n_cg, const double* box, int sgp, double* s_lam, double* s_mu, double* stats);

int orc_gn_cg_step(const orc_desc* g, const double* lam, const double* mu, const double* y,
                   double alpha, double beta, int n_cg, double* s_lam, double* s_mu, double* stats)
{
    return lm_step(g, lam, mu, y, alpha, beta, n_cg, NULL, 0, s_lam, s_mu, stats);
}

static double clampd(double x, double lo, double hi) { return x < lo ? lo : (x > hi ? hi : x); }

/* Euclidean projection of one pixel's (lam, mu) onto the feasible set of the LM solve (O12, N1):
 * the box [box0, box1] x [box2, box3] and, when box4 = c > 0, the linear constraint lam <= c mu ("low
 * attenuation but highly emitting materials are not allowed"; reading R-lin).  If the
 * box projection satisfies lam <= c mu it is the projection; otherwise the projection lies on the
 * line lam = c mu, at the line parameter t* = (c lam + mu) / (c^2 + 1) clamped to the line's segment
 * inside the box. */
static void projK(double* l, double* m, const double* box)
{
    double pl = clampd(*l, box[0], box[1]), pm = clampd(*m, box[2], box[3]);
    const double c = box[4];
    if (c > 0.0 && pl > c * pm) {
        double t = (c * *l + *m) / (c * c + 1.0);
        double tlo = fmax(box[0] / c, box[2]), thi = fmin(box[1] / c, box[3]);
        t = clampd(t, tlo, thi);
        pl = c * t;
        pm = t;
    }
    *l = pl;
    *m = pm;
}

/* the projection of whole images (test entry point) */
void orc_project(double* lam, double* mu, size_t n, const double* box)
{
    for (size_t i = 0; i < n; ++i) projK(&lam[i], &mu[i], box);
}

/* One LM iteration with the box {lam_lo, lam_hi, mu_lo, mu_hi}: CG then projection (sgp = 0, reading
 * R-N1) or the SGP inner solver (sgp = 1, O11).  Stats as orc_gn_cg_step. */
int orc_lm_step_box(const orc_desc* g, const double* lam, const double* mu, const double* y, double alpha,
                    double beta, int n_it, const double* box, int sgp, double* s_lam, double* s_mu, double* stats)
{
    return lm_step(g, lam, mu, y, alpha, beta, n_it, box, sgp, s_lam, s_mu, stats);
}

static int lm_step(const orc_desc* g, const double* lam, const double* mu, const double* y, double alpha,
                   double beta, int n_cg, const double* box, int sgp, double* s_lam, double* s_mu, double* stats)
{
    size_t npx = (size_t)g->batch * g->n_px * g->n_px;
    size_t ns = (size_t)g->batch * g->n_angles * g->n_banks * g->n_det;
    size_t n2 = 2 * npx;
    double* r = (double*)malloc(sizeof(double) * ns);
    double* ys = (double*)malloc(sizeof(double) * ns);
    double* bvec = (double*)malloc(sizeof(double) * n2);
    double* s = (double*)calloc(n2, sizeof(double));
    double* z = (double*)malloc(sizeof(double) * n2);
    double* p = (double*)malloc(sizeof(double) * n2);
    double* q = (double*)malloc(sizeof(double) * n2);
    double* tl = (double*)malloc(sizeof(double) * npx);
    double* tm = (double*)malloc(sizeof(double) * npx);
    double* ut = (double*)malloc(sizeof(double) * n2);
    if (!r || !ys || !bvec || !s || !z || !p || !q || !tl || !tm || !ut) return -2;
    for (int k = 0; k < ST_CG + n_cg + 1; ++k) stats[k] = 0.0;

    /* 1-2: r = F(u) - y, f(u) = 1/2||r||^2 + R(u) */
    double misfit, reg;
    double f0 = objective(g, lam, mu, y, alpha, &misfit, &reg, r, tl);
    /* 3: b = -(J^T r + alpha L^T L u) */
    orc_vjp(g, lam, mu, r, bvec, bvec + npx);
    for (int f = 0; f < 2; ++f) {
        const double* uf = f ? mu : lam;
        orc_laplacian(g->n_px, g->batch, uf, tl);
        orc_laplacian(g->n_px, g->batch, tl, tm);
        for (size_t k = 0; k < npx; ++k) bvec[f * npx + k] = -(bvec[f * npx + k] + alpha * tm[k]);
    }
    {   /* - P^T P u (O10) */
        double* gp = (double*)calloc(2 * npx, sizeof(double));
        if (!gp) return -2;
        prior_apply(lam, mu, gp, gp + npx, npx);
        for (size_t k = 0; k < 2 * npx; ++k) bvec[k] -= gp[k];
        free(gp);
    }
    stats[0] = f0; stats[1] = misfit; stats[2] = reg; stats[3] = sqrt(dot(bvec, bvec, n2));

    hctx H = {g, lam, mu, alpha, beta, npx, ys, tl, tm};
    if (sgp && box) {
        /* 5': SGP (O11) on min q(s) = 1/2 s^T H s - b^T s over {s : u + s in box}, from s0 = 0 (u in
         * the box).  gq = H s - b; d = P(u + s - a gq) - u - s (projection onto the box); stop when
         * <gq, d> >= 0; lam_k = min(1, -<gq,d> / <d,Hd>) (exact minimiser of q on the segment, which
         * stays feasible); s += lam_k d, gq += lam_k H d; a alternates the two Barzilai-Borwein
         * lengths <ds,ds>/<ds,dg> and <ds,dg>/<dg,dg> (ds = lam_k d, dg = lam_k H d), clamped to
         * [1e-10, 1e10]; a_0 = 1.  stats[ST_CG + k] = ||d_k||. */
        double* gq = z;
        double* d = p;
        for (size_t i = 0; i < n2; ++i) gq[i] = -bvec[i];
        double a = 1.0, beta_min2 = 0.0;
        int k;
        for (k = 0; k < n_cg; ++k) {
            for (size_t i = 0; i < npx; ++i) {
                double pl = lam[i] + s[i] - a * gq[i], pm = mu[i] + s[npx + i] - a * gq[npx + i];
                projK(&pl, &pm, box);
                d[i] = pl - lam[i] - s[i];
                d[npx + i] = pm - mu[i] - s[npx + i];
            }
            double gd = dot(gq, d, n2), dd = dot(d, d, n2);
            stats[ST_CG + k] = sqrt(dd);
            if (!(gd < 0.0)) { stats[10] = 1.0; break; }
            apply_H(&H, d, q);
            double dHd = dot(d, q, n2);
            if (k == 0) beta_min2 = 1e-3 * dHd / dd;
            double lk = dHd > 0.0 ? fmin(1.0, -gd / dHd) : 1.0;
            for (size_t i = 0; i < n2; ++i) { s[i] += lk * d[i]; gq[i] += lk * q[i]; }
            double sy = lk * lk * dHd, ss = lk * lk * dd, yy = lk * lk * dot(q, q, n2);
            double an = (k % 2 == 0) ? (sy > 0.0 ? ss / sy : 1e10) : (yy > 0.0 ? sy / yy : 1e10);
            a = an < 1e-10 ? 1e-10 : (an > 1e10 ? 1e10 : an);
        }
        if (k == n_cg) {
            for (size_t i = 0; i < npx; ++i) {
                double pl = lam[i] + s[i] - a * gq[i], pm = mu[i] + s[npx + i] - a * gq[npx + i];
                projK(&pl, &pm, box);
                d[i] = pl - lam[i] - s[i];
                d[npx + i] = pm - mu[i] - s[npx + i];
            }
            stats[ST_CG + n_cg] = sqrt(dot(d, d, n2));
        }
        stats[9] = k;
        stats[11] = beta_min2;
        goto step_done;
    }
    /* 5: CG from s0 = 0 on H s = b */
    memcpy(z, bvec, sizeof(double) * n2);
    memcpy(p, bvec, sizeof(double) * n2);
    double zeta = dot(z, z, n2);
    stats[ST_CG + 0] = sqrt(zeta);
    double beta_min = 0.0;
    int k;
    for (k = 0; k < n_cg; ++k) {
        if (zeta == 0.0) { stats[10] = 1.0; break; }
        apply_H(&H, p, q);
        double gam = dot(p, q, n2);
        if (k == 0) beta_min = 1e-3 * gam / zeta;          /* 1e-3 <b,Hb>/<b,b> */
        if (gam <= 0.0) { stats[10] = 2.0; break; }
        double al = zeta / gam;
        for (size_t i = 0; i < n2; ++i) { s[i] += al * p[i]; z[i] -= al * q[i]; }
        double zeta2 = dot(z, z, n2);
        double bt = zeta2 / zeta;
        for (size_t i = 0; i < n2; ++i) p[i] = z[i] + bt * p[i];
        zeta = zeta2;
        stats[ST_CG + k + 1] = sqrt(zeta);
    }
    stats[9] = k;
    stats[11] = beta_min;
step_done:

    /* (N1) the step actually taken inside the box (a no-op for the feasible SGP step) */
    if (box)
        for (size_t i = 0; i < npx; ++i) {
            double pl = lam[i] + s[i], pm = mu[i] + s[npx + i];
            projK(&pl, &pm, box);
            s[i] = pl - lam[i];
            s[npx + i] = pm - mu[i];
        }
    /* 6: pred = <b,s> - 1/2(||Js||^2 + alpha||Ls||^2) */
    orc_jvp(g, lam, mu, s, s + npx, NULL, ys);
    double js2 = dot(ys, ys, ns);
    double ls2 = 0.0;
    for (int f = 0; f < 2; ++f) {
        orc_laplacian(g->n_px, g->batch, s + f * npx, tl);
        ls2 += dot(tl, tl, npx);
    }
    double bs = dot(bvec, s, n2);
    double ps2 = 2.0 * prior_value(s, s + npx, npx);              /* ||P s||^2, weighted (O10) */
    double pred = bs - 0.5 * (js2 + alpha * ls2 + ps2);
    stats[4] = pred; stats[12] = js2; stats[13] = alpha * ls2 + ps2; stats[14] = bs;

    /* 7: f(u+s), rho */
    for (size_t i = 0; i < npx; ++i) { ut[i] = lam[i] + s[i]; ut[npx + i] = mu[i] + s[npx + i]; }
    if (box)
        for (size_t i = 0; i < npx; ++i) {
            projK(&ut[i], &ut[npx + i], box);
        }
    double mis2, reg2;
    double f1 = objective(g, ut, ut + npx, y, alpha, &mis2, &reg2, r, tl);
    double rho = (f0 - f1) / pred;
    stats[5] = f1; stats[6] = rho;
    /* 8: accept iff pred > 0 and rho > eta = 0.1 (reading R-accept: rho compares the actual with the
     *    predicted decrease, PAPER.md:248 eq:rho_agreement, and only a positive predicted decrease makes
     *    rho > eta a decrease of f); beta update x10 (reject) / x0.2 (rho > 0.75) */
    int acc = pred > 0.0 && rho > 0.1;
    double bn = beta;
    if (!acc) bn = (10.0 * beta > beta_min) ? 10.0 * beta : beta_min;
    else if (rho > 0.75) bn = 0.2 * beta;
    stats[7] = acc; stats[8] = bn;

    memcpy(s_lam, s, sizeof(double) * npx);
    memcpy(s_mu, s + npx, sizeof(double) * npx);
    free(r); free(ys); free(bvec); free(s); free(z); free(p); free(q); free(tl); free(tm); free(ut);
    return 0;
}

/* ------------------------------------------------------------------ O8 Prop. 1 safeguard */
/* m_k(s) of eq:m-function, written out for the stacked operator
 * F~(u) = (F(lam,mu), sqrt(alpha) L lam, sqrt(alpha) L mu), y~ = (y, 0, 0) (reading Q10):
 *   r~ = F~(u) - y~,  F~'_k s = (J s, sqrt(alpha) L s_lam, sqrt(alpha) L s_mu),
 *   m_k(s) = 1/2 ||r~||^2 + <F~'_k s, r~> + 1/2 ||F~'_k s||^2.                                */
static double model_m(const orc_desc* g, const double* lam, const double* mu, const double* r,
                      const double* sl, const double* sm, double alpha, double* js, double* tl,
                      double* tm)
{
    size_t ns = (size_t)g->batch * g->n_angles * g->n_banks * g->n_det;
    size_t npx = (size_t)g->batch * g->n_px * g->n_px;
    double half_rr = 0.5 * dot(r, r, ns), cross = 0.0, half_ss = 0.0;
    orc_jvp(g, lam, mu, sl, sm, NULL, js);                      /* J s (eq:frechet) */
    cross += dot(js, r, ns);
    half_ss += 0.5 * dot(js, js, ns);
    for (int f = 0; f < 2; ++f) {
        orc_laplacian(g->n_px, g->batch, f ? mu : lam, tl);      /* sqrt(alpha) L u-part / sqrt(alpha) */
        orc_laplacian(g->n_px, g->batch, f ? sm : sl, tm);       /* sqrt(alpha) L s-part / sqrt(alpha) */
        half_rr += 0.5 * alpha * dot(tl, tl, npx);
        cross += alpha * dot(tm, tl, npx);
        half_ss += 0.5 * alpha * dot(tm, tm, npx);
    }
    /* the prior rows of F~ (O10): sqrt(alpha1) P1 lam, sqrt(alpha2) P2 mu, linear in u */
    half_rr += prior_value(lam, mu, npx);
    half_ss += prior_value(sl, sm, npx);
    {
        double* gp = (double*)calloc(2 * npx, sizeof(double));
        if (gp) {
            prior_apply(lam, mu, gp, gp + npx, npx);
            cross += dot(gp, sl, npx) + dot(gp + npx, sm, npx);
            free(gp);
        }
    }
    return half_rr + cross + half_ss;
}

/* Proposition 1 / the check of Algorithm 2 for one
 * candidate u~ = (c_lam, c_mu) and the LM step s_k = (s_lam, s_mu) at u_k = (lam, mu):
 *   s~ = u~ - u_k;  rho_k(s~) = (f(u_k) - f(u~)) / (m_k(0) - m_k(s~))   (eq:rho_agreement)
 *   u_{k+1} = u~ if m_k(s~) <= m_k(s_k) and rho_k(s~) > kappa, else u_k + s_k (eq:uk+1_condition)
 * plus m_k(0) - m_k(s~) > 0 (reading R-safeguard: rho undefined / the model does not decrease).
 * out: [0] f(u_k)  [1] f(u~)  [2] m_k(0)  [3] m_k(s~)  [4] m_k(s_k)  [5] rho_k(s~)  [6] accepted.
 * u_next (2 npx, [lam | mu]) receives u_{k+1}.  The whole descriptor (all batch members) is one
 * problem here; the Python wrapper calls it per member.                                           */
int orc_safeguard(const orc_desc* g, const double* lam, const double* mu, const double* y,
                  const double* s_lam, const double* s_mu, const double* c_lam, const double* c_mu,
                  double alpha, double kappa, double* u_next, double* out)
{
    size_t npx = (size_t)g->batch * g->n_px * g->n_px;
    size_t ns = (size_t)g->batch * g->n_angles * g->n_banks * g->n_det;
    double* r = (double*)malloc(sizeof(double) * ns);
    double* js = (double*)malloc(sizeof(double) * ns);
    double* tl = (double*)malloc(sizeof(double) * npx);
    double* tm = (double*)malloc(sizeof(double) * npx);
    double* st = (double*)malloc(sizeof(double) * 2 * npx);
    double* z = (double*)calloc(2 * npx, sizeof(double));
    if (!r || !js || !tl || !tm || !st || !z) return -2;
    double mis, reg;
    double f0 = objective(g, lam, mu, y, alpha, &mis, &reg, r, tl);    /* r = F(u_k) - y */
    for (size_t i = 0; i < npx; ++i) { st[i] = c_lam[i] - lam[i]; st[npx + i] = c_mu[i] - mu[i]; }
    double m0 = model_m(g, lam, mu, r, z, z + npx, alpha, js, tl, tm);
    double mc = model_m(g, lam, mu, r, st, st + npx, alpha, js, tl, tm);
    double ml = model_m(g, lam, mu, r, s_lam, s_mu, alpha, js, tl, tm);
    double fc = objective(g, c_lam, c_mu, y, alpha, &mis, &reg, js, tl);
    double pred = m0 - mc;
    double rho = pred != 0.0 ? (f0 - fc) / pred : 0.0;
    int acc = mc <= ml && pred > 0.0 && rho > kappa;
    for (size_t i = 0; i < npx; ++i) {
        u_next[i] = acc ? c_lam[i] : lam[i] + s_lam[i];
        u_next[npx + i] = acc ? c_mu[i] : mu[i] + s_mu[i];
    }
    out[0] = f0; out[1] = fc; out[2] = m0; out[3] = mc; out[4] = ml; out[5] = rho; out[6] = acc;
    free(r); free(js); free(tl); free(tm); free(st); free(z);
    return 0;
}

/* ------------------------------------------------------------------ O9 LM solve (N1) */
/* n_iter LM iterations: alpha_k = alpha0 / decay^min(k, k_freeze),
 * beta_0 = beta0 then beta_{k+1} = beta_next of iteration k, u_{k+1} = trial point if rho > 0.1 else
 * u_k; with a box the initial guess is clamped and every step projected (lm_step).  lam, mu updated
 * in place; stats: n_iter rows of (ST_CG + n_cg + 1) doubles as orc_gn_cg_step's. */
int orc_lm_solve(const orc_desc* g, double* lam, double* mu, const double* y, int n_iter, int n_cg,
                 double alpha0, double decay, int k_freeze, double beta0, const double* box, int sgp,
                 double* stats)
{
    size_t npx = (size_t)g->batch * g->n_px * g->n_px;
    double* sl = (double*)malloc(sizeof(double) * npx);
    double* sm = (double*)malloc(sizeof(double) * npx);
    if (!sl || !sm) return -2;
    if (box)
        for (size_t i = 0; i < npx; ++i) projK(&lam[i], &mu[i], box);
    double alpha = alpha0, beta = beta0, pscale = 1.0;
    const int row = ST_CG + n_cg + 1;
    for (int k = 0; k < n_iter; ++k) {
        if (k > 0 && k <= k_freeze) { alpha /= decay; pscale /= decay; }   /* (alpha, alpha1, alpha2) / decay^k */
        g_prior.scale = pscale;
        double* st = stats + (size_t)k * row;
        int rc = lm_step(g, lam, mu, y, alpha, beta, n_cg, box, sgp, sl, sm, st);
        if (rc) { g_prior.scale = 1.0; free(sl); free(sm); return rc; }
        if (st[7] != 0.0)
            for (size_t i = 0; i < npx; ++i) {
                double a = lam[i] + sl[i], b = mu[i] + sm[i];
                if (box) projK(&a, &b, box);
                lam[i] = a;
                mu[i] = b;
            }
        beta = st[8];
    }
    g_prior.scale = 1.0;
    free(sl); free(sm);
    return 0;
}

/* H applied to a given p (operator-level parity pin of the GN product). */
int orc_apply_H(const orc_desc* g, const double* lam, const double* mu, double alpha, double beta,
                const double* p, double* out)
{
    size_t npx = (size_t)g->batch * g->n_px * g->n_px;
    size_t ns = (size_t)g->batch * g->n_angles * g->n_banks * g->n_det;
    double* ys = (double*)malloc(sizeof(double) * ns);
    double* tl = (double*)malloc(sizeof(double) * npx);
    double* tm = (double*)malloc(sizeof(double) * npx);
    hctx H = {g, lam, mu, alpha, beta, npx, ys, tl, tm};
    int rc = apply_H(&H, p, out);
    free(ys); free(tl); free(tm);
    return rc;
}

/* Per-ray quadrature on explicit sample values (pin P3 / P9 use it directly). */
double orc_ray_quadrature(int n, const double* lam_s, const double* mu_s, double delta)
{
    double g = 0.0, sum_mu = 0.0;
    for (int i = n - 1; i >= 0; --i) {
        g += lam_s[i] * exp(-delta * (0.5 * mu_s[i] + sum_mu));
        sum_mu += mu_s[i];
    }
    return delta * g;
}

/* Per-ray adjoint coefficients on explicit sample values: dg/dlam_i, dg/dmu_i (pin P9). */
void orc_ray_adjoint(int n, const double* lam_s, const double* mu_s, double delta, double* dl,
                     double* dm)
{
    double sum_mu = 0.0;
    for (int i = n - 1; i >= 0; --i) {
        dl[i] = exp(-delta * (0.5 * mu_s[i] + sum_mu));   /* E_i, scaled below */
        sum_mu += mu_s[i];
    }
    double prefix = 0.0;
    for (int i = 0; i < n; ++i) {
        double le = lam_s[i] * dl[i];
        dm[i] = -delta * delta * (prefix + 0.5 * le);
        prefix += le;
        dl[i] = delta * dl[i];
    }
}
