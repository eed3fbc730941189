// kernels.cu -- the vector kernels of the PGET hot path on sm_100a: image packing for the
// projector (proj.cu), the regulariser, residual and objective reductions and the CG updates of
// the LM iteration.  Reductions use per-member fp64
// block partials over a fixed grid, so every scalar is deterministic.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.h"
#include <cstdlib>

#include "kernels.cuh"

namespace pget {

// ------------------------------------------------------------------------------------------
// image packing: padded P x P images with a zero halo of kHalo pixels, in the normal and in the
// transposed orientation (orientation class 1 of the projector samples the transposed copy).
// Euclidean projection of one pixel's (lam, mu) onto the feasible set (oracle O12): the box, then, if
// lam > c mu, the closest point of the segment of the line lam = c mu inside the box
__device__ __forceinline__ void proj_k(float& l, float& m, const BoxK& k)
{
    float pl = fminf(fmaxf(l, k.b.x), k.b.y), pm = fminf(fmaxf(m, k.b.z), k.b.w);
    if (k.c > 0.f && pl > k.c * pm) {
        float t = (k.c * l + m) / (k.c * k.c + 1.f);
        t = fminf(fmaxf(t, fmaxf(k.b.x / k.c, k.b.z)), fminf(k.b.y / k.c, k.b.w));
        pl = k.c * t;
        pm = t;
    }
    l = pl;
    m = pm;
}

__global__ void pack2_kernel(const float* __restrict__ lam, const float* __restrict__ mu,
                             const float* __restrict__ slam, const float* __restrict__ smu, float2* out,
                             float2* outT, float* ut_lam, float* ut_mu, int N, int P, int B, int has_box,
                             BoxK box)
{
    pdl_entry();
    // has_box: box = (lam_lo, lam_hi, mu_lo, mu_hi) clamps the trial point u + s
    const size_t total = static_cast<size_t>(B) * P * P;
    for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int ip = static_cast<int>(e % P);
        const int jp = static_cast<int>((e / P) % P);
        const size_t m = e / (static_cast<size_t>(P) * P);
        const int i = ip - kHalo, j = jp - kHalo;
        float2 val = make_float2(0.f, 0.f);
        if (i >= 0 && i < N && j >= 0 && j < N) {
            const size_t src = (m * N + j) * N + i;
            val = make_float2(lam[src], mu[src]);
            if (slam) {
                val.x += slam[src];
                val.y += smu[src];
                if (has_box) proj_k(val.x, val.y, box);
                ut_lam[src] = val.x;
                ut_mu[src] = val.y;
            }
        }
        out[e] = val;
        outT[(m * P + ip) * P + jp] = val;
    }
}

__global__ void pack4_kernel(const float* __restrict__ lam, const float* __restrict__ mu,
                             const float* __restrict__ dl, const float* __restrict__ dm, float4* out, float4* outT,
                             int N, int P, int B)
{
    pdl_entry();
    const size_t total = static_cast<size_t>(B) * P * P;
    for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int ip = static_cast<int>(e % P);
        const int jp = static_cast<int>((e / P) % P);
        const size_t m = e / (static_cast<size_t>(P) * P);
        const int i = ip - kHalo, j = jp - kHalo;
        float4 val = make_float4(0.f, 0.f, 0.f, 0.f);
        if (i >= 0 && i < N && j >= 0 && j < N) {
            const size_t src = (m * N + j) * N + i;
            val = make_float4(lam[src], mu[src], dl[src], dm[src]);
        }
        out[e] = val;
        outT[(m * P + ip) * P + jp] = val;
    }
}

// ------------------------------------------------------------------------------------------
// Vector kernels of the GN/LM wrap.  Per-member fp64 block partials, fixed grid -> fixed order.
__device__ __forceinline__ double block_sum(double v, double* sh)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) sh[w] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x == 0)
        for (int k = 0; k < (blockDim.x >> 5); ++k) t += sh[k];
    return t;
}

// (L x)[j][i], zero outside the grid (5-point Laplacian, reading Q10)
__device__ __forceinline__ float lap_at(const float* __restrict__ x, int N, int j, int i)
{
    if (i < 0 || i >= N || j < 0 || j >= N) return 0.f;
    const float c = x[j * N + i];
    float s = 4.f * c;
    if (i > 0) s -= x[j * N + i - 1];
    if (i < N - 1) s -= x[j * N + i + 1];
    if (j > 0) s -= x[(j - 1) * N + i];
    if (j < N - 1) s -= x[(j + 1) * N + i];
    return s;
}

// (P1^T P1 x_lam, P2^T P2 x_mu) weighted, added to (ol, om) at element k of [B][N][N] (priors)
__device__ __forceinline__ void prior_op(const PriorArgs& pr, size_t k, float xl, float xm, float& ol, float& om)
{
    if (pr.m1) { const float m = pr.m1[k]; ol += pr.a1 * (m * m) * xl; }
    if (pr.m2) { const float m = pr.m2[k]; om += pr.a2 * (m * m) * xm; }
}

__device__ __forceinline__ float lap2_at(const float* __restrict__ x, int N, int j, int i)
{
    return 4.f * lap_at(x, N, j, i) - lap_at(x, N, j, i - 1) - lap_at(x, N, j, i + 1) -
           lap_at(x, N, j - 1, i) - lap_at(x, N, j + 1, i);
}

// out = sign * (acc_interior + alpha L^T L x + beta x) over both parts; partial <dotv, out>.
//   grad mode (VJP out):  alpha = beta = 0, sign = 1, dotv = NULL
//   b = -(J^T r + alpha L^T L u):  sign = -1, x = u, beta = 0, dotv = out (||b||^2), also copies
//   q = J^T J p + alpha L^T L p + beta p:  sign = 1, x = p, dotv = p
__global__ void finish_kernel(const double2* __restrict__ part, int G, const float* __restrict__ xl,
                              const float* __restrict__ xm, float alpha, float beta, float sign,
                              float* outl, float* outm, const float* __restrict__ dotl,
                              const float* __restrict__ dotm, double* partial, float* copy1l, float* copy1m,
                              float* copy2l, float* copy2m, float* zerol, float* zerom, int N, PriorArgs pr,
                              const float* betav)
{
    pdl_entry();
    __shared__ double sh[32];
    const int m = blockIdx.y;
    const size_t n2 = static_cast<size_t>(N) * N;
    const size_t base = m * n2;
    double dsum = 0.0;
    for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < n2;
         e += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int i = static_cast<int>(static_cast<unsigned>(e) % static_cast<unsigned>(N)),   // e < N^2 < 2^32
                  j = static_cast<int>(static_cast<unsigned>(e) / static_cast<unsigned>(N));
        double2 a = part[base + e];   // the G fp64 partials of reduce_slots_kernel, in order
        for (int g0 = 1; g0 < G; g0 += 8) {
            double2 b[8];
#pragma unroll
            for (int t = 0; t < 8; ++t)
                b[t] = g0 + t < G ? part[static_cast<size_t>(g0 + t) * gridDim.y * n2 + base + e] : make_double2(0.0, 0.0);
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                if (g0 + t < G) {
                    a.x += b[t].x;
                    a.y += b[t].y;
                }
            }
        }
        float ol = static_cast<float>(a.x), om = static_cast<float>(a.y);
        if (xl) {
            const float* pl = xl + base;
            const float* pm = xm + base;
            const float bt = betav ? betav[m] : beta;   // per-member LM parameter (LM solve)
            ol += alpha * lap2_at(pl, N, j, i) + bt * pl[e];
            om += alpha * lap2_at(pm, N, j, i) + bt * pm[e];
            prior_op(pr, base + e, pl[e], pm[e], ol, om);
        }
        ol *= sign;
        om *= sign;
        outl[base + e] = ol;
        outm[base + e] = om;
        if (copy1l) { copy1l[base + e] = ol; copy1m[base + e] = om; }
        if (copy2l) { copy2l[base + e] = ol; copy2m[base + e] = om; }
        if (zerol) { zerol[base + e] = 0.f; zerom[base + e] = 0.f; }
        if (dotl) dsum += static_cast<double>(ol) * dotl[base + e] + static_cast<double>(om) * dotm[base + e];
    }
    if (partial) {
        const double t = block_sum(dsum, sh);
        if (threadIdx.x == 0) partial[m * gridDim.x + blockIdx.x] = t;
    }
}

// r = y - ymeas (in place into y), partial 1/2||r||^2
__global__ void residual_kernel(float* y, const float* __restrict__ ymeas, double* partial, int nper)
{
    pdl_entry();
    __shared__ double sh[32];
    const int m = blockIdx.y;
    double s = 0.0;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < nper; e += gridDim.x * blockDim.x) {
        const size_t k = static_cast<size_t>(m) * nper + e;
        const float r = y[k] - ymeas[k];
        y[k] = r;
        s += static_cast<double>(r) * r;
    }
    const double t = block_sum(0.5 * s, sh);
    if (threadIdx.x == 0) partial[m * gridDim.x + blockIdx.x] = t;
}

// partial sum of squares of a per-member vector
__global__ void sumsq_kernel(const float* __restrict__ x, double* partial, int nper)
{
    pdl_entry();
    __shared__ double sh[32];
    const int m = blockIdx.y;
    double s = 0.0;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < nper; e += gridDim.x * blockDim.x) {
        const double v = x[static_cast<size_t>(m) * nper + e];
        s += v * v;
    }
    const double t = block_sum(s, sh);
    if (threadIdx.x == 0) partial[m * gridDim.x + blockIdx.x] = t;
}

// partial ||L xl||^2 + ||L xm||^2
__global__ void regsq_kernel(const float* __restrict__ xl, const float* __restrict__ xm, double* partial, int N)
{
    pdl_entry();
    __shared__ double sh[32];
    const int m = blockIdx.y;
    const size_t n2 = static_cast<size_t>(N) * N;
    double s = 0.0;
    for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < n2;
         e += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int i = static_cast<int>(static_cast<unsigned>(e) % static_cast<unsigned>(N)),   // e < N^2 < 2^32
                  j = static_cast<int>(static_cast<unsigned>(e) / static_cast<unsigned>(N));
        const double a = lap_at(xl + m * n2, N, j, i), b = lap_at(xm + m * n2, N, j, i);
        s += a * a + b * b;
    }
    const double t = block_sum(s, sh);
    if (threadIdx.x == 0) partial[m * gridDim.x + blockIdx.x] = t;
}

// priors: partial sum a1 (m1 x_lam)^2 + a2 (m2 x_mu)^2 (twice the penalty)
__global__ void priorsq_kernel(const float* __restrict__ xl, const float* __restrict__ xm, PriorArgs pr,
                               double* partial, int N)
{
    pdl_entry();
    __shared__ double sh[32];
    const int m = blockIdx.y;
    const size_t n2 = static_cast<size_t>(N) * N;
    double s = 0.0;
    for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < n2;
         e += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const size_t k = m * n2 + e;
        if (pr.m1) { const double a = static_cast<double>(pr.m1[k]) * xl[k]; s += static_cast<double>(pr.a1) * a * a; }
        if (pr.m2) { const double a = static_cast<double>(pr.m2[k]) * xm[k]; s += static_cast<double>(pr.a2) * a * a; }
    }
    const double t = block_sum(s, sh);
    if (threadIdx.x == 0) partial[m * gridDim.x + blockIdx.x] = t;
}

// priors: partials sum a m^2 u s (pdot) and sum a (m s)^2 (psq) over both parts
__global__ void priordot_kernel(const float* __restrict__ ul, const float* __restrict__ um,
                                const float* __restrict__ sl, const float* __restrict__ sm, PriorArgs pr,
                                double* pdot, double* psq, int N)
{
    pdl_entry();
    __shared__ double sh[32];
    const int m = blockIdx.y;
    const size_t n2 = static_cast<size_t>(N) * N;
    double d = 0.0, q = 0.0;
    for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < n2;
         e += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const size_t k = m * n2 + e;
        if (pr.m1) {
            const double w = static_cast<double>(pr.a1) * pr.m1[k] * pr.m1[k];
            d += w * ul[k] * sl[k];
            q += w * sl[k] * sl[k];
        }
        if (pr.m2) {
            const double w = static_cast<double>(pr.a2) * pr.m2[k] * pr.m2[k];
            d += w * um[k] * sm[k];
            q += w * sm[k] * sm[k];
        }
    }
    const double td = block_sum(d, sh);
    if (threadIdx.x == 0) pdot[m * gridDim.x + blockIdx.x] = td;
    const double tq = block_sum(q, sh);
    if (threadIdx.x == 0) psq[m * gridDim.x + blockIdx.x] = tq;
}

// partial <a, b> over both parts
__global__ void dot2_kernel(const float* __restrict__ al, const float* __restrict__ am,
                            const float* __restrict__ bl, const float* __restrict__ bm, double* partial, int n2)
{
    pdl_entry();
    __shared__ double sh[32];
    const int m = blockIdx.y;
    const size_t base = static_cast<size_t>(m) * n2;
    double s = 0.0;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n2; e += gridDim.x * blockDim.x)
        s += static_cast<double>(al[base + e]) * bl[base + e] + static_cast<double>(am[base + e]) * bm[base + e];
    const double t = block_sum(s, sh);
    if (threadIdx.x == 0) partial[m * gridDim.x + blockIdx.x] = t;
}

// CG vector updates (skipped for members whose CG stopped)
//   phase 1: s += a p; z -= a q; partial ||z||^2
__global__ void cg_update1_kernel(float* sl, float* sm, float* zl, float* zm, const float* __restrict__ pl,
                                  const float* __restrict__ pm, const float* __restrict__ ql,
                                  const float* __restrict__ qm, const CGState* st, double* partial, int n2)
{
    pdl_entry();
    __shared__ double sh[32];
    const int m = blockIdx.y;
    const CGState c = st[m];
    const size_t base = static_cast<size_t>(m) * n2;
    double s = 0.0;
    if (!c.stop) {
        const float a = static_cast<float>(c.a);
        for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n2; e += gridDim.x * blockDim.x) {
            const size_t k = base + e;
            sl[k] = fmaf(a, pl[k], sl[k]);
            sm[k] = fmaf(a, pm[k], sm[k]);
            const float z1 = fmaf(-a, ql[k], zl[k]);
            const float z2 = fmaf(-a, qm[k], zm[k]);
            zl[k] = z1;
            zm[k] = z2;
            s += static_cast<double>(z1) * z1 + static_cast<double>(z2) * z2;
        }
    }
    const double t = block_sum(s, sh);
    if (threadIdx.x == 0) partial[m * gridDim.x + blockIdx.x] = t;
}

//   phase 2: p = z + bcg p
__global__ void cg_update2_kernel(const float* __restrict__ zl, const float* __restrict__ zm, float* pl,
                                  float* pm, const CGState* st, int n2)
{
    pdl_entry();
    const int m = blockIdx.y;
    const CGState c = st[m];
    if (c.stop) return;
    const float bc = static_cast<float>(c.bcg);
    const size_t base = static_cast<size_t>(m) * n2;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n2; e += gridDim.x * blockDim.x) {
        const size_t k = base + e;
        pl[k] = fmaf(bc, pl[k], zl[k]);
        pm[k] = fmaf(bc, pm[k], zm[k]);
    }
}

__device__ __forceinline__ double psum(const double* partial, int m, int nblk)
{
    double t = 0.0;
    for (int k = 0; k < nblk; ++k) t += partial[m * nblk + k];
    return t;
}

// ---- Prop. 1 safeguard: model values m_k(s) from per-member partial sums
// partial <a, b> and ||b||^2 of per-member vectors (sinograms)
__global__ void dotsq_kernel(const float* __restrict__ a, const float* __restrict__ b, double* pdot, double* psq,
                             int nper)
{
    pdl_entry();
    __shared__ double sh[32];
    const int m = blockIdx.y;
    double d = 0.0, q = 0.0;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < nper; e += gridDim.x * blockDim.x) {
        const size_t k = static_cast<size_t>(m) * nper + e;
        const double bv = b[k];
        d += static_cast<double>(a[k]) * bv;
        q += bv * bv;
    }
    const double td = block_sum(d, sh);
    if (threadIdx.x == 0) pdot[m * gridDim.x + blockIdx.x] = td;
    const double tq = block_sum(q, sh);
    if (threadIdx.x == 0) psq[m * gridDim.x + blockIdx.x] = tq;
}

// partial <L u, L s> and ||L s||^2 over both parts (lam, mu)
__global__ void lapdot_kernel(const float* __restrict__ ul, const float* __restrict__ um, const float* __restrict__ sl,
                              const float* __restrict__ sm, double* pdot, double* psq, int N)
{
    pdl_entry();
    __shared__ double sh[32];
    const int m = blockIdx.y;
    const size_t n2 = static_cast<size_t>(N) * N;
    double d = 0.0, q = 0.0;
    for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < n2;
         e += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int i = static_cast<int>(static_cast<unsigned>(e) % static_cast<unsigned>(N)),   // e < N^2 < 2^32
                  j = static_cast<int>(static_cast<unsigned>(e) / static_cast<unsigned>(N));
        const double a1 = lap_at(ul + m * n2, N, j, i), b1 = lap_at(sl + m * n2, N, j, i);
        const double a2 = lap_at(um + m * n2, N, j, i), b2 = lap_at(sm + m * n2, N, j, i);
        d += a1 * b1 + a2 * b2;
        q += b1 * b1 + b2 * b2;
    }
    const double td = block_sum(d, sh);
    if (threadIdx.x == 0) pdot[m * gridDim.x + blockIdx.x] = td;
    const double tq = block_sum(q, sh);
    if (threadIdx.x == 0) psq[m * gridDim.x + blockIdx.x] = tq;
}

// out = a - b over both parts (s~ = u~ - u)
__global__ void diff2_kernel(const float* __restrict__ al, const float* __restrict__ am, const float* __restrict__ bl,
                             const float* __restrict__ bm, float* ol, float* om, size_t n)
{
    pdl_entry();
    for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < n;
         e += static_cast<size_t>(gridDim.x) * blockDim.x) {
        ol[e] = al[e] - bl[e];
        om[e] = am[e] - bm[e];
    }
}

// one thread per member.  P: [0] 1/2||r||^2  [1] ||Lu||^2  [2] <r,Js~>  [3] ||Js~||^2  [4] <Lu,Ls~>
// [5] ||Ls~||^2  [6..9] the same four for s_k  [10] 1/2||F(u~)-y||^2  [11] ||Lu~||^2
__global__ void guard_scalar_kernel(const double* P, int nblk, int B, double alpha, double kappa,
                                    pget_safeguard_stats* out, int has_prior)
{
    pdl_entry();
    const int m = blockIdx.x * blockDim.x + threadIdx.x;
    if (m >= B) return;
    auto v = [&](int k) { return psum(P + static_cast<size_t>(k) * B * nblk, m, nblk); };
    // priors (the rows sqrt(a1) P1 lam, sqrt(a2) P2 mu of F~): 12 sum a (m u)^2, 13/14 <u, s~>_P and
    // ||s~||_P^2, 15/16 the same for s_k, 17 sum a (m u~)^2
    auto w = [&](int k) { return has_prior ? v(k) : 0.0; };
    pget_safeguard_stats S;
    S.f = v(0) + 0.5 * alpha * v(1) + 0.5 * w(12);
    S.m_cand = S.f + v(2) + alpha * v(4) + w(13) + 0.5 * (v(3) + alpha * v(5) + w(14));
    S.m_lm = S.f + v(6) + alpha * v(8) + w(15) + 0.5 * (v(7) + alpha * v(9) + w(16));
    S.pred_cand = S.f - S.m_cand;
    S.pred_lm = S.f - S.m_lm;
    S.f_cand = v(10) + 0.5 * alpha * v(11) + 0.5 * w(17);
    S.rho_cand = S.pred_cand != 0.0 ? (S.f - S.f_cand) / S.pred_cand : 0.0;
    S.kappa = kappa;
    S.accepted = (S.m_cand <= S.m_lm && S.pred_cand > 0.0 && S.rho_cand > kappa) ? 1 : 0;
    S.pad_ = 0;
    out[m] = S;
}

// u_next = accepted ? u~ : u + s  (per member)
__global__ void guard_select_kernel(const float* __restrict__ ul, const float* __restrict__ um,
                                    const float* __restrict__ sl, const float* __restrict__ sm, const float* cl,
                                    const float* cm, const pget_safeguard_stats* st, float* ol, float* om, int n2)
{
    pdl_entry();
    const int m = blockIdx.y;
    const bool acc = st[m].accepted != 0;
    const size_t base = static_cast<size_t>(m) * n2;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n2; e += gridDim.x * blockDim.x) {
        const size_t k = base + e;
        const float a = acc ? cl[k] : ul[k] + sl[k];
        const float b = acc ? cm[k] : um[k] + sm[k];
        ol[k] = a;
        om[k] = b;
    }
}

// ---- full LM solve
// box projection of the LM step: s <- clamp(u + s) - u (the step actually taken, reading R-N1)
__global__ void project_step_kernel(const float* __restrict__ ul, const float* __restrict__ um, float* sl, float* sm,
                                    size_t n, BoxK box)
{
    pdl_entry();
    for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < n;
         e += static_cast<size_t>(gridDim.x) * blockDim.x) {
        float a = ul[e] + sl[e], b = um[e] + sm[e];
        proj_k(a, b, box);
        sl[e] = a - ul[e];
        sm[e] = b - um[e];
    }
}

// accepted members take the trial point (evaluated by the LM wrap, clamped to the box when one is
// set); every member takes its next LM parameter
__global__ void lm_update_kernel(float* ul, float* um, const float* __restrict__ tl, const float* __restrict__ tm,
                                 const pget_gn_stats* stats, float* betav, int n2)
{
    pdl_entry();
    const int m = blockIdx.y;
    const bool acc = stats[m].accepted != 0;
    const size_t base = static_cast<size_t>(m) * n2;
    if (acc)
        for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n2; e += gridDim.x * blockDim.x) {
            ul[base + e] = tl[base + e];
            um[base + e] = tm[base + e];
        }
    if (blockIdx.x == 0 && threadIdx.x == 0) betav[m] = static_cast<float>(stats[m].beta_next);
}

__global__ void clamp_kernel(float* ul, float* um, size_t n, BoxK box)
{
    pdl_entry();
    for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < n;
         e += static_cast<size_t>(gridDim.x) * blockDim.x) {
        float a = ul[e], b = um[e];
        proj_k(a, b, box);
        ul[e] = a;
        um[e] = b;
    }
}

__global__ void fill_kernel(float* x, float v, int n)
{
    pdl_entry();
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e < n) x[e] = v;
}

// Scalar steps of the LM iteration (one thread per member).
__global__ void scalar_kernel(int op, int k, const double* p0, const double* p1, const double* p2, int nblk,
                              CGState* st, pget_gn_stats* stats, int B, double alpha, double beta_h,
                              const float* betav, const double* pp)
{
    pdl_entry();
    const int m = blockIdx.x * blockDim.x + threadIdx.x;
    if (m >= B) return;
    const double beta = betav ? static_cast<double>(betav[m]) : beta_h;   // per-member LM parameter
    CGState& c = st[m];
    pget_gn_stats& S = stats[m];
    if (op == SC_INIT) {             // p0: 1/2||r||^2, p1: ||Lu||^2, p2: ||b||^2
        const double mis = psum(p0, m, nblk), lq = psum(p1, m, nblk), bb = psum(p2, m, nblk);
        S.misfit = mis;
        S.reg = 0.5 * alpha * lq;
        if (pp) S.reg += 0.5 * psum(pp, m, nblk);   // priors: pp = sum a (m x)^2 of u
        S.f = mis + S.reg;
        S.grad_norm = sqrt(bb);
        S.cg_res[0] = sqrt(bb);
        S.n_cg_done = 0;
        S.breakdown = 0;
        S.beta_min = 0.0;
        S.pred = S.f_trial = S.rho = 0.0;
        S.beta_next = beta;
        S.accepted = 0;
        c.zeta = bb;
        c.stop = 0;
        c.a = 0.0;
        c.bcg = 0.0;
        if (bb == 0.0) { c.stop = 1; S.breakdown = 1; }
    } else if (op == SC_GAMMA) {     // p0: <p, Hp>
        if (c.stop) return;
        const double gam = psum(p0, m, nblk);
        if (k == 0) S.beta_min = 1e-3 * gam / c.zeta;
        if (!(gam > 0.0)) { c.stop = 1; S.breakdown = 2; return; }
        c.a = c.zeta / gam;
    } else if (op == SC_ZETA) {      // p0: ||z||^2
        if (c.stop) return;
        const double z2 = psum(p0, m, nblk);
        c.bcg = z2 / c.zeta;
        c.zeta = z2;
        S.cg_res[k + 1] = sqrt(z2);
        S.n_cg_done = k + 1;
        if (z2 == 0.0) { c.stop = 1; S.breakdown = 1; }
    } else if (op == SC_PRED) {      // p0: ||Js||^2, p1: ||Ls||^2, p2: <b,s>
        const double js2 = psum(p0, m, nblk), ls2 = psum(p1, m, nblk), bs = psum(p2, m, nblk);
        S.js2 = js2;
        S.als2 = alpha * ls2;
        if (pp) S.als2 += psum(pp, m, nblk);   // priors of s
        S.bs = bs;
        S.pred = bs - 0.5 * (js2 + S.als2);
    } else if (op == SC_TRIAL) {     // p0: 1/2||r(u+s)||^2, p1: ||L(u+s)||^2
        double f1 = psum(p0, m, nblk) + 0.5 * alpha * psum(p1, m, nblk);
        if (pp) f1 += 0.5 * psum(pp, m, nblk);   // priors of u + s
        S.f_trial = f1;
        S.rho = (S.f - f1) / S.pred;
        S.accepted = S.pred > 0.0 && S.rho > 0.1;   // reading R-accept
        double bn = beta;
        if (!S.accepted) bn = (10.0 * beta > S.beta_min) ? 10.0 * beta : S.beta_min;
        else if (S.rho > 0.75) bn = 0.2 * beta;
        S.beta_next = bn;
    }
}


// ---- SGP inner solver (O11): gradient projection on the box with Barzilai-Borwein
// lengths and an exact line search, from s = 0; g = H s - b.
__global__ void sgp_init_kernel(const float* __restrict__ bl, const float* __restrict__ bm, float* gl, float* gm,
                                CGState* st, int n2, int B)
{
    pdl_entry();
    const size_t n = static_cast<size_t>(B) * n2;
    for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < n;
         e += static_cast<size_t>(gridDim.x) * blockDim.x) {
        gl[e] = -bl[e];
        gm[e] = -bm[e];
    }
    if (blockIdx.x == 0)
        for (int m = threadIdx.x; m < B; m += blockDim.x) st[m] = CGState{0.0, 1.0, 0.0, 0, 0};
}

// d = P_box(u + s - a g) - u - s; partials <g, d>, <d, d> (zero for a stopped member)
__global__ void sgp_dir_kernel(const float* __restrict__ ul, const float* __restrict__ um,
                               const float* __restrict__ sl, const float* __restrict__ sm,
                               const float* __restrict__ gl, const float* __restrict__ gm, const CGState* st,
                               BoxK box, float* dl, float* dm, double* pgd, double* pdd, int n2)
{
    pdl_entry();
    __shared__ double sh[32];
    const int m = blockIdx.y;
    const size_t base = static_cast<size_t>(m) * n2;
    const bool run = !st[m].stop;
    const float a = static_cast<float>(st[m].a);
    double gd = 0.0, dd = 0.0;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n2; e += gridDim.x * blockDim.x) {
        const size_t k = base + e;
        float d1 = 0.f, d2 = 0.f;
        if (run) {
            const float x1 = ul[k] + sl[k], x2 = um[k] + sm[k];
            float y1 = fmaf(-a, gl[k], x1), y2 = fmaf(-a, gm[k], x2);
            proj_k(y1, y2, box);
            d1 = y1 - x1;
            d2 = y2 - x2;
            gd += static_cast<double>(gl[k]) * d1 + static_cast<double>(gm[k]) * d2;
            dd += static_cast<double>(d1) * d1 + static_cast<double>(d2) * d2;
        }
        dl[k] = d1;
        dm[k] = d2;
    }
    const double t1 = block_sum(gd, sh);
    if (threadIdx.x == 0) pgd[m * gridDim.x + blockIdx.x] = t1;
    const double t2 = block_sum(dd, sh);
    if (threadIdx.x == 0) pdd[m * gridDim.x + blockIdx.x] = t2;
}

// per member: stop when <g, d> >= 0; else lam = min(1, -<g,d>/<d,Hd>), the next BB length (BB1 after
// even steps, BB2 after odd ones, clamped to [1e-10, 1e10]); final_: only ||d|| of the last direction
__global__ void sgp_scalar_kernel(int k, int final_, const double* pgd, const double* pdd, const double* pdhd,
                                  const double* pqq, int nblk, CGState* st, pget_gn_stats* stats, int B)
{
    pdl_entry();
    const int m = blockIdx.x * blockDim.x + threadIdx.x;
    if (m >= B) return;
    CGState& c = st[m];
    pget_gn_stats& S = stats[m];
    if (c.stop) return;
    const double gd = psum(pgd, m, nblk), dd = psum(pdd, m, nblk);
    S.cg_res[k] = sqrt(dd);
    if (final_) return;
    if (!(gd < 0.0)) {
        c.stop = 1;
        S.breakdown = 1;
        S.n_cg_done = k;
        return;
    }
    const double dhd = psum(pdhd, m, nblk), qq = psum(pqq, m, nblk);
    if (k == 0) S.beta_min = 1e-3 * dhd / dd;
    const double lam = dhd > 0.0 ? fmin(1.0, -gd / dhd) : 1.0;
    c.bcg = lam;
    const double sy = lam * lam * dhd, ss = lam * lam * dd, yy = lam * lam * qq;
    double an = (k % 2 == 0) ? (sy > 0.0 ? ss / sy : 1e10) : (yy > 0.0 ? sy / yy : 1e10);
    c.a = an < 1e-10 ? 1e-10 : (an > 1e10 ? 1e10 : an);
    S.n_cg_done = k + 1;
}

// s += lam d, g += lam H d (members not stopped)
__global__ void sgp_update_kernel(float* sl, float* sm, float* gl, float* gm, const float* __restrict__ dl,
                                  const float* __restrict__ dm, const float* __restrict__ ql,
                                  const float* __restrict__ qm, const CGState* st, int n2)
{
    pdl_entry();
    const int m = blockIdx.y;
    if (st[m].stop) return;
    const float lam = static_cast<float>(st[m].bcg);
    const size_t base = static_cast<size_t>(m) * n2;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n2; e += gridDim.x * blockDim.x) {
        const size_t k = base + e;
        sl[k] = fmaf(lam, dl[k], sl[k]);
        sm[k] = fmaf(lam, dm[k], sm[k]);
        gl[k] = fmaf(lam, ql[k], gl[k]);
        gm[k] = fmaf(lam, qm[k], gm[k]);
    }
}

// One CG step after the GN projector, fused into a single cooperative launch (grid-wide syncs):
//   q = H p  (the G fp64 slot partials + alpha L^T L p + beta p),   gamma = <p, q>,
//   a = zeta / gamma,  s += a p,  z -= a q,  zeta' = <z, z>,  p = z + (zeta' / zeta) p,
// with the same fixed-order fp64 block partials (nblk per member) and the same stop rules and
// statistics as finish / scalar(SC_GAMMA) / cg_update1 / scalar(SC_ZETA) / cg_update2.
// Work unit (member m, block-in-member j) -> elements e = j * blockDim + tid (+ nblk * blockDim).
__global__ void cg_fused_kernel(const double2* __restrict__ part, int G, float alpha, float beta_h,
                                const float* betav, float* sl, float* sm, float* zl, float* zm, float* pl,
                                float* pm, float* ql, float* qm, double* pg, double* pz, CGState* st,
                                pget_gn_stats* stats, int k, int N, int B, int nblk, float4* img4n, float4* img4t,
                                int P, PriorArgs pr)
{
    pdl_entry();
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    __shared__ double sh[32];
    const size_t n2 = static_cast<size_t>(N) * N;
    const int units = B * nblk;
    const size_t stride = static_cast<size_t>(nblk) * blockDim.x;
    // CG state double-buffered by step parity: this launch reads st_in and writes st_out only, so no
    // block can see a member's state change while another block of that member still reads it
    CGState* st_in = st + static_cast<size_t>(k & 1) * B;
    CGState* st_out = st + static_cast<size_t>((k + 1) & 1) * B;
    st = st_in;
    // phase 1: q = H p, <p, q> partials
    for (int mj = blockIdx.x; mj < units; mj += gridDim.x) {
        const int m = mj / nblk, j = mj - m * nblk;
        const size_t base = static_cast<size_t>(m) * n2;
        double dsum = 0.0;
        const float beta = betav ? betav[m] : beta_h;
        if (!st[m].stop) {
            for (size_t e = static_cast<size_t>(j) * blockDim.x + threadIdx.x; e < n2; e += stride) {
                const int i = static_cast<int>(static_cast<unsigned>(e) % static_cast<unsigned>(N)),   // e < N^2 < 2^32
                          jj = static_cast<int>(static_cast<unsigned>(e) / static_cast<unsigned>(N));
                double2 a = part[base + e];
                // the G partials in order; eight loads issued before their additions (latency-bound)
                for (int g0 = 1; g0 < G; g0 += 8) {
                    double2 b[8];
#pragma unroll
                    for (int t = 0; t < 8; ++t)
                        b[t] = g0 + t < G ? part[static_cast<size_t>(g0 + t) * B * n2 + base + e] : make_double2(0.0, 0.0);
#pragma unroll
                    for (int t = 0; t < 8; ++t) {
                        if (g0 + t < G) {
                            a.x += b[t].x;
                            a.y += b[t].y;
                        }
                    }
                }
                const float* xl = pl + base;
                const float* xm = pm + base;
                float ol = static_cast<float>(a.x) + alpha * lap2_at(xl, N, jj, i) + beta * xl[e];
                float om = static_cast<float>(a.y) + alpha * lap2_at(xm, N, jj, i) + beta * xm[e];
                prior_op(pr, base + e, xl[e], xm[e], ol, om);
                ql[base + e] = ol;
                qm[base + e] = om;
                dsum += static_cast<double>(ol) * xl[e] + static_cast<double>(om) * xm[e];
            }
        }
        const double t = block_sum(dsum, sh);
        if (threadIdx.x == 0) pg[mj] = t;
    }
    grid.sync();
    // phase 2: a = zeta / <p, q>; s += a p; z -= a q; ||z||^2 partials
    for (int mj = blockIdx.x; mj < units; mj += gridDim.x) {
        const int m = mj / nblk, j = mj - m * nblk;
        const size_t base = static_cast<size_t>(m) * n2;
        const CGState c = st[m];
        double gam = 0.0;
        for (int q = 0; q < nblk; ++q) gam += pg[m * nblk + q];
        double zs = 0.0;
        if (!c.stop && gam > 0.0) {
            const float a = static_cast<float>(c.zeta / gam);
            for (size_t e = static_cast<size_t>(j) * blockDim.x + threadIdx.x; e < n2; e += stride) {
                const size_t q = base + e;
                sl[q] = fmaf(a, pl[q], sl[q]);
                sm[q] = fmaf(a, pm[q], sm[q]);
                const float z1 = fmaf(-a, ql[q], zl[q]);
                const float z2 = fmaf(-a, qm[q], zm[q]);
                zl[q] = z1;
                zm[q] = z2;
                zs += static_cast<double>(z1) * z1 + static_cast<double>(z2) * z2;
            }
        }
        const double t = block_sum(zs, sh);
        if (threadIdx.x == 0) pz[mj] = t;
    }
    grid.sync();
    // phase 3: p = z + (zeta' / zeta) p; state and statistics (unit (m, 0), thread 0)
    for (int mj = blockIdx.x; mj < units; mj += gridDim.x) {
        const int m = mj / nblk, j = mj - m * nblk;
        const size_t base = static_cast<size_t>(m) * n2;
        const CGState c = st[m];
        double gam = 0.0, z2 = 0.0;
        for (int q = 0; q < nblk; ++q) {
            gam += pg[m * nblk + q];
            z2 += pz[m * nblk + q];
        }
        const bool run = !c.stop && gam > 0.0;
        const double bcg = run ? z2 / c.zeta : 0.0;
        if (run && z2 != 0.0) {
            const float bc = static_cast<float>(bcg);
            for (size_t e = static_cast<size_t>(j) * blockDim.x + threadIdx.x; e < n2; e += stride) {
                const size_t q = base + e;
                const float p1 = fmaf(bc, pl[q], zl[q]), p2 = fmaf(bc, pm[q], zm[q]);
                pl[q] = p1;
                pm[q] = p2;
                if (img4n) {   // the next GN product's packed (dlam, dmu) halves, both orientations (pack4)
                    const int i = static_cast<int>(static_cast<unsigned>(e) % static_cast<unsigned>(N)) + kHalo,
                              jj = static_cast<int>(static_cast<unsigned>(e) / static_cast<unsigned>(N)) + kHalo;
                    reinterpret_cast<float2*>(img4n + (static_cast<size_t>(m) * P + jj) * P + i)[1] = make_float2(p1, p2);
                    reinterpret_cast<float2*>(img4t + (static_cast<size_t>(m) * P + i) * P + jj)[1] = make_float2(p1, p2);
                }
            }
        }
        if (j == 0 && threadIdx.x == 0) st_out[m] = c;   // carried over (stopped members keep theirs)
        if (j == 0 && threadIdx.x == 0 && !c.stop) {
            CGState& w = st_out[m];
            pget_gn_stats& S = stats[m];
            if (k == 0) S.beta_min = 1e-3 * gam / c.zeta;
            if (!(gam > 0.0)) {
                w.stop = 1;
                S.breakdown = 2;
            } else {
                w.a = c.zeta / gam;
                w.bcg = bcg;
                w.zeta = z2;
                S.cg_res[k + 1] = sqrt(z2);
                S.n_cg_done = k + 1;
                if (z2 == 0.0) { w.stop = 1; S.breakdown = 1; }
            }
        }
    }
}

}  // namespace pget

namespace pget {
bool pdl_enabled()
{
    static const bool on = [] {
        const char* ev = std::getenv("PGET_PDL");
        return !(ev && std::atoi(ev) == 0);
    }();
    return on;
}

// flag = 1 if any element is NaN or +-inf (pget_check_finite)
__global__ void finite_scan_kernel(const float* __restrict__ x, size_t n, int32_t* flag)
{
    pdl_entry();
    bool bad = false;
    for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < n;
         e += static_cast<size_t>(gridDim.x) * blockDim.x)
        bad |= !isfinite(x[e]);
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicExch(flag, 1);
}
}  // namespace pget
