// kernels.cu -- sm_100a kernels of the PGET hot path.
//
// Ray-driven projector: one CTA per (batch member,
// angle-bank); one lane per ray, 32 adjacent sub-rays per warp; the padded
// lambda/mu image is staged into shared memory in bands of rows, visited in
// detector-first order so that every ray's attenuation suffix sum
//     A_i = Delta (mu_i / 2 + sum_{k>i} mu_k)          (B mu; reading Q8)
// is a per-lane recurrence in registers carried across bands.  One ex2 per sample.
//   MODE_FWD : y      = sum_j w_j Delta sum_i lam_i E_i                 (eq:fwd_model)
//   MODE_JVP : + dy   = sum_j w_j Delta sum_i (dlam_i - lam_i dA_i) E_i  (eq:frechet)
//   MODE_VJP : sweep A gives G = sum_i lam_i E_i per ray; sweep B scatters
//              a_lam(i) = w_r Delta E_i and a_mu(i) = -w_r Delta^2 (G - Q_i - lam_i E_i / 2)
//              (Q_i = sum_{k>i} lam_k E_k) with the transposed bilinear weights into a
//              shared-memory band accumulator (no global atomics in the sample loop),
//              flushed once per band.
//   MODE_GN  : sweep A = fused JVP of p; per-detector w = sum_j w_j (Jp)_ray in shared
//              memory; sweep B = VJP with those weights -> J^T J p   (eq:LMA-step)
// Sample positions are 32.32 fixed point (exact integer stepping); the bilinear
// fraction is taken from the low word (23 bits, rounded), see internal.h RayP.
#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.h"
#include "kernels.cuh"

namespace pget {

__device__ __forceinline__ float frac23(int64_t x)
{
    return __uint_as_float((static_cast<uint32_t>(x) >> 9) | 0x3f800000u) - 1.0f;
}

__device__ __forceinline__ int hi32(int64_t x) { return static_cast<int>(x >> 32); }

__device__ __forceinline__ float ex2(float x)
{
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// bilinear lerp of a (lam, mu) pair: a=(j0,i0) b=(j0,i0+1) c=(j0+1,i0) d=(j0+1,i0+1)
__device__ __forceinline__ float2 bilerp2(float2 a, float2 b, float2 c, float2 d, float fu, float fv)
{
    const float2 m1 = make_float2(-1.f, -1.f);
    const float2 u2 = make_float2(fu, fu), v2 = make_float2(fv, fv);
    const float2 top = __ffma2_rn(u2, __ffma2_rn(a, m1, b), a);
    const float2 bot = __ffma2_rn(u2, __ffma2_rn(c, m1, d), c);
    return __ffma2_rn(v2, __ffma2_rn(top, m1, bot), top);
}

__device__ __forceinline__ float2 lo2(float4 x) { return make_float2(x.x, x.y); }
__device__ __forceinline__ float2 hi2(float4 x) { return make_float2(x.z, x.w); }

// Cooperative copy of `nfloat` floats (multiple of 4, 16-B aligned) global -> shared.
__device__ __forceinline__ void stage(float* __restrict__ dst, const float* __restrict__ src, int nfloat)
{
    const float4* s4 = reinterpret_cast<const float4*>(src);
    float4* d4 = reinterpret_cast<float4*>(dst);
    const int n4 = nfloat >> 2;
    for (int k = threadIdx.x; k < n4; k += blockDim.x) d4[k] = __ldg(s4 + k);
}

__device__ __forceinline__ void zero_smem(float* dst, int nfloat)
{
    float4* d4 = reinterpret_cast<float4*>(dst);
    const int n4 = nfloat >> 2;
    for (int k = threadIdx.x; k < n4; k += blockDim.x) d4[k] = make_float4(0.f, 0.f, 0.f, 0.f);
}

// Band k of nb: j0 rows [r0, r1), staged rows [r0, r1] (the +1 row for the bilinear j0+1).
__device__ __forceinline__ void band_rows(int k, int Rb, int Hp, int& r0, int& r1)
{
    r0 = k * Rb;
    r1 = min(r0 + Rb, Hp - 1);
}

// ------------------------------------------------------------------------------------------
// Sweep A: forward (+ fused JVP) recurrence over all bands.
//   NF = 2: staged (lam, mu); NF = 4: staged (lam, mu, dlam, dmu).
// State per ray k (registers): i[k] next sample, S[k] = -Delta log2e sum_{k>i} mu,
// g[k] = sum lam E, and for NF = 4: dS[k] = Delta sum_{k>i} dmu, dg[k].
template <int NF, int MAXR>
__device__ __forceinline__ void sweep_a(const ProjArgs& A, const float* __restrict__ img, float* sbuf,
                                        const RayP* __restrict__ rays, int dir, int nvalid,
                                        float (&g)[MAXR], float (&dg)[MAXR])
{
    const int T = blockDim.x;
    const int Wp = A.Wp, Hp = A.Hp, Rb = A.RbA;
    const int nb = (Hp - 1 + Rb - 1) / Rb;
    int icur[MAXR];
    float S[MAXR], dS[MAXR];
#pragma unroll
    for (int k = 0; k < MAXR; ++k) {
        const int r = threadIdx.x + k * T;
        icur[k] = (r < nvalid) ? rays[r].ihi : -1;
        S[k] = 0.f; g[k] = 0.f; dS[k] = 0.f; dg[k] = 0.f;
    }
    const float cf = A.cf, ch = A.ch, dl = A.delta, dlh = 0.5f * A.delta;
    for (int kb = 0; kb < nb; ++kb) {
        const int band = dir > 0 ? nb - 1 - kb : kb;
        int r0, r1;
        band_rows(band, Rb, Hp, r0, r1);
        __syncthreads();   // previous band fully consumed
        stage(sbuf, img + static_cast<size_t>(r0) * Wp * NF, (r1 - r0 + 1) * Wp * NF);
        __syncthreads();
#pragma unroll
        for (int k = 0; k < MAXR; ++k) {
            const int r = threadIdx.x + k * T;
            if (r >= nvalid) continue;
            int i = icur[k];
            const RayP rp = rays[r];
            if (i < rp.ilo) continue;
            int64_t u = rp.U0 + static_cast<int64_t>(i) * rp.dU;
            int64_t v = rp.V0 + static_cast<int64_t>(i) * rp.dV;
            float s = S[k], gg = g[k], ds = dS[k], dgg = dg[k];
            while (i >= rp.ilo) {
                const int iv = hi32(v);
                if (iv < r0 || iv >= r1) break;
                const int iu = hi32(u);
                const float fu = frac23(u), fv = frac23(v);
                const int o = (iv - r0) * Wp + iu;
                float lam, mu, dlam = 0.f, dmu = 0.f;
                if (NF == 2) {
                    const float2* p = reinterpret_cast<const float2*>(sbuf) + o;
                    const float2 x = bilerp2(p[0], p[1], p[Wp], p[Wp + 1], fu, fv);
                    lam = x.x; mu = x.y;
                } else {
                    const float4* p = reinterpret_cast<const float4*>(sbuf) + o;
                    const float4 a = p[0], b = p[1], c = p[Wp], d = p[Wp + 1];
                    const float2 x = bilerp2(lo2(a), lo2(b), lo2(c), lo2(d), fu, fv);
                    const float2 y = bilerp2(hi2(a), hi2(b), hi2(c), hi2(d), fu, fv);
                    lam = x.x; mu = x.y; dlam = y.x; dmu = y.y;
                }
                const float E = ex2(fmaf(mu, ch, s));     // exp(-Delta (mu_i/2 + sum_{k>i} mu_k))
                gg = fmaf(lam, E, gg);
                s = fmaf(mu, cf, s);
                if (NF == 4) {
                    const float dA = fmaf(dmu, dlh, ds);    // Delta (dmu_i/2 + sum_{k>i} dmu_k)
                    dgg = fmaf(fmaf(-lam, dA, dlam), E, dgg);
                    ds = fmaf(dmu, dl, ds);
                }
                --i;
                u -= rp.dU;
                v -= rp.dV;
            }
            icur[k] = i; S[k] = s; g[k] = gg; dS[k] = ds; dg[k] = dgg;
        }
    }
}

__device__ __forceinline__ void sadd(float* p, float v) { atomicAdd(p, v); }

// Sweep B: adjoint scatter.  kl[k] = w_r Delta, km[k] = -w_r Delta^2, G[k] = sum lam E (sweep A).
template <int MAXR>
__device__ __forceinline__ void sweep_b(const ProjArgs& A, const float* __restrict__ img, float* sbuf,
                                        float* sacc, float2* __restrict__ gacc,
                                        const RayP* __restrict__ rays, int dir, int nvalid,
                                        const float (&kl)[MAXR], const float (&km)[MAXR],
                                        const float (&G)[MAXR])
{
    const int T = blockDim.x;
    const int Wp = A.Wp, Hp = A.Hp, Rb = A.RbB;
    const int nb = (Hp - 1 + Rb - 1) / Rb;
    int icur[MAXR];
    float S[MAXR], Q[MAXR];
#pragma unroll
    for (int k = 0; k < MAXR; ++k) {
        const int r = threadIdx.x + k * T;
        icur[k] = (r < nvalid && kl[k] != 0.f) ? rays[r].ihi : -1;
        S[k] = 0.f; Q[k] = 0.f;
    }
    const float cf = A.cf, ch = A.ch;
    for (int kb = 0; kb < nb; ++kb) {
        const int band = dir > 0 ? nb - 1 - kb : kb;
        int r0, r1;
        band_rows(band, Rb, Hp, r0, r1);
        const int nrow = r1 - r0 + 1;
        __syncthreads();
        stage(sbuf, img + static_cast<size_t>(r0) * Wp * 2, nrow * Wp * 2);
        zero_smem(sacc, nrow * Wp * 2);
        __syncthreads();
#pragma unroll
        for (int k = 0; k < MAXR; ++k) {
            const int r = threadIdx.x + k * T;
            if (r >= nvalid) continue;
            int i = icur[k];
            const RayP rp = rays[r];
            if (i < rp.ilo) continue;
            int64_t u = rp.U0 + static_cast<int64_t>(i) * rp.dU;
            int64_t v = rp.V0 + static_cast<int64_t>(i) * rp.dV;
            float s = S[k], q = Q[k];
            const float kll = kl[k], kmm = km[k], GG = G[k];
            while (i >= rp.ilo) {
                const int iv = hi32(v);
                if (iv < r0 || iv >= r1) break;
                const int iu = hi32(u);
                const float fu = frac23(u), fv = frac23(v);
                const int o = (iv - r0) * Wp + iu;
                const float2* p = reinterpret_cast<const float2*>(sbuf) + o;
                const float2 x = bilerp2(p[0], p[1], p[Wp], p[Wp + 1], fu, fv);
                const float E = ex2(fmaf(x.y, ch, s));
                const float le = x.x * E;
                const float al = kll * E;
                const float am = kmm * (GG - q - 0.5f * le);
                q += le;
                s = fmaf(x.y, cf, s);
                // transposed bilinear weights
                const float2 av = make_float2(al, am);
                const float2 tv = __fmul2_rn(av, make_float2(fv, fv));       // row j0+1
                const float2 bv = __ffma2_rn(tv, make_float2(-1.f, -1.f), av); // row j0
                const float2 c11 = __fmul2_rn(tv, make_float2(fu, fu));
                const float2 c10 = __ffma2_rn(c11, make_float2(-1.f, -1.f), tv);
                const float2 c01 = __fmul2_rn(bv, make_float2(fu, fu));
                const float2 c00 = __ffma2_rn(c01, make_float2(-1.f, -1.f), bv);
                float* a0 = sacc + 2 * o;
                sadd(a0 + 0, c00.x); sadd(a0 + 1, c00.y);
                sadd(a0 + 2, c01.x); sadd(a0 + 3, c01.y);
                float* a1 = a0 + 2 * Wp;
                sadd(a1 + 0, c10.x); sadd(a1 + 1, c10.y);
                sadd(a1 + 2, c11.x); sadd(a1 + 3, c11.y);
                --i;
                u -= rp.dU;
                v -= rp.dV;
            }
            icur[k] = i; S[k] = s; Q[k] = q;
        }
        __syncthreads();
        // flush the band accumulator (rows r0..r1) into the member's global accumulator
        const float2* sa2 = reinterpret_cast<const float2*>(sacc);
        float2* gdst = gacc + static_cast<size_t>(r0) * Wp;
        for (int e = threadIdx.x; e < nrow * Wp; e += blockDim.x) {
            const float2 val = sa2[e];
            if (val.x != 0.f || val.y != 0.f) atomicAdd(gdst + e, val);
        }
    }
}

template <int MODE, int MAXR>
__global__ void __launch_bounds__(1024, 1) proj_kernel(ProjArgs A)
{
    extern __shared__ __align__(16) float smem[];
    const int ab = blockIdx.x % A.n_ab;
    const int m = blockIdx.x / A.n_ab;
    const int T = blockDim.x;
    const int dir = A.abdir[ab];
    const RayP* rays = A.rays + static_cast<size_t>(ab) * A.R;
    const size_t imgsz = static_cast<size_t>(A.Hp) * A.Wp;
    float* sbuf = smem;
    float* rout = smem + A.rout_off;   // 2 * R_pad floats

    float g[MAXR], dg[MAXR];
    if (MODE == MODE_FWD || MODE == MODE_VJP)
        sweep_a<2, MAXR>(A, reinterpret_cast<const float*>(A.img2 + m * imgsz), sbuf, rays, dir, A.R, g, dg);
    else
        sweep_a<4, MAXR>(A, reinterpret_cast<const float*>(A.img4 + m * imgsz), sbuf, rays, dir, A.R, g, dg);

    const int J = A.J;
    if (MODE == MODE_FWD || MODE == MODE_JVP) {
#pragma unroll
        for (int k = 0; k < MAXR; ++k) {
            const int r = threadIdx.x + k * T;
            if (r < A.R) {
                rout[r] = A.delta * g[k];
                if (MODE == MODE_JVP) rout[A.R_pad + r] = A.delta * dg[k];
            }
        }
        __syncthreads();
        const size_t obase = (static_cast<size_t>(m) * A.n_ab + ab) * A.n_det;
        for (int d = threadIdx.x; d < A.n_det; d += T) {
            float acc = 0.f, dacc = 0.f;
            for (int j = 0; j < J; ++j) {
                const float wj = A.w[j];
                acc = fmaf(wj, rout[d * J + j], acc);
                if (MODE == MODE_JVP) dacc = fmaf(wj, rout[A.R_pad + d * J + j], dacc);
            }
            if (A.y) A.y[obase + d] = acc;
            if (MODE == MODE_JVP) A.dy[obase + d] = dacc;
        }
        return;
    }

    // adjoint weights per ray
    float kl[MAXR], km[MAXR];
    if (MODE == MODE_GN) {
#pragma unroll
        for (int k = 0; k < MAXR; ++k) {
            const int r = threadIdx.x + k * T;
            if (r < A.R) rout[r] = A.delta * dg[k];     // (J p)_ray
        }
        __syncthreads();
    }
    const size_t wbase = (static_cast<size_t>(m) * A.n_ab + ab) * A.n_det;
#pragma unroll
    for (int k = 0; k < MAXR; ++k) {
        const int r = threadIdx.x + k * T;
        kl[k] = 0.f; km[k] = 0.f;
        if (r < A.R) {
            const int d = r / J, j = r - d * J;
            float wd;
            if (MODE == MODE_GN) {
                wd = 0.f;
                for (int jj = 0; jj < J; ++jj) wd = fmaf(A.w[jj], rout[d * J + jj], wd);
            } else {
                wd = A.win[wbase + d];
            }
            const float wr = A.w[j] * wd;
            kl[k] = wr * A.delta;
            km[k] = -wr * A.delta * A.delta;
        }
    }
    float* sacc = smem + A.acc_off;
    sweep_b<MAXR>(A, reinterpret_cast<const float*>(A.img2 + m * imgsz), sbuf, sacc, A.acc + m * imgsz, rays,
                  dir, A.R, kl, km, g);
}

// ------------------------------------------------------------------------------------------
// image packing: padded interleaved images with a zero halo of kHalo pixels
__global__ void pack2_kernel(const float* __restrict__ lam, const float* __restrict__ mu,
                             const float* __restrict__ slam, const float* __restrict__ smu, float2* out,
                             float* ut_lam, float* ut_mu, int N, int Hp, int Wp, int B)
{
    const size_t total = static_cast<size_t>(B) * Hp * Wp;
    for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int ip = static_cast<int>(e % Wp);
        const int jp = static_cast<int>((e / Wp) % Hp);
        const size_t m = e / (static_cast<size_t>(Wp) * Hp);
        const int i = ip - kHalo, j = jp - kHalo;
        float2 val = make_float2(0.f, 0.f);
        if (i >= 0 && i < N && j >= 0 && j < N) {
            const size_t src = (m * N + j) * N + i;
            val = make_float2(lam[src], mu[src]);
            if (slam) {
                val.x += slam[src];
                val.y += smu[src];
                ut_lam[src] = val.x;
                ut_mu[src] = val.y;
            }
        }
        out[e] = val;
    }
}

__global__ void pack4_kernel(const float* __restrict__ lam, const float* __restrict__ mu,
                             const float* __restrict__ dl, const float* __restrict__ dm, float4* out, int N,
                             int Hp, int Wp, int B)
{
    const size_t total = static_cast<size_t>(B) * Hp * Wp;
    for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int ip = static_cast<int>(e % Wp);
        const int jp = static_cast<int>((e / Wp) % Hp);
        const size_t m = e / (static_cast<size_t>(Wp) * Hp);
        const int i = ip - kHalo, j = jp - kHalo;
        float4 val = make_float4(0.f, 0.f, 0.f, 0.f);
        if (i >= 0 && i < N && j >= 0 && j < N) {
            const size_t src = (m * N + j) * N + i;
            val = make_float4(lam[src], mu[src], dl[src], dm[src]);
        }
        out[e] = val;
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

__device__ __forceinline__ float lap2_at(const float* __restrict__ x, int N, int j, int i)
{
    return 4.f * lap_at(x, N, j, i) - lap_at(x, N, j, i - 1) - lap_at(x, N, j, i + 1) -
           lap_at(x, N, j - 1, i) - lap_at(x, N, j + 1, i);
}

// out = sign * (acc_interior + alpha L^T L x + beta x) over both parts; partial <dotv, out>.
//   grad mode (VJP out):  alpha = beta = 0, sign = 1, dotv = NULL
//   b = -(J^T r + alpha L^T L u):  sign = -1, x = u, beta = 0, dotv = out (||b||^2), also copies
//   q = J^T J p + alpha L^T L p + beta p:  sign = 1, x = p, dotv = p
__global__ void finish_kernel(const float2* __restrict__ acc, const float* __restrict__ xl,
                              const float* __restrict__ xm, float alpha, float beta, float sign,
                              float* outl, float* outm, const float* __restrict__ dotl,
                              const float* __restrict__ dotm, double* partial, float* copy1l, float* copy1m,
                              float* copy2l, float* copy2m, float* zerol, float* zerom, int N, int Hp, int Wp)
{
    __shared__ double sh[32];
    const int m = blockIdx.y;
    const size_t n2 = static_cast<size_t>(N) * N;
    const size_t base = m * n2;
    double dsum = 0.0;
    for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < n2;
         e += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int i = static_cast<int>(e % N), j = static_cast<int>(e / N);
        const float2 a = acc[(static_cast<size_t>(m) * Hp + j + kHalo) * Wp + i + kHalo];
        float ol = a.x, om = a.y;
        if (xl) {
            const float* pl = xl + base;
            const float* pm = xm + base;
            ol += alpha * lap2_at(pl, N, j, i) + beta * pl[e];
            om += alpha * lap2_at(pm, N, j, i) + beta * pm[e];
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
    __shared__ double sh[32];
    const int m = blockIdx.y;
    const size_t n2 = static_cast<size_t>(N) * N;
    double s = 0.0;
    for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < n2;
         e += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int i = static_cast<int>(e % N), j = static_cast<int>(e / N);
        const double a = lap_at(xl + m * n2, N, j, i), b = lap_at(xm + m * n2, N, j, i);
        s += a * a + b * b;
    }
    const double t = block_sum(s, sh);
    if (threadIdx.x == 0) partial[m * gridDim.x + blockIdx.x] = t;
}

// partial <a, b> over both parts
__global__ void dot2_kernel(const float* __restrict__ al, const float* __restrict__ am,
                            const float* __restrict__ bl, const float* __restrict__ bm, double* partial, int n2)
{
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

// Scalar steps of the LM iteration (one thread per member).
__global__ void scalar_kernel(int op, int k, const double* p0, const double* p1, const double* p2, int nblk,
                              CGState* st, pget_gn_stats* stats, int B, double alpha, double beta)
{
    const int m = blockIdx.x * blockDim.x + threadIdx.x;
    if (m >= B) return;
    CGState& c = st[m];
    pget_gn_stats& S = stats[m];
    if (op == SC_INIT) {             // p0: 1/2||r||^2, p1: ||Lu||^2, p2: ||b||^2
        const double mis = psum(p0, m, nblk), lq = psum(p1, m, nblk), bb = psum(p2, m, nblk);
        S.misfit = mis;
        S.reg = 0.5 * alpha * lq;
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
        S.bs = bs;
        S.pred = bs - 0.5 * (js2 + alpha * ls2);
    } else if (op == SC_TRIAL) {     // p0: 1/2||r(u+s)||^2, p1: ||L(u+s)||^2
        const double f1 = psum(p0, m, nblk) + 0.5 * alpha * psum(p1, m, nblk);
        S.f_trial = f1;
        S.rho = (S.f - f1) / S.pred;
        S.accepted = S.rho > 0.1;
        double bn = beta;
        if (!S.accepted) bn = (10.0 * beta > S.beta_min) ? 10.0 * beta : S.beta_min;
        else if (S.rho > 0.75) bn = 0.2 * beta;
        S.beta_next = bn;
    }
}

}  // namespace pget

namespace pget {

// Host launcher of the projector (instantiates every (MODE, MAXR) pair).
template <int MODE>
static cudaError_t launch_mode(int maxr, const ProjArgs& A, int grid, int block, size_t smem, cudaStream_t s)
{
    switch (maxr) {
    case 1: proj_kernel<MODE, 1><<<grid, block, smem, s>>>(A); break;
    case 2: proj_kernel<MODE, 2><<<grid, block, smem, s>>>(A); break;
    case 4: proj_kernel<MODE, 4><<<grid, block, smem, s>>>(A); break;
    default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_proj(int mode, int maxr, const ProjArgs& A, int grid, int block, size_t smem, cudaStream_t s)
{
    switch (mode) {
    case MODE_FWD: return launch_mode<MODE_FWD>(maxr, A, grid, block, smem, s);
    case MODE_JVP: return launch_mode<MODE_JVP>(maxr, A, grid, block, smem, s);
    case MODE_VJP: return launch_mode<MODE_VJP>(maxr, A, grid, block, smem, s);
    case MODE_GN: return launch_mode<MODE_GN>(maxr, A, grid, block, smem, s);
    }
    return cudaErrorInvalidValue;
}

template <int MODE>
static cudaError_t attr_mode(size_t smem)
{
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(proj_kernel<MODE, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem))) return e;
    if ((e = cudaFuncSetAttribute(proj_kernel<MODE, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem))) return e;
    return cudaFuncSetAttribute(proj_kernel<MODE, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

cudaError_t set_proj_smem_limit(size_t smem)
{
    cudaError_t e;
    if ((e = attr_mode<MODE_FWD>(smem))) return e;
    if ((e = attr_mode<MODE_JVP>(smem))) return e;
    if ((e = attr_mode<MODE_VJP>(smem))) return e;
    return attr_mode<MODE_GN>(smem);
}

}  // namespace pget
