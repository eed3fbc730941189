// sid.cu -- the pixel-basis model variant (N3, reading R-pb): exact intersection lengths d_{m,n,k}
// of eq:d_fwd_model, optionally with the collimator response r and the
// opening-angle correction c of reading R-N3.
//
// lam, mu are constant on each pixel.  A ray crosses pixels k_1..k_M (increasing t, the detector at
// +t) with lengths l_q; the ray from pixel k_q starts at the midpoint of its chord:
//     A_q = l_q mu_q / 2 + sum_{p>q} l_p mu_p,   g_ray = sum_q r_q lam_q exp(-c_q A_q),
//     r_q = l_q (x W_j(d_q) with the response), c_q = 1 (or 1 + c_slope d_q), d_q = det_radius - t_q,
//     y_d = sum_j w_j g_ray(d, j)  (w_j = 1 with the response: W_j is inside the ray sum).
// JVP: dg = sum_q r_q (dlam_q - lam_q c_q dA_q) E_q;  VJP: a_lam(q) = w r_q E_q,
// a_mu(q) = -w l_q (sum_{p<q} r_p lam_p c_p E_p + r_q lam_q c_q E_q / 2).
//
// Design.  A CTA per (angle-bank, chunk of whole detectors, member), ~128 rays, one
// thread per ray, images read through L1/L2 from the packed padded float2 / float4 images (a ray reads one pixel per crossing; adjacent
// lanes trace adjacent rays, so a warp's reads fall on a few neighbouring pixels).  The traversal
// (Siddon's crossing merge, walked from the detector end so the optical depth accumulates) is fp64
// with the oracle's exact operation order (explicit _rn intrinsics, no contraction): every pixel
// index and interval length is the oracle's bit for bit, including the measure-zero lines that run
// along a pixel edge.  The sums are fp32 with Kahan compensation, exponentials by ex2.approx.  The
// adjoint scatters into a 64-bit fixed-point accumulator per member in global memory (integer
// red.global.add: order-independent, so the result is deterministic) at a power-of-two scale from
// per-member magnitude bounds taken in a first pass; a last pass converts it to the fp64 partials the
// finish / CG kernels read.
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>
#include <mutex>
#include <type_traits>

#include "kernels.cuh"

#ifndef PGET_SID_CHUNK
#define PGET_SID_CHUNK 1   // CTAs of whole detectors, ~128 rays (0: one CTA per angle-bank; experiment switch)
#endif
#ifndef PGET_SID_MINB
#define PGET_SID_MINB 1   // CTAs per SM the register allocation targets (experiment switch)
#endif

namespace pget {

namespace {

constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ float sx2(float x)
{
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ void kadd(float& s, float& c, float x)   // Kahan: s - c is the sum
{
    const float y = x - c;   // c: what the last rounded add gained beyond its inputs
    const float t = s + y;
    c = (t - s) - y;
    s = t;
}

// The line of ray r of angle-bank ab in pixel units (the oracle's o14_cross, same fp64 operations)
struct Line {
    double X0, Y0, wX, wY, iX, iY, tin, tout;
};

__device__ __forceinline__ bool line_of(const SidArgs& A, int ab, int r, Line& L)
{
    const double c = A.dir[2 * ab], s = A.dir[2 * ab + 1];
    const double sigma = A.off[static_cast<size_t>(ab % A.nB) * A.R + r];
    const double hN = 0.5 * static_cast<double>(A.N);
    L.X0 = __dmul_rn(__dadd_rn(__dmul_rn(-sigma, s), 1.0), hN);
    L.Y0 = __dmul_rn(__dadd_rn(__dmul_rn(sigma, c), 1.0), hN);
    L.wX = __dmul_rn(c, hN);
    L.wY = __dmul_rn(s, hN);
    L.iX = L.iY = 0.0;
    double tin = -INFINITY, tout = INFINITY;
    const double Nd = static_cast<double>(A.N);
    auto axis = [&](double X0, double w, double& inv) -> bool {
        if (w == 0.0) return X0 > 0.0 && X0 < Nd;
        inv = __ddiv_rn(1.0, w);
        const double t1 = __dmul_rn(__dsub_rn(0.0, X0), inv), t2 = __dmul_rn(__dsub_rn(Nd, X0), inv);
        const double lo = t1 < t2 ? t1 : t2, hi = t1 < t2 ? t2 : t1;
        if (lo > tin) tin = lo;
        if (hi < tout) tout = hi;
        return true;
    };
    if (!axis(L.X0, L.wX, L.iX) || !axis(L.Y0, L.wY, L.iY)) return false;
    L.tin = tin;
    L.tout = tout;
    return tin < tout;
}

// Edge crossings of one axis, walked towards decreasing t: t_e = (e - X0) / w for e in [0, N], only
// those strictly inside (tin, tout).  next() returns the current one (-inf when exhausted).
struct Edges {
    int e, de, N;
    double X0, inv, tin, t;
    __device__ __forceinline__ double te(int k) const { return __dmul_rn(__dsub_rn(static_cast<double>(k), X0), inv); }
    __device__ __forceinline__ void init(double X0_, double w, double inv_, double tin_, double tout, int N_)
    {
        X0 = X0_; inv = inv_; tin = tin_; N = N_;
        if (w == 0.0) { t = -INFINITY; e = -1; de = 0; return; }
        de = inv > 0.0 ? -1 : 1;   // decreasing t
        const double Xe = __dadd_rn(X0, __dmul_rn(tout, w));
        int k = inv > 0.0 ? static_cast<int>(floor(Xe)) : static_cast<int>(ceil(Xe));
        k = max(0, min(N, k));
        while (k >= 0 && k <= N && !(te(k) < tout)) k += de;
        while (k - de >= 0 && k - de <= N && te(k - de) < tout) k -= de;
        e = k;
        set();
    }
    __device__ __forceinline__ void set()
    {
        t = (e >= 0 && e <= N) ? te(e) : -INFINITY;
        if (!(t > tin)) t = -INFINITY;
    }
    __device__ __forceinline__ void step() { e += de; set(); }
};

// Walk the crossings of a line from the detector end: visit(fetch(row, col), row, col, l, tm) per
// interval of positive length, in order of decreasing t.  (Measured: issuing each pixel load one
// interval ahead of its use, with the traversal as a generator, made every mode 5-15 % slower.)
template <class Fe, class F>
__device__ __forceinline__ void walk(const Line& L, int N, Fe&& fetch, F&& visit)
{
    Edges ex, ey;
    ex.init(L.X0, L.wX, L.iX, L.tin, L.tout, N);
    ey.init(L.Y0, L.wY, L.iY, L.tin, L.tout, N);
    double tc = L.tout;
    while (true) {
        const double tn = fmax(fmax(ex.t, ey.t), L.tin);
        const double l = __dsub_rn(tc, tn);
        if (l > 0.0) {
            const double tm = __dmul_rn(0.5, __dadd_rn(tn, tc));
            int col = static_cast<int>(floor(__dadd_rn(L.X0, __dmul_rn(tm, L.wX))));
            int row = static_cast<int>(floor(__dadd_rn(L.Y0, __dmul_rn(tm, L.wY))));
            col = max(0, min(N - 1, col));
            row = max(0, min(N - 1, row));
            visit(fetch(row, col), row, col, l, tm);
        }
        if (!(tn > L.tin)) break;
        const bool sx = ex.t == tn, sy = ey.t == tn;
        if (sx) ex.step();
        if (sy) ey.step();
        tc = tn;
    }
}

// the response of reading R-N3 at distance d (fp32): c = 1 + c_slope d, W_j(d) = normalised Gaussian
// of width sig0 (1 + r_slope d) over the J sub-ray offsets (A.dj2 = delta_k^2 log2(e))
__device__ __forceinline__ void resp(const SidArgs& A, int j, double tm, float& cq, float& W)
{
    const float d = static_cast<float>(__dsub_rn(A.det_radius, tm));
    cq = fmaf(A.c_slope, d, 1.f);
    const float sg = A.sig0 * fmaf(A.r_slope, d, 1.f);
    const float k = -0.5f / (sg * sg);
    float sum = 0.f, wj = 0.f;
    for (int q = 0; q < A.J; ++q) {
        const float e = sx2(A.dj2[q] * k);
        sum += e;
        if (q == j) wj = e;
    }
    W = wj / sum;
}

struct RayState {
    float s, sc;        // -log2(e) sum_{visited} l mu  (Kahan pair)
    float g, gc;        // sum r lam E (forward) or sum r lam c E (adjoint G)
    float ds, dsc;      // sum l dmu
    float dg, dgc;      // JVP sum
    float gabs, lsum;   // adjoint bounds: sum r |lam| c E, sum r E
};

// one ray of MODE: FWD (g), JVP (g, dg), VJP / GN pass 1 (G, bounds; GN also (J p))
template <int MODE, bool VAR>
__device__ __forceinline__ RayState ray_sums(const SidArgs& A, int m, int ab, int r)
{
    RayState st = {};
    Line L;
    if (!line_of(A, ab, r, L)) return st;
    const int j = r % A.J;
    const size_t base = static_cast<size_t>(m) * A.P * A.P;
    constexpr bool F4 = MODE == MODE_JVP || MODE == MODE_GN;
    using Px = typename std::conditional<F4, float4, float2>::type;
    auto fetch = [&](int row, int col) -> Px {
        const size_t o = base + static_cast<size_t>(row + kHalo) * A.P + (col + kHalo);
        if constexpr (F4) return __ldg(A.img4 + o);
        else return __ldg(A.img2 + o);
    };
    walk(L, A.N, fetch, [&](const Px& x, int, int, double l, double tm) {
        float lam = x.x, mu = x.y, dlam = 0.f, dmu = 0.f;
        if constexpr (F4) {
            dlam = x.z;
            dmu = x.w;
        }
        const float lf = static_cast<float>(l);
        float cq = 1.f, rq = lf;
        if constexpr (VAR) {
            float W;
            resp(A, j, tm, cq, W);
            rq = W * lf;
        }
        const float kl = -kLog2e * lf;
        const float arg = fmaf(mu, 0.5f * kl, st.s) - st.sc;   // -log2(e) A_q
        kadd(st.s, st.sc, mu * kl);
        const float E = sx2(VAR ? cq * arg : arg);
        if constexpr (MODE == MODE_FWD) {
            kadd(st.g, st.gc, rq * lam * E);
        } else {
            const float le = rq * lam * (VAR ? cq : 1.f) * E;
            kadd(st.g, st.gc, MODE == MODE_JVP ? rq * lam * E : le);
            if constexpr (MODE != MODE_JVP) {
                st.gabs += fabsf(le);
                st.lsum += rq * E;
            }
        }
        if constexpr (F4) {
            const float dA = fmaf(0.5f * lf, dmu, st.ds - st.dsc);   // l dmu / 2 + sum_{p>q} l dmu
            kadd(st.ds, st.dsc, lf * dmu);
            const float jt = rq * fmaf(-lam * (VAR ? cq : 1.f), dA, dlam);
            kadd(st.dg, st.dgc, jt * E);
        }
    });
    return st;
}

// ---- forward / JVP: per-ray sums, then the sub-ray weighting into the detector readings
template <int MODE, bool VAR>
__global__ void __launch_bounds__(256, PGET_SID_MINB) sid_proj_kernel(SidArgs A)
{
    pdl_entry();
    extern __shared__ float rout[];   // [2 dpc J]: the CTA's rays
    const int ab = blockIdx.x / A.nch, ch = blockIdx.x - ab * A.nch, m = blockIdx.y;
    const int d0 = ch * A.dpc, d1 = min(A.n_det, d0 + A.dpc), ra = d0 * A.J, nr = (d1 - d0) * A.J;
    for (int t = threadIdx.x; t < nr; t += blockDim.x) {
        const RayState st = ray_sums<MODE, VAR>(A, m, ab, ra + t);
        rout[t] = st.g - st.gc;
        if (MODE == MODE_JVP) rout[nr + t] = st.dg - st.dgc;
    }
    __syncthreads();
    const size_t ob = (static_cast<size_t>(m) * A.n_ab + ab) * A.n_det;
    for (int d = d0 + threadIdx.x; d < d1; d += blockDim.x) {
        float acc = 0.f, dacc = 0.f;
        for (int j = 0; j < A.J; ++j) {
            acc = fmaf(A.wj[j], rout[(d - d0) * A.J + j], acc);
            if (MODE == MODE_JVP) dacc = fmaf(A.wj[j], rout[nr + (d - d0) * A.J + j], dacc);
        }
        if (A.y) A.y[ob + d] = acc;
        if (MODE == MODE_JVP) A.dy[ob + d] = dacc;
    }
}

// ---- adjoint pass 1 (VJP: weights from A.win; GN: the (J p) of A.img4's p): per ray the weight w_r,
// G (compensated) into A.ray, and the member's magnitude bounds max|w| sum r E, max|w| l_max sum r|lam|cE
template <int MODE, bool VAR>
__global__ void __launch_bounds__(256, PGET_SID_MINB) sid_adj_a_kernel(SidArgs A)
{
    pdl_entry();
    extern __shared__ float rout[];   // [dpc J]: GN (J p) per ray of the CTA
    __shared__ float red[2][32];
    const int ab = blockIdx.x / A.nch, ch = blockIdx.x - ab * A.nch, m = blockIdx.y, R = A.R, J = A.J;
    const int d0 = ch * A.dpc, d1 = min(A.n_det, d0 + A.dpc), ra = d0 * J, re = d1 * J;
    const size_t rb = (static_cast<size_t>(m) * A.n_ab + ab) * R;
    for (int r = ra + threadIdx.x; r < re; r += blockDim.x) {
        const RayState st = ray_sums<MODE, VAR>(A, m, ab, r);
        A.ray[rb + r] = make_float4(0.f, st.g, st.gc, 0.f);
        A.raybd[rb + r] = make_float2(st.lsum, st.gabs);
        if (MODE == MODE_GN) rout[r - ra] = st.dg - st.dgc;
    }
    __syncthreads();
    float bl = 0.f, bm = 0.f;
    const size_t ob = (static_cast<size_t>(m) * A.n_ab + ab) * A.n_det;
    for (int r = ra + threadIdx.x; r < re; r += blockDim.x) {
        const int d = r / J, j = r - d * J;
        float wd;
        if (MODE == MODE_GN) {
            wd = 0.f;
            for (int q = 0; q < J; ++q) wd = fmaf(A.wj[q], rout[(d - d0) * J + q], wd);
        } else {
            wd = A.win[ob + d];
        }
        const float wr = A.wj[j] * wd;
        A.ray[rb + r].x = wr;
        const float2 bd = A.raybd[rb + r];
        bl = fmaxf(bl, fabsf(wr) * bd.x);
        bm = fmaxf(bm, fabsf(wr) * A.lmax * bd.y);
    }
    for (int o = 16; o > 0; o >>= 1) {
        bl = fmaxf(bl, __shfl_xor_sync(0xffffffffu, bl, o));
        bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, o));
    }
    if ((threadIdx.x & 31) == 0) {
        red[0][threadIdx.x >> 5] = bl;
        red[1][threadIdx.x >> 5] = bm;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 1; k < static_cast<int>(blockDim.x >> 5); ++k) {
            bl = fmaxf(bl, red[0][k]);
            bm = fmaxf(bm, red[1][k]);
        }
        // non-negative floats order as their bit patterns: an order-independent (deterministic) max
        atomicMax(A.bound + 2 * m, __float_as_uint(bl));
        atomicMax(A.bound + 2 * m + 1, __float_as_uint(bm));
    }
}

// the fixed-point scale of a plane: every pixel's sum of |contributions| is at most nhits x bound;
// S = 2^(61 - e) with nhits x bound < 2^e keeps it below 2^61 (exact power-of-two scaling both ways)
__device__ __forceinline__ double fx_scale(unsigned bits, double nhits)
{
    const double b = static_cast<double>(__uint_as_float(bits)) * nhits;
    if (!(b > 0.0) || !isfinite(b)) return 1.0;
    int e;
    frexp(b, &e);
    return ldexp(1.0, 61 - e);
}

__device__ __forceinline__ void red_u64(unsigned long long* p, double v)
{
    const long long q = __double2ll_rn(v);
    atomicAdd(p, static_cast<unsigned long long>(q));   // two's complement: signed sums wrap exactly
}

// ---- adjoint pass 2: walk again (the same E bit for bit) and scatter the adjoint weights
template <bool VAR>
__global__ void __launch_bounds__(256, PGET_SID_MINB) sid_adj_b_kernel(SidArgs A, bool f4)
{
    pdl_entry();
    const int ab = blockIdx.x / A.nch, ch = blockIdx.x - ab * A.nch, m = blockIdx.y, R = A.R;
    const int d0 = ch * A.dpc, d1 = min(A.n_det, d0 + A.dpc);
    const size_t rb = (static_cast<size_t>(m) * A.n_ab + ab) * R;
    const double Sl = fx_scale(A.bound[2 * m], A.nhits), Sm = fx_scale(A.bound[2 * m + 1], A.nhits);
    const size_t n2 = static_cast<size_t>(A.N) * A.N;
    unsigned long long* accl = A.acc + static_cast<size_t>(m) * 2 * n2;
    unsigned long long* accm = accl + n2;
    const size_t base = static_cast<size_t>(m) * A.P * A.P;
    for (int r = d0 * A.J + threadIdx.x; r < d1 * A.J; r += blockDim.x) {
        const float4 rv = A.ray[rb + r];
        const float w = rv.x, G = rv.y, Gc = rv.z;
        if (w == 0.f) continue;
        Line L;
        if (!line_of(A, ab, r, L)) continue;
        const int j = r % A.J;
        float s = 0.f, sc = 0.f, Q = 0.f, Qc = 0.f;
        auto fetch = [&](int row, int col) -> float2 {
            const size_t o = base + static_cast<size_t>(row + kHalo) * A.P + (col + kHalo);
            if (f4) {
                const float4 x = __ldg(A.img4 + o);
                return make_float2(x.x, x.y);
            }
            return __ldg(A.img2 + o);
        };
        walk(L, A.N, fetch, [&](const float2& x, int row, int col, double l, double tm) {
            const float lam = x.x, mu = x.y;
            const float lf = static_cast<float>(l);
            float cq = 1.f, rq = lf;
            if constexpr (VAR) {
                float W;
                resp(A, j, tm, cq, W);
                rq = W * lf;
            }
            const float kl = -kLog2e * lf;
            const float arg = fmaf(mu, 0.5f * kl, s) - sc;
            kadd(s, sc, mu * kl);
            const float E = sx2(VAR ? cq * arg : arg);
            const float le = rq * lam * (VAR ? cq : 1.f) * E;
            const float al = w * rq * E;
            const float am = -w * lf * (((G - Q) - (Gc - Qc)) - 0.5f * le);
            kadd(Q, Qc, le);
            const size_t px = static_cast<size_t>(row) * A.N + col;
            red_u64(accl + px, static_cast<double>(al) * Sl);
            red_u64(accm + px, static_cast<double>(am) * Sm);
        });
    }
}

// ---- adjoint pass 3: fixed point -> the fp64 partials (G = 1) of the finish / CG kernels
__global__ void __launch_bounds__(256, PGET_SID_MINB) sid_adj_fin_kernel(SidArgs A, double2* gacc)
{
    pdl_entry();
    const int m = blockIdx.y;
    const size_t n2 = static_cast<size_t>(A.N) * A.N;
    const double il = 1.0 / fx_scale(A.bound[2 * m], A.nhits), im = 1.0 / fx_scale(A.bound[2 * m + 1], A.nhits);
    const unsigned long long* accl = A.acc + static_cast<size_t>(m) * 2 * n2;
    const unsigned long long* accm = accl + n2;
    for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < n2;
         e += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const double a = static_cast<double>(static_cast<long long>(accl[e])) * il;
        const double b = static_cast<double>(static_cast<long long>(accm[e])) * im;
        gacc[static_cast<size_t>(m) * n2 + e] = make_double2(a, b);
    }
}

}  // namespace

// CTAs of whole detectors (the sub-ray weighting stays in shared memory), about 128 rays each, one ray
// per thread: (angle-bank, detector chunk, member) -- thousands of small CTAs instead of one CTA per
// angle-bank looping over its rays in rounds of 256 (whose last round and last wave ran mostly idle)
static SidArgs sid_chunks(const SidArgs& A0, int& nt)
{
    SidArgs A = A0;
    if (!PGET_SID_CHUNK) {   // one CTA of 256 threads per angle-bank (the first design)
        A.dpc = A.n_det;
        A.nch = 1;
        nt = 256;
        return A;
    }
    const int nch0 = std::max(1, (A.R + 127) / 128);
    A.dpc = std::max(1, (A.n_det + nch0 - 1) / nch0);
    A.nch = (A.n_det + A.dpc - 1) / A.dpc;
    nt = std::min(256, std::max(32, (A.dpc * A.J + 31) / 32 * 32));
    return A;
}

cudaError_t launch_sid_proj(int mode, bool var, const SidArgs& A0, cudaStream_t s)
{
    int nt;
    const SidArgs A = sid_chunks(A0, nt);
    const dim3 grid(A.n_ab * A.nch, A.B);
    const size_t sm = 2 * sizeof(float) * A.dpc * A.J;
    if (mode == MODE_FWD)
        return var ? launch_k(sid_proj_kernel<MODE_FWD, true>, grid, nt, sm, s, A)
                   : launch_k(sid_proj_kernel<MODE_FWD, false>, grid, nt, sm, s, A);
    return var ? launch_k(sid_proj_kernel<MODE_JVP, true>, grid, nt, sm, s, A)
               : launch_k(sid_proj_kernel<MODE_JVP, false>, grid, nt, sm, s, A);
}

cudaError_t launch_sid_adj(int mode, bool var, const SidArgs& A0, double2* gacc, cudaStream_t s)
{
    int nt;
    const SidArgs A = sid_chunks(A0, nt);
    const dim3 grid(A.n_ab * A.nch, A.B);
    const size_t n2 = static_cast<size_t>(A.N) * A.N;
    cudaError_t e = cudaMemsetAsync(A.bound, 0, 2 * sizeof(unsigned) * A.B, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(A.acc, 0, 2 * n2 * sizeof(unsigned long long) * A.B, s);
    const size_t sm = sizeof(float) * A.dpc * A.J;
    if (e == cudaSuccess) {
        if (mode == MODE_GN)
            e = var ? launch_k(sid_adj_a_kernel<MODE_GN, true>, grid, nt, sm, s, A)
                    : launch_k(sid_adj_a_kernel<MODE_GN, false>, grid, nt, sm, s, A);
        else
            e = var ? launch_k(sid_adj_a_kernel<MODE_VJP, true>, grid, nt, sm, s, A)
                    : launch_k(sid_adj_a_kernel<MODE_VJP, false>, grid, nt, sm, s, A);
    }
    const bool f4 = mode == MODE_GN;
    if (e == cudaSuccess)
        e = var ? launch_k(sid_adj_b_kernel<true>, grid, nt, 0, s, A, f4)
                : launch_k(sid_adj_b_kernel<false>, grid, nt, 0, s, A, f4);
    if (e == cudaSuccess) {
        const int nb = static_cast<int>(std::min<size_t>((n2 + 255) / 256, 1024));
        e = launch_k(sid_adj_fin_kernel, dim3(nb, A.B), 256, 0, s, A, gacc);
    }
    return e;
}

// the dynamic shared memory the kernels need (2 R floats), raised process-wide and never lowered: a
// handle with fewer rays created later must not break an earlier, larger one
cudaError_t set_sid_smem_limit(size_t bytes)
{
    static std::mutex mu;
    static size_t high = 48 * 1024;   // the default limit
    std::lock_guard<std::mutex> lk(mu);
    if (bytes <= high) return cudaSuccess;
    cudaError_t e = cudaSuccess;
    const int b = static_cast<int>(bytes);
    for (auto k : {sid_proj_kernel<MODE_FWD, false>, sid_proj_kernel<MODE_FWD, true>, sid_proj_kernel<MODE_JVP, false>,
                   sid_proj_kernel<MODE_JVP, true>})
        if (e == cudaSuccess) e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
    for (auto k : {sid_adj_a_kernel<MODE_VJP, false>, sid_adj_a_kernel<MODE_VJP, true>, sid_adj_a_kernel<MODE_GN, false>,
                   sid_adj_a_kernel<MODE_GN, true>})
        if (e == cudaSuccess) e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
    if (e == cudaSuccess) high = bytes;
    return e;
}

}  // namespace pget
