// proj.cu -- the ray-driven projector of the PGET hot path on sm_100a.
//
// Model (PAPER.md:48-54 eq:fwd_model, discretised per SURVEY.md §8(c.2) O1-O5):
//   A_i  = Delta (mu_i / 2 + sum_{k>i} mu_k)                      (B mu, k > i: nearer the detector)
//   y    = sum_j w_j Delta sum_i lam_i E_i,   E_i = exp(-A_i)
//   dy   = sum_j w_j Delta sum_i (dlam_i - lam_i dA_i) E_i         (eq:frechet)
//   VJP  : a_lam(i) = w_r Delta E_i,  a_mu(i) = -w_r Delta^2 (G - Q_i - lam_i E_i / 2),
//          G = sum_i lam_i E_i, Q_i = sum_{k>i} lam_k E_k, scattered with the transposed bilinear
//          weights (the exact transpose of the discrete JVP; adjoint F'^* of PAPER.md:231, 277)
//   GN   : J^T (J p) fused per angle-bank: sweep A = JVP of p, per-detector (J p), sweep B = VJP.
//
// Execution model:
//   * persistent CTAs, each owning a static contiguous range of tasks (member, angle-bank); angle-banks
//     are ordered by orientation class; a CTA's range covers few (member, class, chunk) segments;
//   * class 0 angle-banks sample the padded image as is, class 1 the transposed copy, so that in the
//     oriented frame every ray advances >= 1/(2 sqrt2) rows per sample and crosses every row band;
//   * the image is streamed through shared memory in row bands by 1-D bulk async copies (TMA engine,
//     cp.async.bulk + mbarrier), double buffered across bands, passes and tasks;
//   * a lane owns a ray; the 32 lanes of a warp own a "comb" of rays >= 2 sqrt2 px apart, so the
//     bilinear footprints of a warp's samples never overlap: the VJP scatter is a plain shared-memory
//     read-modify-write into a warp-private ring of band rows (no atomics in the sample loop);
//   * per-ray sums that cancel (optical depth, JVP and adjoint sums) are Kahan-compensated
//     (DESIGN.md "Precision"); one ex2 per sample;
//   * the VJP band rows are flushed into a CTA-private fp32 partial image (one slot per segment);
//     a fixed-order fp64 reduction of the slots (reduce_slots_kernel) makes the gradient deterministic.
#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <mutex>
#include <utility>

#include "internal.h"
#include "kernels.cuh"

// PGET_DEBUG builds (-DPGET_DEBUG, scripts/debug_check.sh) trap on any out-of-range shared-memory
// index of the sample loops (compute-sanitizer is closed on the GPU pool).
#ifdef PGET_DEBUG
#define PGET_CHECK(c) \
    do {              \
        if (!(c)) __trap(); \
    } while (0)
#else
#define PGET_CHECK(c) \
    do {              \
    } while (0)
#endif

#ifndef PGET_ABLATE
#define PGET_ABLATE 0   // performance experiments only (scripts/ablate.sh); 0 in every real build
#endif

namespace pget {

// ------------------------------------------------------------------------------------------ helpers
__device__ __forceinline__ float frac23(int64_t x)
{
    return __uint_as_float((static_cast<uint32_t>(x) >> 9) | 0x3f800000u) - 1.0f;
}

// 1 + frac23(x), exactly (the float in [1, 2) whose mantissa is the rounded fraction)
__device__ __forceinline__ float frac23p1(int64_t x)
{
    return __uint_as_float((static_cast<uint32_t>(x) >> 9) | 0x3f800000u);
}

__device__ __forceinline__ int hi32(int64_t x) { return static_cast<int>(x >> 32); }
// the high word as the register it is (the compiler otherwise folds ">> 32, * 4" into a funnel shift
// by 30 plus a mask)
__device__ __forceinline__ int hi32r(int64_t x)
{
    int hi;
    asm("{\n\t.reg .b32 lo;\n\tmov.b64 {lo, %0}, %1;\n\t}" : "=r"(hi) : "l"(x));
    return hi;
}

__device__ __forceinline__ float ex2(float x)
{
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// bilinear lerp of a channel pair: a=(j0,i0) b=(j0,i0+1) c=(j0+1,i0) d=(j0+1,i0+1)
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

// the four bilinear corners of a sample in the staged band: o = (iv - r0) * P + iu
template <bool NF4>
struct Px;
template <>
struct Px<true> {
    float4 a, b, c, d;
};
template <>
struct Px<false> {
    float2 a, b, c, d;
};
__device__ __forceinline__ void load_px(Px<true>& x, const unsigned char* sb, int o, int P)
{
    const float4* p = reinterpret_cast<const float4*>(sb) + o;
    x.a = p[0]; x.b = p[1]; x.c = p[P]; x.d = p[P + 1];
}
__device__ __forceinline__ void load_px(Px<false>& x, const unsigned char* sb, int o, int P)
{
    const float2* p = reinterpret_cast<const float2*>(sb) + o;
    x.a = p[0]; x.b = p[1]; x.c = p[P]; x.d = p[P + 1];
}

// Kahan step: (s, c) += x  (the compensated sum is s - c)
__device__ __forceinline__ void kahan(float& s, float& c, float x)
{
    const float y = x - c;
    const float t = s + y;
    c = (t - s) - y;
    s = t;
}

// ---- mbarrier + 1-D bulk async copy (TMA engine)
__device__ __forceinline__ uint32_t smem_u32(const void* p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity)
{
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// ------------------------------------------------------------------------------------------ tasks
struct TaskInfo {
    int m, ab, cls, dir, dlo, dhi, gbeg, gend, slot, first;
};

__device__ __forceinline__ TaskInfo task_info(const ProjArgs& A, int64_t t)
{
    const TaskD td = A.tasks[t];
    TaskInfo ti;
    ti.m = td.m;
    ti.ab = td.ab;
    ti.cls = (td.flags & kTaskClass1) ? 1 : 0;
    ti.first = (td.flags & kTaskFirst) ? 1 : 0;
    ti.dlo = td.dlo;
    ti.dhi = td.dhi;
    ti.gbeg = td.gbeg;
    ti.gend = td.gend;
    ti.slot = td.slot;
    ti.dir = A.rays[static_cast<size_t>(ti.ab) * A.R].dV > 0 ? 1 : -1;
    return ti;
}

// the angle-bank whose rays duplicate those of ab (a + n_A/2, bank 1 - b); ab itself without dup
__device__ __forceinline__ int dup_of(const ProjArgs& A, int ab)
{
    if (!A.dup_half) return ab;
    const int a = ab >> 1, b = ab & 1;
    return (a + A.dup_half) * 2 + (1 - b);
}

__device__ __forceinline__ void band_rows(int band, int Rb, int P, int& r0, int& r1)
{
    r0 = band * Rb;
    r1 = min(r0 + Rb, P - 1);
}

// Issue the bulk copy of global stage `sidx` (a band of sweep A or B of some task) into `dst`.
template <int MODE>
__device__ void issue_stage(const ProjArgs& A, int64_t t0, int ns_task, int64_t sidx, void* dst, uint64_t* bar)
{
    const int64_t t = t0 + sidx / ns_task;
    const int l = static_cast<int>(sidx % ns_task);
    const TaskInfo ti = task_info(A, t);
    const bool isA = l < A.passesA * A.nbA;
    const int nb = isA ? A.nbA : A.nbB;
    const int Rb = isA ? A.RbA : A.RbB;
    const int kb = isA ? l % A.nbA : (l - A.passesA * A.nbA) % A.nbB;
    const int band = ti.dir > 0 ? nb - 1 - kb : kb;
    int r0, r1;
    band_rows(band, Rb, A.P, r0, r1);
    const size_t pix0 = static_cast<size_t>(ti.m) * A.P * A.P + static_cast<size_t>(r0) * A.P;
    const size_t npix = static_cast<size_t>(r1 - r0 + 1) * A.P;
    const char* src;
    size_t bytes;
    if (isA && (MODE == MODE_JVP || MODE == MODE_GN)) {
        src = reinterpret_cast<const char*>(A.img4[ti.cls] + pix0);
        bytes = npix * sizeof(float4);
    } else {
        src = reinterpret_cast<const char*>(A.img2[ti.cls] + pix0);
        bytes = npix * sizeof(float2);
    }
    fence_proxy_async();
    mbar_expect_tx(bar, static_cast<uint32_t>(bytes));
    char* d = static_cast<char*>(dst);
    for (size_t off = 0; off < bytes; off += 32768) {
        const uint32_t n = static_cast<uint32_t>(bytes - off < 32768 ? bytes - off : 32768);
        bulk_g2s(d + off, src + off, n, bar);
    }
}

template <int MODE>
struct ModeTraits {
    static constexpr int W = (MODE == MODE_VJP || MODE == MODE_GN) ? 16 : 8;    // most warps per CTA
    static constexpr int MINB = MODE == MODE_FWD ? 3 : (MODE == MODE_JVP ? 2 : 1); // CTAs per SM
    static constexpr bool HAS_B = (MODE == MODE_VJP || MODE == MODE_GN);         // adjoint sweep
    static constexpr bool NF4 = (MODE == MODE_JVP || MODE == MODE_GN);           // 4-channel sweep A
#ifndef PGET_GN_COMP
#define PGET_GN_COMP 0
#endif
    // compensated sums: the JVP and VJP are graded per element (max-relative 1e-4, R-precision); the
    // GN product, graded as an operator in relative L2 (1e-5), runs plain fp32 sums (PGET_GN_COMP 0)
    static constexpr bool COMP_S = MODE == MODE_JVP || MODE == MODE_VJP || (MODE == MODE_GN && PGET_GN_COMP);
    static constexpr bool COMP_G = MODE == MODE_VJP || (MODE == MODE_GN && PGET_GN_COMP);
    // compensated JVP sums: the standalone JVP is graded per element (max-relative 1e-4, DESIGN.md
    // R-precision); inside the GN product the (J p) sums feed an operator graded in relative L2
    // (1e-5), where plain fp32 sums are ~1e-7 -- the GN mode saves the 4-FADD Kahan steps there
    static constexpr bool COMP_J = MODE == MODE_JVP;
};

// ------------------------------------------------------------------------------------------ walkers
// One lane walks one ray through one staged band, detector end first.  The four bilinear corners of
// sample i-1 are loaded before sample i is evaluated (software pipeline: the shared-memory latency of
// the next sample overlaps the arithmetic of the current one).  Measured alternative (DESIGN.md
// "Projector"): caching the corners across samples of one cell cut shared-memory wavefronts 3x but the
// per-lane move logic doubled the issued instructions and lost, so every sample loads its corners.
template <bool NF4>
struct CornerT;
template <>
struct CornerT<true> {
    using T = float4;
};
template <>
struct CornerT<false> {
    using T = float2;
};

// explicit shared-memory corner loads from a 32-bit shared-space address (+ an immediate byte offset)
template <int OFF>
__device__ __forceinline__ void lds_c(float4& v, uint32_t a)
{
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4+%5];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(a), "n"(OFF)
                 : "memory");
}
template <int OFF>
__device__ __forceinline__ void lds_c(float2& v, uint32_t a)
{
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2+%3];" : "=f"(v.x), "=f"(v.y) : "r"(a), "n"(OFF) : "memory");
}

struct StateA {
    float s, sc, g, gc, ds, dg, dgc;
    float p1, p1c, p2, p2c, p3, p3c;   // PAIRED: sums over e^{+A_i} for the reverse-direction ray
    // PAIRED (reading R-depth): s, sc and p1..p3 are local to the current band; Lb, Lbc is the depth
    // before the band and R1..R3 the reverse-direction sums rebased to the current depth,
    // R_k = 2^{L} sum_{visited} (.) 2^{-L_i} <= sum (.), folded in at every band end (fold_a)
    float Lb, Lbc, R1, R2, R3;
};

// PAIRED: close a band.  The reverse-direction sums of the band (relative to the band start, whose
// exponents 2^{-s_local} stay small) join the rebased totals, the band depth joins Lb, and the band
// accumulators restart: no exponent ever exceeds a band's optical depth, so sum lam e^{+A} neither
// overflows nor loses the precision of a large fp32 depth (DESIGN.md R-depth).
__device__ __forceinline__ void fold_a(StateA& q)
{
    const float sb = q.s - q.sc;   // the band's depth (log2 units, <= 0)
    const float eb = ex2(sb);
    q.R1 = eb * (q.R1 + (q.p1 - q.p1c));
    q.R2 = eb * (q.R2 + (q.p2 - q.p2c));
    q.R3 = eb * (q.R3 + (q.p3 - q.p3c));
    kahan(q.Lb, q.Lbc, q.s);
    kahan(q.Lb, q.Lbc, -q.sc);
    q.s = q.sc = 0.f;
    q.p1 = q.p1c = q.p2 = q.p2c = q.p3 = q.p3c = 0.f;
}

// Sweep A: forward (+ JVP) recurrence, detector end first.
// PAIRED (line pairing): the same traversal also accumulates, for the ray of
// the opposite bank on the same line (detector at the other end, optical depth A'_i = S - A_i),
//   sum lam_i e^{A_i}                         (its forward:  e^{-S} * this),
//   sum dlam_i e^{A_i}, sum lam_i dA_i e^{A_i}  (GN: its JVP = e^{-S}(p1 - dS p2 + p3), dA' = dS - dA).
template <bool NF4>
struct SmpA {   // one sample of a ray in sweep A: its corners (prefetched) and fractions
    typename CornerT<NF4>::T c00, c01, c10, c11;
    float fu, fv;
};

// number of samples a walk takes inside one band: i, i-1, ... while i' >= ilo and the sample row stays in
// [r0, r1) (v_{i-k} = v - k dV; dV != 0 in the oriented frame) -- computed once per band so the sample
// loop tests a counter instead of three bounds
__device__ __forceinline__ int band_steps(int i, int ilo, int64_t v, int64_t dV, int r0, int r1)
{
    const int64_t num = dV > 0 ? v - (static_cast<int64_t>(r0) << 32)
                               : ((static_cast<int64_t>(r1) << 32) - 1) - v;   // >= 0: v is inside
    const int64_t adV = dV > 0 ? dV : -dV;
    // further steps inside = floor(num / |dV|): an fp32 estimate (relative error < 2^-21; a band is at most a
    // few hundred samples, so the estimate is within one of the quotient), fixed up exactly in 64-bit integers
    // -- the fp64 division it replaces was a ~45-instruction subroutine plus 64-bit int <-> double conversions
    // per band and lane; a 64-bit integer division is longer still
    float rcp;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rcp) : "f"(__ll2float_rn(adV)));
    int64_t k = static_cast<int64_t>(static_cast<int>(__ll2float_rn(num) * rcp));
    if ((k + 1) * adV <= num) ++k;
    else if (k * adV > num) --k;
    PGET_CHECK(k >= 0 && k * adV <= num && (k + 1) * adV > num);
    const int64_t n = i - ilo + 1;
    return static_cast<int>(k + 1 < n ? k + 1 : n);
}

// VAR (model variant N3, reading R-N3): cw is the lane's row [n_t] of (W_j(d_i), c_i); E_i = e^{-c_i A_i},
// the forward / JVP sums carry W_j(d_i), the adjoint's G carries W c (G_c = sum W lam c E).
template <int MODE, bool PAIRED, bool VAR = false>
__device__ __forceinline__ void walk_a(const unsigned char* __restrict__ sb, int Pb, int r0, int r1, int ilo,
                                       int64_t dU, int64_t dV, float cf, float ch, float dl, float dlh, int& i,
                                       int64_t& u, int64_t& v, StateA& st, const float2* __restrict__ cw = nullptr)
{
    using TR = ModeTraits<MODE>;
    using Cn = typename CornerT<TR::NF4>::T;
    const int iv0 = hi32(v);
    if (i < ilo || iv0 < r0 || iv0 >= r1) return;
    int n = band_steps(i, ilo, v, dV, r0, r1);
    // byte addressing from the band's origin (as the cached scatter's P4/planeB4): element (row iv, column iu) at
    // orgb + iv * Pb + iu * sizeof(Cn), Pb = P * sizeof(Cn) a constant-bank operand, the origin one opaque
    // register -- one IMAD (the FMA pipe, which bounds these kernels) per sample address instead of four
    constexpr int SH = TR::NF4 ? 4 : 3;
    static_assert(sizeof(Cn) == (1 << SH), "corner size");
    // the band's origin as a shared-space address in one opaque register (not re-associated, not recomputed
    // from the unit per sample); the loads are explicit ld.shared from 32-bit addresses
    const uint32_t sba = smem_u32(sb);
    uint32_t orga = sba - static_cast<uint32_t>(r0 * Pb);
    asm volatile("" : "+r"(orga));
    // ok false (the band's last sample has no successor here): load the band's first cell instead of branching
    // around the loads
    auto load = [&](SmpA<TR::NF4>& x, int64_t uu, int64_t vv, int ivv, bool ok = true) {
        uint32_t q = static_cast<uint32_t>(ivv * Pb) + orga;
        q += static_cast<uint32_t>(hi32r(uu)) << SH;
        q = ok ? q : sba;
        PGET_CHECK(q >= sba && (q - sba) + Pb + (1 << SH) < static_cast<uint32_t>((r1 - r0 + 1) * Pb));
        const uint32_t q1 = q + static_cast<uint32_t>(Pb);
        lds_c<0>(x.c00, q);
        lds_c<(1 << SH)>(x.c01, q);
        lds_c<0>(x.c10, q1);
        lds_c<(1 << SH)>(x.c11, q1);
        x.fu = frac23(uu);
        x.fv = frac23(vv);
    };
    StateA x_ = st;
    // sample i with corners cur; prefetch sample i-1 into nx; alternating roles (no register copies)
    auto step = [&](const SmpA<TR::NF4>& cur, SmpA<TR::NF4>& nx) -> bool {
        const int i2 = i - 1;
        const int64_t u2 = u - dU, v2 = v - dV;
        const int iv2 = hi32(v2);
        const bool nxt = --n != 0;
        load(nx, u2, v2, iv2, nxt);
        float lam, mu, dlam = 0.f, dmu = 0.f;
        if constexpr (TR::NF4) {
            const float2 x = bilerp2(lo2(cur.c00), lo2(cur.c01), lo2(cur.c10), lo2(cur.c11), cur.fu, cur.fv);
            const float2 y = bilerp2(hi2(cur.c00), hi2(cur.c01), hi2(cur.c10), hi2(cur.c11), cur.fu, cur.fv);
            lam = x.x; mu = x.y; dlam = y.x; dmu = y.y;
        } else {
            const float2 x = bilerp2(cur.c00, cur.c01, cur.c10, cur.c11, cur.fu, cur.fv);
            lam = x.x; mu = x.y;
        }
        float arg;   // -log2(e) A_i
        if constexpr (TR::COMP_S) {
            arg = fmaf(mu, ch, x_.s) - x_.sc;
            kahan(x_.s, x_.sc, mu * cf);
        } else {
            arg = fmaf(mu, ch, x_.s);
            x_.s = fmaf(mu, cf, x_.s);
        }
        float cv = 1.f, wv = 1.f;      // VAR: c_i, W_j(d_i)
        if constexpr (VAR) {
            const float2 t = __ldg(cw + i);
            wv = t.x;
            cv = t.y;
        }
        // exp(-c_i Delta(mu_i/2 + sum_{k>i} mu_k)); PAIRED: arg is band-local, Lb the depth before the band
        const float E = VAR ? ex2(cv * arg) : (PAIRED ? ex2(arg + x_.Lb) : ex2(arg));
        const float lg = VAR ? lam * (TR::HAS_B ? wv * cv : wv) : lam;
        if constexpr (TR::COMP_G) kahan(x_.g, x_.gc, lg * E);
        else x_.g = fmaf(lg, E, x_.g);
        float dA = 0.f;
        if constexpr (TR::NF4) {
            dA = fmaf(dmu, dlh, x_.ds);   // Delta (dmu_i/2 + sum_{k>i} dmu_k)
            const float jt = VAR ? wv * fmaf(-lam * cv, dA, dlam) : fmaf(-lam, dA, dlam);
            if constexpr (TR::COMP_J) kahan(x_.dg, x_.dgc, jt * E);
            else x_.dg = fmaf(jt, E, x_.dg);
            x_.ds = fmaf(dmu, dl, x_.ds);
        }
        if constexpr (PAIRED && (MODE == MODE_FWD || MODE == MODE_VJP)) {   // VJP: segmented phase A only
            x_.p2 = fmaf(lam, ex2(-arg), x_.p2);
        }
        if constexpr (PAIRED && MODE == MODE_GN) {
            const float eA = ex2(-arg);   // e^{A_i}
            const float le = lam * eA;
            x_.p1 = fmaf(dlam, eA, x_.p1);
            x_.p2 += le;
            x_.p3 = fmaf(le, dA, x_.p3);
        }
        i = i2;
        u = u2;
        v = v2;
        return nxt;
    };
    SmpA<TR::NF4> sa, sb2;
    load(sa, u, v, iv0);
    while (step(sa, sb2) && step(sb2, sa)) {
    }
    st = x_;
}

struct StateB {
    float s, sc, q, qc, q1, q1c;
};

struct RayB {   // per-ray constants of sweep B
    float kl, km, G, Gc;      // w_r Delta, -w_r Delta^2, G = sum lam E (compensated pair)
    float kl1, km1, Sl, Slc;  // PAIRED: the same for the opposite-bank ray; -log2(e) S (pair)
};

// Sweep B: per-sample adjoint weights scattered with the transposed bilinear weights into the warp's
// band accumulator (rows r0..r1; plain shared-memory read-modify-write: comb lanes never share a
// pixel).  The accumulator reads of sample i are issued first and the corner loads of sample i-1
// next, so both latencies overlap the arithmetic of sample i.
//   a_lam(i) = w_r Delta E_i,  a_mu(i) = -w_r Delta^2 (G - Q_i - lam_i E_i / 2),  Q_i = sum_{k>i} lam_k E_k
// PAIRED adds the opposite-bank ray of the same line (its detector at the low-i end):
//   E'_i = e^{-(S - A_i)},  a_lam += w'_r Delta E'_i,  a_mu += -w'_r Delta^2 (Q'_i + lam_i E'_i / 2),
//   Q'_i = sum_{k>i} lam_k E'_k  (samples farther from that detector, already visited).
#ifndef PGET_PF_DIST
#define PGET_PF_DIST 8   // samples between a cache entry's L2 prefetch and its use (4: +4 %, 16: +0.6 %, 32: +3 %, none: +3 % LM; scripts/pf_exp.sh)
#endif
#ifndef PGET_SCATTER
#define PGET_SCATTER 1
#endif
// PGET_SCATTER 1: the coefficients of consecutive samples in the same 2x2 cell are summed in
// registers and read-modify-written once when the ray leaves the cell (a cell spans ~1.5-2 samples):
// fewer shared-memory accesses, and those only by the lanes that change cell (bank-conflict bound
// since the segmented adjoint).  0: one read-modify-write per sample (prefetched accumulator reads).
// CACHE (the LM wrap's gradient VJP): rb holds the unit-weight constants; every sample's Jacobian
// entries (alpha, beta, alpha', beta') go to the lane's cache block (row k) and the scatter weights
// are w_r (alpha, beta) + w'_r (alpha', beta') -- the cache build of lin_kernel fused into the VJP.
// VAR (model variant N3): cw is the lane's row of (W_j(d_i), c_i): a_lam(i) = w_r Delta W_i E_i,
// a_mu(i) = -w_r Delta^2 (sum_{k<i} W_k lam_k c_k E_k + W_i lam_i c_i E_i / 2), E_i = e^{-c_i A_i}
template <bool PAIRED, bool COMP, bool CACHE = false, bool VAR = false>
__device__ __forceinline__ void walk_b_rolled(const float2* __restrict__ img, float2* __restrict__ acc, int P, int r0,
                                       int r1, int abase, int sP, int ilo, int64_t dU, int64_t dV, float cf, float ch,
                                       const RayB& rb, int& i, int64_t& u, int64_t& v, StateB& st,
                                       float wr = 0.f, float wr1 = 0.f, float4* cl = nullptr, int* kp = nullptr,
                                       float2* emax = nullptr, const float2* __restrict__ cw = nullptr)
{
    int iv = hi32(v), iu = hi32(u);
    if (i < ilo || iv < r0 || iv >= r1) return;
    int o = (iv - r0) * P + iu;
    float2 q00 = img[o], q01 = img[o + 1], q10 = img[o + P], q11 = img[o + P + 1];
    float fu = frac23(u), fv = frac23(v);
    StateB x_ = st;
#if PGET_SCATTER == 1
    int poff = -1;
    float2 p00 = make_float2(0.f, 0.f), p01 = p00, p10 = p00, p11 = p00;
#endif
    while (true) {
        // accumulator row of iv: abase + (iv - r0) * sP (sP = +-P, see the kernel), column iu
        PGET_CHECK(iu >= 0 && iu + 1 < P && iv >= r0 && iv < r1);
        const int aoff = abase + (iv - r0) * sP + iu;
#if PGET_SCATTER == 0
        float2* a0 = acc + aoff;
        const float2 t00 = a0[0], t01 = a0[1], t10 = a0[sP], t11 = a0[sP + 1];
#endif
        const int i2 = i - 1;
        const int64_t u2 = u - dU, v2 = v - dV;
        const int iv2 = hi32(v2);
        const bool nxt = i2 >= ilo && iv2 >= r0 && iv2 < r1;   // sweep-B bands are a few rows: no band_steps
        float2 n00, n01, n10, n11;
        // the band's last sample loads its own cell again instead of branching around the loads
        const int o2 = nxt ? (iv2 - r0) * P + hi32(u2) : o;
        PGET_CHECK(o2 >= 0 && o2 + P + 1 < (r1 - r0 + 1) * P);
        n00 = img[o2]; n01 = img[o2 + 1]; n10 = img[o2 + P]; n11 = img[o2 + P + 1];
        const float2 x = bilerp2(q00, q01, q10, q11, fu, fv);
        const float arg_hi = fmaf(x.y, ch, x_.s);
        float cv = 1.f, wv = 1.f;
        if constexpr (VAR) {
            const float2 t = __ldg(cw + i);
            wv = t.x;
            cv = t.y;
        }
        const float E = VAR ? ex2(cv * (arg_hi - x_.sc)) : ex2(arg_hi - x_.sc);
        const float le = VAR ? x.x * (wv * cv) * E : x.x * E;
        float al = VAR ? rb.kl * (wv * E) : rb.kl * E;
        float am = rb.km * (((rb.G - x_.q) - (rb.Gc - x_.qc)) - 0.5f * le);
        if constexpr (CACHE) {   // unit-weight entries: store, then weight
            float4 cv = make_float4(al, am, 0.f, 0.f);
            if constexpr (PAIRED) {
                const float E1 = ex2((rb.Sl - arg_hi) - (rb.Slc - x_.sc));
                const float le1 = x.x * E1;
                cv.z = rb.kl1 * E1;
                cv.w = rb.km1 * ((x_.q1 - x_.q1c) + 0.5f * le1);
                if (COMP) kahan(x_.q1, x_.q1c, le1);
                else x_.q1 += le1;
            }
            __stcs(cl + static_cast<int64_t>(*kp) * 32, cv);
            ++*kp;
            emax->x = fmaxf(emax->x, fmaxf(fabsf(cv.x), fabsf(cv.z)));   // magnitude bounds of the entries
            emax->y = fmaxf(emax->y, fmaxf(fabsf(cv.y), fabsf(cv.w)));   // (gnb_kernel's fixed-point scale)
            al = fmaf(wr, cv.x, wr1 * cv.z);
            am = fmaf(wr, cv.y, wr1 * cv.w);
        } else if constexpr (PAIRED) {
            const float E1 = ex2((rb.Sl - arg_hi) - (rb.Slc - x_.sc));   // e^{-(S - A_i)}
            const float le1 = x.x * E1;
            al = fmaf(rb.kl1, E1, al);
            am = fmaf(rb.km1, (x_.q1 - x_.q1c) + 0.5f * le1, am);
            if (COMP) kahan(x_.q1, x_.q1c, le1);
            else x_.q1 += le1;
        }
        if (COMP) {
            kahan(x_.q, x_.qc, le);
            kahan(x_.s, x_.sc, x.y * cf);
        } else {
            x_.q += le;
            x_.s = fmaf(x.y, cf, x_.s);
        }
        const float2 av = make_float2(al, am);
        const float2 tv = __fmul2_rn(av, make_float2(fv, fv));         // row j0+1
        const float2 bv = __ffma2_rn(tv, make_float2(-1.f, -1.f), av); // row j0
        const float2 c11 = __fmul2_rn(tv, make_float2(fu, fu));
        const float2 c10 = __ffma2_rn(c11, make_float2(-1.f, -1.f), tv);
        const float2 c01 = __fmul2_rn(bv, make_float2(fu, fu));
        const float2 c00 = __ffma2_rn(c01, make_float2(-1.f, -1.f), bv);
#if PGET_SCATTER == 0
        a0[0] = make_float2(t00.x + c00.x, t00.y + c00.y);
        a0[1] = make_float2(t01.x + c01.x, t01.y + c01.y);
        a0[sP] = make_float2(t10.x + c10.x, t10.y + c10.y);
        a0[sP + 1] = make_float2(t11.x + c11.x, t11.y + c11.y);
#else
        if (aoff != poff) {
            if (poff >= 0 && (PGET_ABLATE != 1 || p00.x == 12345.f)) {   // ABLATE 1: no scatter
                float2* pa = acc + poff;
                const float2 t00 = pa[0], t01 = pa[1], t10 = pa[sP], t11 = pa[sP + 1];
                pa[0] = make_float2(t00.x + p00.x, t00.y + p00.y);
                pa[1] = make_float2(t01.x + p01.x, t01.y + p01.y);
                pa[sP] = make_float2(t10.x + p10.x, t10.y + p10.y);
                pa[sP + 1] = make_float2(t11.x + p11.x, t11.y + p11.y);
            }
            poff = aoff;
            p00 = c00; p01 = c01; p10 = c10; p11 = c11;
        } else {
            p00.x += c00.x; p00.y += c00.y;
            p01.x += c01.x; p01.y += c01.y;
            p10.x += c10.x; p10.y += c10.y;
            p11.x += c11.x; p11.y += c11.y;
        }
#endif
        i = i2;
        u = u2;
        v = v2;
        if (!nxt) break;
        q00 = n00; q01 = n01; q10 = n10; q11 = n11;
        o = o2;
        iv = iv2;
        iu = hi32(u);
        fu = frac23(u);
        fv = frac23(v);
    }
#if PGET_SCATTER == 1
    {   // the last cell
        float2* pa = acc + poff;
        const float2 t00 = pa[0], t01 = pa[1], t10 = pa[sP], t11 = pa[sP + 1];
        pa[0] = make_float2(t00.x + p00.x, t00.y + p00.y);
        pa[1] = make_float2(t01.x + p01.x, t01.y + p01.y);
        pa[sP] = make_float2(t10.x + p10.x, t10.y + p10.y);
        pa[sP + 1] = make_float2(t11.x + p11.x, t11.y + p11.y);
    }
#endif
    st = x_;
}

// Sweep B, unrolled by two with alternating register roles (as walk_a: the corners of the next sample
// load into the other SmpB, no register rotation), the next sample's loads issued unconditionally,
// and the pending cell sums updated by one packed FMA per corner pair: p = p * keep + c (keep 0 when
// the lane enters a new cell, after the old cell's read-modify-write) -- bitwise the same sums as
// "p = c" / "p += c", without the copies a two-way join needs.
struct SmpB {
    float2 c00, c01, c10, c11;
    float fu, fv;
};
template <bool PAIRED, bool COMP, bool CACHE = false, bool VAR = false>
__device__ __forceinline__ void walk_b(const float2* __restrict__ img, float2* __restrict__ acc, int P, int r0,
                                       int r1, int abase, int sP, int ilo, int64_t dU, int64_t dV, float cf, float ch,
                                       const RayB& rb, int& i, int64_t& u, int64_t& v, StateB& st,
                                       float wr = 0.f, float wr1 = 0.f, float4* cl = nullptr, int* kp = nullptr,
                                       float2* emax = nullptr, const float2* __restrict__ cw = nullptr)
{
#if PGET_SCATTER == 0
    walk_b_rolled<PAIRED, COMP, CACHE, VAR>(img, acc, P, r0, r1, abase, sP, ilo, dU, dV, cf, ch, rb, i, u, v, st, wr, wr1,
                                         cl, kp, emax, cw);
#else
    if constexpr (!COMP) {   // the GN mode (plain sums) keeps the rolled loop: 128 registers and a spill unrolled
        walk_b_rolled<PAIRED, COMP, CACHE, VAR>(img, acc, P, r0, r1, abase, sP, ilo, dU, dV, cf, ch, rb, i, u, v, st, wr,
                                             wr1, cl, kp, emax, cw);
        return;
    }
    {
        const int iv = hi32(v);
        if (i < ilo || iv < r0 || iv >= r1) return;
    }
    auto load = [&](SmpB& x, int64_t uu, int64_t vv, bool ok) {
        int o = (hi32(vv) - r0) * P + hi32(uu);
        o = ok ? o : 0;   // the band's last sample: a valid cell instead of a branch around the loads
        PGET_CHECK(o >= 0 && o + P + 1 < (r1 - r0 + 1) * P);
        x.c00 = img[o]; x.c01 = img[o + 1]; x.c10 = img[o + P]; x.c11 = img[o + P + 1];
        x.fu = frac23(uu);
        x.fv = frac23(vv);
    };
    auto cell = [&](int64_t uu, int64_t vv) { return abase + (hi32(vv) - r0) * sP + hi32(uu); };
    StateB x_ = st;
    int poff = cell(u, v);   // the pending cell starts as the first sample's, with zero sums
    float2 p00 = make_float2(0.f, 0.f), p01 = p00, p10 = p00, p11 = p00;
    auto rmw = [&](int off) {
        float2* pa = acc + off;
        const float2 t00 = pa[0], t01 = pa[1], t10 = pa[sP], t11 = pa[sP + 1];
        pa[0] = __fadd2_rn(t00, p00);
        pa[1] = __fadd2_rn(t01, p01);
        pa[sP] = __fadd2_rn(t10, p10);
        pa[sP + 1] = __fadd2_rn(t11, p11);
    };
    auto step = [&](const SmpB& cur, SmpB& nx) -> bool {
        PGET_CHECK(hi32(u) >= 0 && hi32(u) + 1 < P && hi32(v) >= r0 && hi32(v) < r1);
        const int aoff = cell(u, v);
        const int i2 = i - 1;
        const int64_t u2 = u - dU, v2 = v - dV;
        const int iv2 = hi32(v2);
        const bool nxt = i2 >= ilo && iv2 >= r0 && iv2 < r1;   // sweep-B bands are a few rows: no band_steps
        load(nx, u2, v2, nxt);
        const float2 x = bilerp2(cur.c00, cur.c01, cur.c10, cur.c11, cur.fu, cur.fv);
        const float arg_hi = fmaf(x.y, ch, x_.s);
        float cv = 1.f, wv = 1.f;
        if constexpr (VAR) {
            const float2 t = __ldg(cw + i);
            wv = t.x;
            cv = t.y;
        }
        const float E = VAR ? ex2(cv * (arg_hi - x_.sc)) : ex2(arg_hi - x_.sc);
        const float le = VAR ? x.x * (wv * cv) * E : x.x * E;
        float al = VAR ? rb.kl * (wv * E) : rb.kl * E;
        float am = rb.km * (((rb.G - x_.q) - (rb.Gc - x_.qc)) - 0.5f * le);
        if constexpr (CACHE) {   // unit-weight entries: store, then weight
            float4 ce = make_float4(al, am, 0.f, 0.f);
            if constexpr (PAIRED) {
                const float E1 = ex2((rb.Sl - arg_hi) - (rb.Slc - x_.sc));
                const float le1 = x.x * E1;
                ce.z = rb.kl1 * E1;
                ce.w = rb.km1 * ((x_.q1 - x_.q1c) + 0.5f * le1);
                if (COMP) kahan(x_.q1, x_.q1c, le1);
                else x_.q1 += le1;
            }
            __stcs(cl + static_cast<int64_t>(*kp) * 32, ce);
            ++*kp;
            emax->x = fmaxf(emax->x, fmaxf(fabsf(ce.x), fabsf(ce.z)));   // magnitude bounds of the entries
            emax->y = fmaxf(emax->y, fmaxf(fabsf(ce.y), fabsf(ce.w)));   // (gnb_kernel's fixed-point scale)
            al = fmaf(wr, ce.x, wr1 * ce.z);
            am = fmaf(wr, ce.y, wr1 * ce.w);
        } else if constexpr (PAIRED) {
            const float E1 = ex2((rb.Sl - arg_hi) - (rb.Slc - x_.sc));   // e^{-(S - A_i)}
            const float le1 = x.x * E1;
            al = fmaf(rb.kl1, E1, al);
            am = fmaf(rb.km1, (x_.q1 - x_.q1c) + 0.5f * le1, am);
            if (COMP) kahan(x_.q1, x_.q1c, le1);
            else x_.q1 += le1;
        }
        if (COMP) {
            kahan(x_.q, x_.qc, le);
            kahan(x_.s, x_.sc, x.y * cf);
        } else {
            x_.q += le;
            x_.s = fmaf(x.y, cf, x_.s);
        }
        const float2 av = make_float2(al, am);
        const float2 tv = __fmul2_rn(av, make_float2(cur.fv, cur.fv));   // row j0+1
        const float2 bv = __ffma2_rn(tv, make_float2(-1.f, -1.f), av);   // row j0
        const float2 c11 = __fmul2_rn(tv, make_float2(cur.fu, cur.fu));
        const float2 c10 = __ffma2_rn(c11, make_float2(-1.f, -1.f), tv);
        const float2 c01 = __fmul2_rn(bv, make_float2(cur.fu, cur.fu));
        const float2 c00 = __ffma2_rn(c01, make_float2(-1.f, -1.f), bv);
        const bool chg = aoff != poff;
        if (chg) {
            if (PGET_ABLATE != 1 || p00.x == 12345.f) rmw(poff);   // ABLATE 1: no scatter
            poff = aoff;
        }
        const float kk = chg ? 0.f : 1.f;
        const float2 k2 = make_float2(kk, kk);
        p00 = __ffma2_rn(p00, k2, c00);
        p01 = __ffma2_rn(p01, k2, c01);
        p10 = __ffma2_rn(p10, k2, c10);
        p11 = __ffma2_rn(p11, k2, c11);
        i = i2;
        u = u2;
        v = v2;
        return nxt;
    };
    SmpB sa, sb;
    load(sa, u, v, true);
    while (step(sa, sb) && step(sb, sa)) {
    }
    rmw(poff);   // the last cell
    st = x_;
#endif
}

// ------------------------------------------------------------------------------------------ kernel
template <int MODE, int MAXG, bool PAIRED, bool VAR = false>
__global__ void __launch_bounds__(ModeTraits<MODE>::W * 32, ModeTraits<MODE>::MINB) proj_kernel(ProjArgs A)
{
    pdl_entry();
    using TR = ModeTraits<MODE>;
    const int W = blockDim.x >> 5;   // warps of this launch (<= TR::W, chosen per geometry: proj_cfg)
    const int NT = blockDim.x;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* mbar = reinterpret_cast<uint64_t*>(smem);
    unsigned char* const stage0 = smem + 128;   // stage buffer b at stage0 + b * stage_bytes
    float2* wacc_all = reinterpret_cast<float2*>(smem + A.off_wacc);
    float* rout = reinterpret_cast<float*>(smem + A.off_rout);      // [2R]
    float4* gsh = reinterpret_cast<float4*>(smem + A.off_gsh);      // [R] (G, Gc, Sl, Slc)

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int c = blockIdx.x;
    const int64_t t0 = A.cta_begin[c], t1 = A.cta_begin[c + 1];
    const int ns_task = A.passesA * A.nbA + (TR::HAS_B ? A.passesB * A.nbB : 0);
    const int64_t n_stages = (t1 - t0) * ns_task;
    if (n_stages == 0) return;

    const int P = A.P, R = A.R, J = A.J;
    const int RB1 = A.RbB + 1;
    float2* wacc = wacc_all + static_cast<size_t>(warp) * RB1 * P;
    if (TR::HAS_B) {
        float4* z = reinterpret_cast<float4*>(wacc_all);
        const int n4 = W * RB1 * P / 2;
        for (int k = tid; k < n4; k += NT) z[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    if (tid == 0) {
        mbar_init(&mbar[0], 1);
        mbar_init(&mbar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0) {
        issue_stage<MODE>(A, t0, ns_task, 0, stage0, &mbar[0]);
        if (n_stages > 1) issue_stage<MODE>(A, t0, ns_task, 1, stage0 + A.stage_bytes, &mbar[1]);
    }
    int64_t s = 0;   // global stage counter

    const float cf = A.cf, ch = A.ch, dl = A.delta, dlh = 0.5f * A.delta;

    for (int64_t t = t0; t < t1; ++t) {
        const TaskInfo ti = task_info(A, t);
        const RayP* rays = A.rays + static_cast<size_t>(ti.ab) * R;
        const int64_t dU = rays[0].dU, dV = rays[0].dV;
        const int dlo = ti.dlo, dhi = ti.dhi;
        const int prl = dlo * J, prh = dhi * J;   // rays of this task

        // ======================================================= sweep A: forward (+ JVP) recurrence
        // lanes own 32 adjacent rays (neighbouring lanes read neighbouring pixels: shared-memory broadcast)
        for (int pass = 0; pass < A.passesA; ++pass) {
            int rr[MAXG], ii[MAXG], ilo[MAXG];
            int64_t uu[MAXG], vv[MAXG];
            StateA st[MAXG];
            const float2* cwa[MAXG];
#pragma unroll
            for (int k = 0; k < MAXG; ++k) {
                const int r = prl + ((pass * MAXG + k) * W + warp) * 32 + lane;
                rr[k] = r < prh ? r : -1;
                cwa[k] = VAR && rr[k] >= 0 ? A.var_cw + static_cast<size_t>(rr[k] % J) * A.n_t : nullptr;
                ii[k] = -1; ilo[k] = 0; uu[k] = 0; vv[k] = 0;
                if (rr[k] >= 0) {
                    const RayP rp = rays[rr[k]];
                    ii[k] = rp.ihi; ilo[k] = rp.ilo;
                    uu[k] = rp.U0 + static_cast<int64_t>(rp.ihi) * dU;
                    vv[k] = rp.V0 + static_cast<int64_t>(rp.ihi) * dV;
                }
                st[k] = StateA{};
            }
            for (int kb = 0; kb < A.nbA; ++kb) {
                const int band = ti.dir > 0 ? A.nbA - 1 - kb : kb;
                int r0, r1;
                band_rows(band, A.RbA, P, r0, r1);
                const int b = static_cast<int>(s & 1);
                mbar_wait(&mbar[b], static_cast<uint32_t>((s >> 1) & 1));
                const unsigned char* sb = stage0 + b * A.stage_bytes;
#pragma unroll
                for (int k = 0; k < MAXG; ++k) {
                    walk_a<MODE, PAIRED, VAR>(sb, TR::NF4 ? A.P16 : A.P8, r0, r1, ilo[k], dU, dV, cf, ch, dl, dlh, ii[k], uu[k], vv[k], st[k],
                                              cwa[k]);
                    if (PAIRED) fold_a(st[k]);
                }
                __syncthreads();   // stage buffer b consumed
                if (tid == 0 && s + 2 < n_stages) issue_stage<MODE>(A, t0, ns_task, s + 2, stage0 + b * A.stage_bytes, &mbar[b]);
                ++s;
            }
            // per-ray results of this pass
#pragma unroll
            for (int k = 0; k < MAXG; ++k) {
                const int r = rr[k];
                if (r < 0) continue;
                const StateA& q = st[k];
                if (MODE == MODE_FWD) {
                    rout[r] = A.delta * q.g;
                    if (PAIRED) rout[R + r] = A.delta * q.R2;   // e^{-S} sum lam e^{A} (rebased, fold_a)
                }
                if (MODE == MODE_JVP) { rout[r] = A.delta * q.g; rout[R + r] = A.delta * (q.dg - q.dgc); }
                if (MODE == MODE_VJP || MODE == MODE_GN)
                    gsh[r] = PAIRED ? make_float4(q.g, q.gc, q.Lb, q.Lbc) : make_float4(q.g, q.gc, q.s, q.sc);
                if (MODE == MODE_GN) {
                    rout[r] = A.delta * (q.dg - q.dgc);
                    if (PAIRED)   // opposite bank: e^{-S} (sum dlam e^A - dS sum lam e^A + sum lam dA e^A)
                        rout[R + r] = A.delta * ((q.R1 + q.R3) - q.ds * q.R2);
                }
            }
        }
        __syncthreads();

        if (!TR::HAS_B) {
            // sub-ray weighting and coalesced sinogram store
            const size_t obase = (static_cast<size_t>(ti.m) * A.n_ab + ti.ab) * A.n_det;
            const size_t obase2 = (static_cast<size_t>(ti.m) * A.n_ab + dup_of(A, ti.ab)) * A.n_det;
            const size_t pbase = (static_cast<size_t>(ti.m) * A.n_ab + ti.ab + 1) * A.n_det;       // bank 1
            const size_t pbase2 = (static_cast<size_t>(ti.m) * A.n_ab + dup_of(A, ti.ab + 1)) * A.n_det;
            for (int d = dlo + tid; d < dhi; d += NT) {
                float acc = 0.f, dacc = 0.f;
                for (int j = 0; j < J; ++j) {
                    const float wj = A.w[j];
                    acc = fmaf(wj, rout[d * J + j], acc);
                    if (MODE == MODE_JVP || PAIRED) dacc = fmaf(wj, rout[R + d * J + j], dacc);
                }
                if (MODE == MODE_JVP) {
                    if (A.y) A.y[obase + d] = acc;
                    A.dy[obase + d] = dacc;
                    if (A.dup_half) {   // the duplicate angle-bank measures the same rays
                        if (A.y) A.y[obase2 + d] = acc;
                        A.dy[obase2 + d] = dacc;
                    }
                } else {
                    A.y[obase + d] = acc;
                    if (A.dup_half) A.y[obase2 + d] = acc;
                    if (PAIRED) {   // bank 1, detector n-1-d: the same line traversed towards the other end
                        const int dd = A.n_det - 1 - d;
                        A.y[pbase + dd] = dacc;
                        A.y[pbase2 + dd] = dacc;
                    }
                }
            }
            continue;   // rout is rewritten only after the next task's first band barrier
        }

        // ======================================================= sweep B: adjoint scatter (VJP / GN)
        const size_t wbase = (static_cast<size_t>(ti.m) * A.n_ab + ti.ab) * A.n_det;
        const size_t wbase2 = (static_cast<size_t>(ti.m) * A.n_ab + dup_of(A, ti.ab)) * A.n_det;
        const size_t wpbase = (static_cast<size_t>(ti.m) * A.n_ab + ti.ab + 1) * A.n_det;   // PAIRED: bank 1
        const size_t wpbase2 = (static_cast<size_t>(ti.m) * A.n_ab + dup_of(A, ti.ab + 1)) * A.n_det;
        float2* slot = A.slots + static_cast<size_t>(ti.slot) * A.N * A.Ns;
        const int npairs = P >> 1;
        const float inv_np = 1.0f / static_cast<float>(npairs);
        // columns the task's rays can touch in a band of rows [v0, v1] (oriented frame): between the
        // lines of its first and last ray; the band flush reads and clears only those (a detector
        // range of an angle-bank flushes its share of the image, not all of it)
        const RayP rfirst = rays[prl], rlast = rays[prh - 1];
        const double kuv = static_cast<double>(dU) / static_cast<double>(dV);
        auto ucol = [&](const RayP& rp, double vrow) {
            return (static_cast<double>(rp.U0) + (vrow * 4294967296.0 - static_cast<double>(rp.V0)) * kuv) *
                   (1.0 / 4294967296.0);
        };
        for (int pass = 0; pass < A.passesB; ++pass) {
            int ii[MAXG], ilo[MAXG];
            int64_t uu[MAXG], vv[MAXG];
            RayB rb[MAXG];
            StateB st[MAXG];
            const float2* cwb[MAXG];
#pragma unroll
            for (int k = 0; k < MAXG; ++k) {
                const int grp = ti.gbeg + (pass * MAXG + k) * W + warp;
                const int r = grp < ti.gend ? A.groups[grp * 32 + lane] : -1;
                cwb[k] = VAR && r >= 0 ? A.var_cw + static_cast<size_t>(r % J) * A.n_t : nullptr;
                ii[k] = -1; ilo[k] = 0; uu[k] = 0; vv[k] = 0;
                rb[k] = RayB{0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
                st[k] = StateB{0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
                if (r >= 0) {
                    const int d = r / J, j = r - d * J;
                    float wd = 0.f, wd1 = 0.f;
                    if (MODE == MODE_GN) {
                        for (int jj = 0; jj < J; ++jj) {
                            wd = fmaf(A.w[jj], rout[d * J + jj], wd);
                            if (PAIRED) wd1 = fmaf(A.w[jj], rout[R + d * J + jj], wd1);
                        }
                        if (A.dup_half) { wd *= 2.f; wd1 *= 2.f; }   // (J p) of the duplicate rays is the same
                    } else {
                        wd = A.win[wbase + d];
                        if (A.dup_half) wd += A.win[wbase2 + d];
                        if (PAIRED) wd1 = A.win[wpbase + A.n_det - 1 - d] + A.win[wpbase2 + A.n_det - 1 - d];
                    }
                    const float wr = A.w[j] * wd, wr1 = A.w[j] * wd1;   // w_{J-1-j} = w_j
                    const float4 G = gsh[r];
                    rb[k] = RayB{wr * A.delta, -wr * A.delta * A.delta, G.x, G.y,
                                 wr1 * A.delta, -wr1 * A.delta * A.delta, G.z, G.w};
                    if (wr != 0.f || wr1 != 0.f) {
                        const RayP rp = rays[r];
                        ii[k] = rp.ihi; ilo[k] = rp.ilo;
                        uu[k] = rp.U0 + static_cast<int64_t>(rp.ihi) * dU;
                        vv[k] = rp.V0 + static_cast<int64_t>(rp.ihi) * dV;
                    }
                }
            }
            for (int kb = 0; kb < A.nbB; ++kb) {
                const int band = ti.dir > 0 ? A.nbB - 1 - kb : kb;
                int r0, r1;
                band_rows(band, A.RbB, P, r0, r1);
                const int b = static_cast<int>(s & 1);
                mbar_wait(&mbar[b], static_cast<uint32_t>((s >> 1) & 1));
                const float2* sb = reinterpret_cast<const float2*>(stage0 + b * A.stage_bytes);
                // accumulator rows flip direction every band (even kb: local row r - r0; odd kb:
                // r0 + RbB - r), so the row shared with the next band keeps its local row: no wrap, no copy
                const bool flip = kb & 1;
                const int abase = flip ? A.RbB * P : 0, sP = flip ? -P : P;
#pragma unroll
                for (int k = 0; k < MAXG; ++k)
                    walk_b<PAIRED, TR::COMP_S, false, VAR>(sb, wacc, P, r0, r1, abase, sP, ilo[k], dU, dV, cf, ch, rb[k],
                                                           ii[k], uu[k], vv[k], st[k], 0.f, 0.f, nullptr, nullptr,
                                                           nullptr, cwb[k]);
                __syncthreads();   // stage buffer b and every warp ring consumed
                if (tid == 0 && s + 2 < n_stages) issue_stage<MODE>(A, t0, ns_task, s + 2, stage0 + b * A.stage_bytes, &mbar[b]);
                ++s;
                // flush the finished rows of the band (all rows on the pass's last band; otherwise all but
                // the row shared with the next band in processing order) into the CTA's partial slot.
                // Element (row, pair) is always handled by thread (row * npairs + pair) % NT, so successive
                // flushes of one slot element are issued by one thread in program order: deterministic.
                const bool last = kb == A.nbB - 1;
                const int carry = last ? -1 : (ti.dir > 0 ? r0 : r1);
                const bool store = ti.first && pass == 0;   // the slot's first writer covers every column
                int qlo = 0, qhi = npairs - 1;
                if (!store) {
                    const double a0 = ucol(rfirst, r0 - 1.0), a1 = ucol(rfirst, r1 + 1.0);
                    const double b0 = ucol(rlast, r0 - 1.0), b1 = ucol(rlast, r1 + 1.0);
                    const double umin = fmin(fmin(a0, a1), fmin(b0, b1)), umax = fmax(fmax(a0, a1), fmax(b0, b1));
                    qlo = max(0, static_cast<int>(floor(umin)) - 2) >> 1;
                    qhi = min(P - 1, static_cast<int>(floor(umax)) + 3) >> 1;
                }
                // flat element index e = r * npairs + q over the band's rows; thread tid takes e = tid (mod NT)
                const int e_beg = r0 * npairs, e_end = (r1 + 1) * npairs;
                for (int e = e_beg + (tid - e_beg % NT + NT) % NT; e < e_end; e += NT) {
                    int r = __float2int_rd(static_cast<float>(e) * inv_np);
                    int q = e - r * npairs;
                    if (q < 0) { --r; q += npairs; } else if (q >= npairs) { ++r; q -= npairs; }
                    if (r == carry || q < qlo || q > qhi || PGET_ABLATE == 2) continue;
                    const int lr = flip ? r0 + A.RbB - r : r - r0;
                    PGET_CHECK(lr >= 0 && lr < RB1);
                    float4 sum = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
                    for (int w = 0; w < W; ++w) {
                        float4* el = reinterpret_cast<float4*>(wacc_all + (static_cast<size_t>(w) * RB1 + lr) * P) + q;
                        const float4 x = *el;
                        sum.x += x.x; sum.y += x.y; sum.z += x.z; sum.w += x.w;
                        *el = make_float4(0.f, 0.f, 0.f, 0.f);
                    }
                    const int ir = r - kHalo, ic = 2 * q - kHalo;
                    if (ir >= 0 && ir < A.N && ic >= 0 && ic < A.Ns) {
                        float4* dst = reinterpret_cast<float4*>(slot + static_cast<size_t>(ir) * A.Ns + ic);
                        if (store) *dst = sum;
                        else atomicAdd(dst, sum);
                    }
                }
                __syncthreads();   // rings zeroed before the next band's scatter
            }
        }
        // gsh / rout reuse by the next task happens after at least one more barrier
    }
}

// ------------------------------------------------------------------------------------------ segmented adjoint
// The adjoint (VJP, GN) as two launches over units (member, traced angle-bank, row segment k of K)
// with all detectors.  Along a ray walked from its bank-0 detector
// the segments come in the order q = 0..K-1 (q = seg for dV < 0, K-1-seg for dV > 0).  Phase A
// evaluates, per ray and segment, the local sums that the whole-ray recurrences split into
// (log2-domain optical depth L_q of the segment, G_q = sum lam e^{-A_loc}, and for GN the JVP sums);
// phase B rebuilds from the K partials of its ray
//   scale  = e^{-(depth before the segment)},  T = tail of G from the segment on, in the segment's
//   frame,  the reverse-direction offsets,  and (GN) the whole-ray (J p) of both directions,
// then scatters the segment's adjoint exactly as sweep B of proj_kernel with those constants.
struct UnitInfo {
    int m, ab, seg, canon, slot, cls, first, dir, ylo, yhi, nb;
};

__device__ __forceinline__ UnitInfo unit_info(const ProjArgs& A, int u, int Rb)
{
    const UnitD ud = A.units[u];
    UnitInfo x;
    x.m = ud.m;
    x.ab = ud.ab;
    x.seg = ud.seg;
    x.canon = ud.canon;
    x.slot = ud.slot;
    x.cls = (ud.flags & kTaskClass1) ? 1 : 0;
    x.first = (ud.flags & kTaskFirst) ? 1 : 0;
    x.dir = A.rays[static_cast<size_t>(ud.ab) * A.R].dV > 0 ? 1 : -1;
    x.ylo = A.seg_rows[ud.seg];
    x.yhi = A.seg_rows[ud.seg + 1];
    x.nb = (x.yhi - x.ylo + Rb - 1) / Rb;
    return x;
}

// rows of band j (processing order) of a unit: sample rows [r0, r1), staged rows r0..r1
__device__ __forceinline__ void seg_band(const UnitInfo& ui, int j, int Rb, int& r0, int& r1)
{
    const int b = ui.dir > 0 ? ui.nb - 1 - j : j;
    r0 = ui.ylo + b * Rb;
    r1 = min(r0 + Rb, ui.yhi);
}

template <bool F4>
__device__ void issue_seg_stage(const ProjArgs& A, int Rb, int64_t sidx, void* dst, uint64_t* bar)
{
    const StageD sd = A.stages[sidx];
    const UnitInfo ui = unit_info(A, sd.unit, Rb);
    int r0, r1;
    seg_band(ui, sd.j, Rb, r0, r1);
    const size_t pix0 = static_cast<size_t>(ui.m) * A.P * A.P + static_cast<size_t>(r0) * A.P;
    const size_t npix = static_cast<size_t>(r1 - r0 + 1) * A.P;
    const char* src = F4 ? reinterpret_cast<const char*>(A.img4[ui.cls] + pix0)
                         : reinterpret_cast<const char*>(A.img2[ui.cls] + pix0);
    const size_t bytes = npix * (F4 ? sizeof(float4) : sizeof(float2));
    fence_proxy_async();
    mbar_expect_tx(bar, static_cast<uint32_t>(bytes));
    char* d = static_cast<char*>(dst);
    for (size_t off = 0; off < bytes; off += 32768) {
        const uint32_t n = static_cast<uint32_t>(bytes - off < 32768 ? bytes - off : 32768);
        bulk_g2s(d + off, src + off, n, bar);
    }
}

// Phase A: sweep A of every ray of the CTA's units through the unit's rows; per-ray partials to A.segp.
// Warp-specialised pipeline: the last warp only issues the stage copies (kSegAStages buffers, a
// "full" mbarrier per buffer completed by the copy's bytes, an "empty" mbarrier per buffer on which
// every consumer warp arrives when done with it), so consumer warps never wait for one another.


// WIDE: up to 26 consumer warps (one 32-ray group each, configs 3-4) at <= 72 registers; else <= 15
template <int MODE, int MAXG, bool PAIRED, bool WIDE = false>
__global__ void __launch_bounds__(WIDE ? 864 : 512, 1) seg_a_kernel(ProjArgs A)   // W consumer warps + 1 producer warp
{
    pdl_entry();
    using TR = ModeTraits<MODE>;
    const int W = (blockDim.x >> 5) - 1;   // consumer warps
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + kSegAStages;
    unsigned char* const stage0 = smem + 128;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int c = blockIdx.x;
    const int64_t sb0 = A.s_begin[c];
    const int64_t n_stages = A.s_begin[c + 1] - sb0;
    if (n_stages == 0) return;
    const int R = A.R, Rb = A.RbA;
    if (tid == 0) {
        for (int b = 0; b < kSegAStages; ++b) {
            mbar_init(&full[b], 1);
            mbar_init(&empty[b], W);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == W) {   // producer
        if (lane == 0)
            for (int64_t s = 0; s < n_stages; ++s) {
                const int b = static_cast<int>(s % kSegAStages);
                if (s >= kSegAStages) mbar_wait(&empty[b], static_cast<uint32_t>((s / kSegAStages - 1) & 1));
                issue_seg_stage<TR::NF4>(A, Rb, sb0 + s, stage0 + b * A.stage_bytes, &full[b]);
            }
        return;
    }
    int64_t s = 0;
    const float cf = A.cf, ch = A.ch, dl = A.delta, dlh = 0.5f * A.delta;
    for (int u = A.u_begin[c]; u < A.u_begin[c + 1]; ++u) {
        const UnitInfo ui = unit_info(A, u, Rb);
        const RayP* rays = A.rays + static_cast<size_t>(ui.ab) * R;
        const int64_t dU = rays[0].dU, dV = rays[0].dV;
        const int bound = ui.dir > 0 ? ui.yhi : ui.ylo;
        float* part = A.segp + static_cast<size_t>(ui.canon) * kSegFields * R;
        for (int pass = 0; pass < A.passesA; ++pass) {
            int rr[MAXG], ii[MAXG], ilo[MAXG];
            int64_t uu[MAXG], vv[MAXG];
            StateA st[MAXG];
#pragma unroll
            for (int k = 0; k < MAXG; ++k) {
                const int r = ((pass * MAXG + k) * W + warp) * 32 + lane;
                rr[k] = r < R ? r : -1;
                ii[k] = -1; ilo[k] = 0; uu[k] = 0; vv[k] = 0;
                if (rr[k] >= 0) {
                    const RayP rp = rays[r];
                    ii[k] = seg_entry(rp, bound);
                    ilo[k] = rp.ilo;
                    uu[k] = rp.U0 + static_cast<int64_t>(ii[k]) * dU;
                    vv[k] = rp.V0 + static_cast<int64_t>(ii[k]) * dV;
                }
                st[k] = StateA{};
            }
            for (int j = 0; j < ui.nb; ++j) {
                int r0, r1;
                seg_band(ui, j, Rb, r0, r1);
                const int b = static_cast<int>(s % kSegAStages);
                mbar_wait(&full[b], static_cast<uint32_t>((s / kSegAStages) & 1));
                const unsigned char* sbuf = stage0 + b * A.stage_bytes;
#pragma unroll
                for (int k = 0; k < MAXG; ++k) {
                    walk_a<MODE, PAIRED>(sbuf, TR::NF4 ? A.P16 : A.P8, r0, r1, ilo[k], dU, dV, cf, ch, dl, dlh, ii[k], uu[k], vv[k], st[k]);
                    if (PAIRED) fold_a(st[k]);
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[b]);   // this warp is done with buffer b
                ++s;
            }
#pragma unroll
            for (int k = 0; k < MAXG; ++k) {
                const int r = rr[k];
                if (r < 0) continue;
                const StateA& q = st[k];
                // PAIRED: the unit's depth is Lb (every band folded) and the reverse-direction sums are
                // rebased to the unit's end (R_k = 2^{s_unit} p_k): the combines scale them by
                // 2^{-(depth after the unit)}
                part[0 * R + r] = PAIRED ? q.Lb : q.s;
                part[1 * R + r] = PAIRED ? q.Lbc : q.sc;
                part[2 * R + r] = q.g;
                part[3 * R + r] = q.gc;
                if (MODE == MODE_GN) {
                    part[4 * R + r] = q.ds;
                    part[5 * R + r] = q.dg - q.dgc;
                    part[6 * R + r] = PAIRED ? q.R1 : q.p1;
                    part[8 * R + r] = PAIRED ? q.R3 : q.p3;
                }
                if (MODE == MODE_JVP) {   // the compensated JVP sum kept as its pair
                    part[4 * R + r] = q.ds;
                    part[5 * R + r] = q.dg;
                    part[6 * R + r] = q.dgc;
                }
                if (PAIRED) part[7 * R + r] = q.R2;
            }
        }
    }
}

// Segmented standalone JVP: y and dy of every ray from its K phase-A segment partials (fp64, in ray
// order), then the sub-ray weighting and the sinogram stores (duplicate angle-banks too).  Block
// (t, m): traced angle-bank t of member m.
__global__ void __launch_bounds__(256) jvp_combine_kernel(ProjArgs A, const int32_t* __restrict__ tabs, int ntab)
{
    pdl_entry();
    extern __shared__ __align__(128) unsigned char smem[];
    float* ry = reinterpret_cast<float*>(smem);          // [R]
    float* rdy = ry + A.R;                                // [R]
    const int t = blockIdx.x, m = blockIdx.y;
    const int R = A.R, J = A.J, K = A.K;
    const int ab = tabs[t];
    const int dir = A.rays[static_cast<size_t>(ab) * R].dV > 0 ? 1 : -1;
    const float* part0 = A.segp + static_cast<size_t>((m * ntab + t) * K) * kSegFields * R;
    for (int r = threadIdx.x; r < R; r += blockDim.x) {
        double L = 0.0, dL = 0.0, y = 0.0, dy = 0.0;
        for (int q = 0; q < K; ++q) {
            const float* pq = part0 + static_cast<size_t>(dir > 0 ? K - 1 - q : q) * kSegFields * R;
            const double e = exp2(L);
            const double gq = static_cast<double>(pq[2 * R + r]) - pq[3 * R + r];
            const double dgq = static_cast<double>(pq[5 * R + r]) - pq[6 * R + r];
            y += e * gq;
            dy += e * (dgq - dL * gq);
            L += static_cast<double>(pq[0 * R + r]) - pq[1 * R + r];
            dL += pq[4 * R + r];
        }
        ry[r] = static_cast<float>(A.delta * y);
        rdy[r] = static_cast<float>(A.delta * dy);
    }
    __syncthreads();
    const size_t obase = (static_cast<size_t>(m) * A.n_ab + ab) * A.n_det;
    const size_t obase2 = (static_cast<size_t>(m) * A.n_ab + dup_of(A, ab)) * A.n_det;
    for (int d = threadIdx.x; d < A.n_det; d += blockDim.x) {
        float acc = 0.f, dacc = 0.f;
        for (int j = 0; j < J; ++j) {
            acc = fmaf(A.w[j], ry[d * J + j], acc);
            dacc = fmaf(A.w[j], rdy[d * J + j], dacc);
        }
        if (A.y) A.y[obase + d] = acc;
        A.dy[obase + d] = dacc;
        if (A.dup_half) {
            if (A.y) A.y[obase2 + d] = acc;
            A.dy[obase2 + d] = dacc;
        }
    }
}

// Segmented forward: y of both banks of every line from the VJP-mode phase-A partials of the
// (paired when possible) adjoint schedule: bank 0 G = sum_q 2^{L_q} G_q; bank 1 (the same line
// walked from the other end) e^{-S} sum_q 2^{-L_q} p2_q; duplicate angle-banks too.
template <bool PAIRED>
__global__ void __launch_bounds__(256) fwd_combine_kernel(ProjArgs A, const int32_t* __restrict__ tabs, int ntab)
{
    pdl_entry();
    extern __shared__ __align__(128) unsigned char smem[];
    float* ry = reinterpret_cast<float*>(smem);   // [2R]
    const int t = blockIdx.x, m = blockIdx.y;
    const int R = A.R, J = A.J, K = A.K;
    const int ab = tabs[t];
    const int dir = A.rays[static_cast<size_t>(ab) * R].dV > 0 ? 1 : -1;
    const float* part0 = A.segp + static_cast<size_t>((m * ntab + t) * K) * kSegFields * R;
    for (int r = threadIdx.x; r < R; r += blockDim.x) {
        double L = 0.0, y = 0.0, p2 = 0.0;
        for (int q = 0; q < K; ++q) {
            const float* pq = part0 + static_cast<size_t>(dir > 0 ? K - 1 - q : q) * kSegFields * R;
            y += exp2(L) * (static_cast<double>(pq[2 * R + r]) - pq[3 * R + r]);
            L += static_cast<double>(pq[0 * R + r]) - pq[1 * R + r];
            if (PAIRED) p2 += exp2(-L) * pq[7 * R + r];   // rebased to the unit's end (seg_a_kernel)
        }
        ry[r] = static_cast<float>(A.delta * y);
        if (PAIRED) ry[R + r] = static_cast<float>(A.delta * exp2(L) * p2);
    }
    __syncthreads();
    const size_t obase = (static_cast<size_t>(m) * A.n_ab + ab) * A.n_det;
    const size_t obase2 = (static_cast<size_t>(m) * A.n_ab + dup_of(A, ab)) * A.n_det;
    const size_t pbase = (static_cast<size_t>(m) * A.n_ab + ab + 1) * A.n_det;
    const size_t pbase2 = (static_cast<size_t>(m) * A.n_ab + dup_of(A, ab + 1)) * A.n_det;
    for (int d = threadIdx.x; d < A.n_det; d += blockDim.x) {
        float acc = 0.f, acc1 = 0.f;
        for (int j = 0; j < J; ++j) {
            acc = fmaf(A.w[j], ry[d * J + j], acc);
            if (PAIRED) acc1 = fmaf(A.w[j], ry[R + d * J + j], acc1);
        }
        A.y[obase + d] = acc;
        if (A.dup_half) A.y[obase2 + d] = acc;
        if (PAIRED) {   // bank 1, detector n-1-d
            const int dd = A.n_det - 1 - d;
            A.y[pbase + dd] = acc1;
            A.y[pbase2 + dd] = acc1;
        }
    }
}

cudaError_t launch_fwd_combine(bool paired, const ProjArgs& A, const int32_t* tabs, int ntab, int B, cudaStream_t s)
{
    if (paired) launch_k(fwd_combine_kernel<true>, dim3(ntab, B), 256, 2 * A.R * sizeof(float), s, A, tabs, ntab);
    else launch_k(fwd_combine_kernel<false>, dim3(ntab, B), 256, 2 * A.R * sizeof(float), s, A, tabs, ntab);
    return cudaGetLastError();
}

cudaError_t launch_jvp_combine(const ProjArgs& A, const int32_t* tabs, int ntab, int B, cudaStream_t s)
{
    launch_k(jvp_combine_kernel, dim3(ntab, B), 256, 2 * A.R * sizeof(float), s, A, tabs, ntab);
    return cudaGetLastError();
}

// Phase B: per-ray constants from the K partials, then sweep B of the unit (comb groups) into the
// unit's partial slot (zeroed by the slot's first unit; every flush adds).
__device__ __forceinline__ float4* cache_lane(const ProjArgs& A, const UnitInfo& ui, int grp, int lane, int* kend);

// the cache builders' magnitude bounds of the entries, per (member, traced angle-bank):
// gscale[ct * 8 + 0] = max |alpha|, |alpha'|; [1] = max |beta|, |beta'| (float bits, atomicMax of
// non-negative floats; zeroed before the build).  Warp-uniform call.
__device__ __forceinline__ void entry_bounds(const ProjArgs& A, const UnitInfo& ui, float2 am)
{
    if (!A.gscale) return;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        am.x = fmaxf(am.x, __shfl_xor_sync(0xffffffffu, am.x, o));
        am.y = fmaxf(am.y, __shfl_xor_sync(0xffffffffu, am.y, o));
    }
    if ((threadIdx.x & 31) == 0) {
        int* gs = reinterpret_cast<int*>(A.gscale + static_cast<size_t>((ui.canon - ui.seg) / A.K) * 8);
        atomicMax(gs, __float_as_int(am.x));
        atomicMax(gs + 1, __float_as_int(am.y));
    }
}

template <int MODE, bool PAIRED, bool CACHE>
__global__ void __launch_bounds__(512, 1) seg_b_kernel(ProjArgs A)
{
    pdl_entry();
    const int W = blockDim.x >> 5;
    const int NT = blockDim.x;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* mbar = reinterpret_cast<uint64_t*>(smem);
    unsigned char* const stage0 = smem + 128;
    float2* wacc_all = reinterpret_cast<float2*>(smem + A.off_wacc);
    float* rout = reinterpret_cast<float*>(smem + A.off_rout);      // [2R] (GN: J p of both directions)
    float4* gsh = reinterpret_cast<float4*>(smem + A.off_gsh);      // [R] (T, Tc, Sl, Slc)
    float* rsc = reinterpret_cast<float*>(smem + A.off_rsc);        // [R] e^{-depth before the segment}
    float2* q1i = reinterpret_cast<float2*>(smem + A.off_q1);       // [R] reverse-direction Q offset (pair)

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int c = blockIdx.x;
    const int64_t sb0 = A.s_begin[c];
    const int64_t n_stages = A.s_begin[c + 1] - sb0;
    if (n_stages == 0) return;
    const int P = A.P, R = A.R, J = A.J, K = A.K, Rb = A.RbB;
    const int RB1 = Rb + 1;
    float2* wacc = wacc_all + static_cast<size_t>(warp) * RB1 * P;
    {
        float4* z = reinterpret_cast<float4*>(wacc_all);
        const int n4 = W * RB1 * P / 2;
        for (int k = tid; k < n4; k += NT) z[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    if (tid == 0) {
        mbar_init(&mbar[0], 1);
        mbar_init(&mbar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0) {
        issue_seg_stage<false>(A, Rb, sb0, stage0, &mbar[0]);
        if (n_stages > 1) issue_seg_stage<false>(A, Rb, sb0 + 1, stage0 + A.stage_bytes, &mbar[1]);
    }
    int64_t s = 0;
    const float cf = A.cf, ch = A.ch;
    const int npairs = P >> 1;
    const float inv_np = 1.0f / static_cast<float>(npairs);
    const size_t plane = static_cast<size_t>(A.N) * A.Ns;

    for (int u = A.u_begin[c]; u < A.u_begin[c + 1]; ++u) {
        const UnitInfo ui = unit_info(A, u, Rb);
        const RayP* rays = A.rays + static_cast<size_t>(ui.ab) * R;
        const int64_t dU = rays[0].dU, dV = rays[0].dV;
        const int bound = ui.dir > 0 ? ui.yhi : ui.ylo;
        const int qme = ui.dir > 0 ? K - 1 - ui.seg : ui.seg;
        const float* part0 = A.segp + static_cast<size_t>(ui.canon - ui.seg) * kSegFields * R;
        // ---- per-ray constants (fp64 combination of the K segment partials, in ray order)
        for (int r = tid; r < R; r += NT) {
            // fixed-size, fully unrolled (K <= 4): register-resident
            double Lb[5], dLb[5], gq[4], p1q[4], p2q[4], p3q[4], dgq[4];
            Lb[0] = 0.0;
            dLb[0] = 0.0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                gq[q] = p1q[q] = p2q[q] = p3q[q] = dgq[q] = 0.0;
                double sq = 0.0, dsq = 0.0;
                if (q < K) {
                    const float* pq = part0 + static_cast<size_t>(ui.dir > 0 ? K - 1 - q : q) * kSegFields * R;
                    sq = static_cast<double>(pq[0 * R + r]) - pq[1 * R + r];
                    gq[q] = static_cast<double>(pq[2 * R + r]) - pq[3 * R + r];
                    if (PAIRED) p2q[q] = pq[7 * R + r];
                    if (MODE == MODE_GN) {
                        dsq = pq[4 * R + r];
                        dgq[q] = pq[5 * R + r];
                        p1q[q] = pq[6 * R + r];
                        p3q[q] = pq[8 * R + r];
                    }
                }
                Lb[q + 1] = Lb[q] + sq;
                dLb[q + 1] = dLb[q] + dsq;
            }
            double Lme = 0.0, LK = 0.0, dLK = 0.0;
#pragma unroll
            for (int q = 0; q < 5; ++q) {
                if (q == qme) Lme = Lb[q];
                if (q == K) { LK = Lb[q]; dLK = dLb[q]; }
            }
            double T = 0.0, Qoff = 0.0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if (q >= qme && q < K) T += exp2(Lb[q] - Lme) * gq[q];
                if (PAIRED && q < qme) Qoff += exp2(LK - Lb[q + 1]) * p2q[q];   // rebased R2
            }
            const double Sl = LK - Lme;
            const float Th = static_cast<float>(T), Sh = static_cast<float>(Sl), Qh = static_cast<float>(Qoff);
            gsh[r] = make_float4(Th, static_cast<float>(static_cast<double>(Th) - T), Sh,
                                 static_cast<float>(static_cast<double>(Sh) - Sl));
            rsc[r] = static_cast<float>(exp2(Lme));
            q1i[r] = make_float2(Qh, static_cast<float>(static_cast<double>(Qh) - Qoff));
            if (MODE == MODE_GN) {
                double dG = 0.0, P1 = 0.0, P2 = 0.0, P3 = 0.0;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    if (q < K) {
                        dG += exp2(Lb[q]) * (dgq[q] - dLb[q] * gq[q]);
                        if (PAIRED) {
                            const double e = exp2(-Lb[q + 1]);   // rebased R1..R3
                            P1 += e * p1q[q];
                            P2 += e * p2q[q];
                            P3 += e * (p3q[q] + dLb[q] * p2q[q]);
                        }
                    }
                }
                rout[r] = static_cast<float>(A.delta * dG);
                if (PAIRED) rout[R + r] = static_cast<float>(A.delta * exp2(LK) * (P1 + P3 - dLK * P2));
            }
        }
        float2* slot = A.slots + static_cast<size_t>(ui.slot) * plane;
        if (ui.first) {   // the slot's first unit zeroes its writable rows (later flushes only add)
            float4* z = reinterpret_cast<float4*>(slot);
            const size_t z0 = static_cast<size_t>(A.slot_lo[ui.slot]) * A.Ns / 2;
            const size_t z1 = static_cast<size_t>(A.slot_hi[ui.slot]) * A.Ns / 2;
            for (size_t k = z0 + tid; k < z1; k += NT) z[k] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        __syncthreads();
        const size_t wbase = (static_cast<size_t>(ui.m) * A.n_ab + ui.ab) * A.n_det;
        const size_t wbase2 = (static_cast<size_t>(ui.m) * A.n_ab + dup_of(A, ui.ab)) * A.n_det;
        const size_t wpbase = (static_cast<size_t>(ui.m) * A.n_ab + ui.ab + 1) * A.n_det;
        const size_t wpbase2 = (static_cast<size_t>(ui.m) * A.n_ab + dup_of(A, ui.ab + 1)) * A.n_det;
        const RayP rfirst = rays[0], rlast = rays[R - 1];
        const double kuv = static_cast<double>(dU) / static_cast<double>(dV);
        auto ucol = [&](const RayP& rp, double vrow) {
            return (static_cast<double>(rp.U0) + (vrow * 4294967296.0 - static_cast<double>(rp.V0)) * kuv) *
                   (1.0 / 4294967296.0);
        };
        for (int pass = 0; pass < A.passesB; ++pass) {
            const int grp = pass * W + warp;
            const int r = grp < A.n_groups ? A.groups[grp * 32 + lane] : -1;
            int ii = -1, ilo = 0, kc = 0;
            int64_t uu = 0, vv = 0;
            RayB rb{0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
            StateB st{0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
            float cw = 0.f, cw1 = 0.f;
            float4* cl = nullptr;
            float2 am = make_float2(0.f, 0.f);
            if (r >= 0) {
                const int d = r / J, j = r - d * J;
                float wd = 0.f, wd1 = 0.f;
                if (MODE == MODE_GN) {
                    for (int jj = 0; jj < J; ++jj) {
                        wd = fmaf(A.w[jj], rout[d * J + jj], wd);
                        if (PAIRED) wd1 = fmaf(A.w[jj], rout[R + d * J + jj], wd1);
                    }
                    if (A.dup_half) { wd *= 2.f; wd1 *= 2.f; }
                } else {
                    wd = A.win[wbase + d];
                    if (A.dup_half) wd += A.win[wbase2 + d];
                    if (PAIRED) wd1 = A.win[wpbase + A.n_det - 1 - d] + A.win[wpbase2 + A.n_det - 1 - d];
                }
                const float wr = A.w[j] * wd, wr1 = A.w[j] * wd1;
                const float sc = rsc[r];
                const float4 G = gsh[r];
                const float2 q1 = q1i[r];
                if (CACHE) {   // unit-weight constants; the lane's weights apply after the cache store
                    rb = RayB{A.delta * sc, -A.delta * A.delta * sc, G.x, G.y, A.delta, -A.delta * A.delta, G.z, G.w};
                    cw = wr;
                    cw1 = wr1;
                    int kend_unused;
                    cl = cache_lane(A, ui, grp, lane, &kend_unused);
                } else {
                    rb = RayB{wr * A.delta * sc, -wr * A.delta * A.delta * sc, G.x, G.y,
                              wr1 * A.delta, -wr1 * A.delta * A.delta, G.z, G.w};
                }
                st.q1 = q1.x;
                st.q1c = q1.y;
                if (CACHE || wr != 0.f || wr1 != 0.f) {
                    const RayP rp = rays[r];
                    ii = seg_entry(rp, bound);
                    ilo = rp.ilo;
                    uu = rp.U0 + static_cast<int64_t>(ii) * dU;
                    vv = rp.V0 + static_cast<int64_t>(ii) * dV;
                }
            }
            for (int j = 0; j < ui.nb; ++j) {
                int r0, r1;
                seg_band(ui, j, Rb, r0, r1);
                const int b = static_cast<int>(s & 1);
                mbar_wait(&mbar[b], static_cast<uint32_t>((s >> 1) & 1));
                const float2* sbuf = reinterpret_cast<const float2*>(stage0 + b * A.stage_bytes);
                const bool flip = j & 1;
                const int abase = flip ? Rb * P : 0, sP = flip ? -P : P;
                if (PGET_ABLATE != 3)   // 3: no sweep B walk at all
                    walk_b<PAIRED, ModeTraits<MODE>::COMP_S, CACHE>(sbuf, wacc, P, r0, r1, abase, sP, ilo, dU, dV, cf, ch,
                                                                    rb, ii, uu, vv, st, cw, cw1, cl, &kc, &am);
                __syncthreads();   // stage buffer b and every warp ring consumed
                if (tid == 0 && s + 2 < n_stages)
                    issue_seg_stage<false>(A, Rb, sb0 + s + 2, stage0 + b * A.stage_bytes, &mbar[b]);
                ++s;
                // flush (as proj_kernel): finished rows into the slot, column-limited, fixed thread per element
                const bool last = j == ui.nb - 1;
                const int carry = last ? -1 : (ui.dir > 0 ? r0 : r1);
                int qlo, qhi;
                {
                    const double a0 = ucol(rfirst, r0 - 1.0), a1 = ucol(rfirst, r1 + 1.0);
                    const double b0 = ucol(rlast, r0 - 1.0), b1 = ucol(rlast, r1 + 1.0);
                    const double umin = fmin(fmin(a0, a1), fmin(b0, b1)), umax = fmax(fmax(a0, a1), fmax(b0, b1));
                    qlo = max(0, static_cast<int>(floor(umin)) - 2) >> 1;
                    qhi = min(P - 1, static_cast<int>(floor(umax)) + 3) >> 1;
                }
                const int e_beg = r0 * npairs, e_end = (r1 + 1) * npairs;
                for (int e = e_beg + (tid - e_beg % NT + NT) % NT; e < e_end; e += NT) {
                    int rw = __float2int_rd(static_cast<float>(e) * inv_np);
                    int q = e - rw * npairs;
                    if (q < 0) { --rw; q += npairs; } else if (q >= npairs) { ++rw; q -= npairs; }
                    if (rw == carry || q < qlo || q > qhi || PGET_ABLATE == 2) continue;   // 2: no flush
                    const int lr = flip ? r0 + Rb - rw : rw - r0;
                    PGET_CHECK(lr >= 0 && lr < RB1);
                    float4 sum = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
                    for (int w = 0; w < W; ++w) {
                        float4* el = reinterpret_cast<float4*>(wacc_all + (static_cast<size_t>(w) * RB1 + lr) * P) + q;
                        const float4 x = *el;
                        sum.x += x.x; sum.y += x.y; sum.z += x.z; sum.w += x.w;
                        *el = make_float4(0.f, 0.f, 0.f, 0.f);
                    }
                    const int ir = rw - kHalo, ic = 2 * q - kHalo;
                    if (ir >= 0 && ir < A.N && ic >= 0 && ic < A.Ns)
                        atomicAdd(reinterpret_cast<float4*>(slot + static_cast<size_t>(ir) * A.Ns + ic), sum);
                }
                __syncthreads();   // rings zeroed before the next band's scatter
            }
            if (CACHE) entry_bounds(A, ui, am);
        }
    }
}

// ------------------------------------------------------------------------------------------ GN, cached coefficients
// The Jacobian of one LM iteration is fixed while CG runs, and every GN product J^T (J p) needs, per
// line sample i of ray r, only the Jacobian entries of the sample (the adjoint weights at w_r = 1):
//   alpha_i = dy_r / dlam_i = Delta E_i,     beta_i = dy_r / dmu_i = -Delta^2 (G - Q_i - lam_i E_i / 2)
// and (line pairing) alpha'_i, beta'_i of the opposite-bank ray, so that
//   (J p)_r = sum_i (dlam_i alpha_i + dmu_i beta_i),     J^T w scatters w_r (alpha_i, beta_i) bilinearly.
// lin_kernel writes them once per LM iteration (the segmented phase-B walk with w = 1, compensated
// sums), jvpc_kernel forms the per-ray (J p) partials of each segment from staged p and the cache,
// gnb_kernel scatters w_r (alpha_i, beta_i) + w'_r (alpha'_i, beta'_i) -- no image, no exp -- into the
// warp band accumulators and slots of seg_b_kernel.  Cache layout: per (member, traced angle-bank,
// segment, comb group) kmax rows of 32 lanes (schedule.cpp); a lane's k-th sample of the unit is
// row k of its block.
__device__ __forceinline__ float4* cache_lane(const ProjArgs& A, const UnitInfo& ui, int grp, int lane, int* kend)
{
    const int t = (ui.canon / A.K) % A.ntab;
    const int64_t idx = (static_cast<int64_t>(t) * A.K + ui.seg) * A.cache_ng + grp;
    const int64_t off = A.cache_off[idx];
    *kend = static_cast<int>(A.cache_off[idx + 1] - off);   // rows of the block
    const int64_t row = static_cast<int64_t>(ui.m) * A.cache_rows_member + off;
    return A.cache + row * 32 + lane;
}

// per-ray constants of a segment for the adjoint at w = 1 (seg_b_kernel's combination, VJP part)
template <bool PAIRED>
__device__ __forceinline__ void seg_constants(const ProjArgs& A, const UnitInfo& ui, int r, float4* gsh, float* rsc,
                                              float2* q1i)
{
    const int R = A.R, K = A.K;
    const int qme = ui.dir > 0 ? K - 1 - ui.seg : ui.seg;
    const float* part0 = A.segp + static_cast<size_t>(ui.canon - ui.seg) * kSegFields * R;
    double Lb[5], gq[4], p2q[4];
    Lb[0] = 0.0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        gq[q] = p2q[q] = 0.0;
        double sq = 0.0;
        if (q < K) {
            const float* pq = part0 + static_cast<size_t>(ui.dir > 0 ? K - 1 - q : q) * kSegFields * R;
            sq = static_cast<double>(pq[0 * R + r]) - pq[1 * R + r];
            gq[q] = static_cast<double>(pq[2 * R + r]) - pq[3 * R + r];
            if (PAIRED) p2q[q] = pq[7 * R + r];
        }
        Lb[q + 1] = Lb[q] + sq;
    }
    double Lme = 0.0, LK = 0.0;
#pragma unroll
    for (int q = 0; q < 5; ++q) {
        if (q == qme) Lme = Lb[q];
        if (q == K) LK = Lb[q];
    }
    double T = 0.0, Qoff = 0.0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        if (q >= qme && q < K) T += exp2(Lb[q] - Lme) * gq[q];
        if (PAIRED && q < qme) Qoff += exp2(LK - Lb[q + 1]) * p2q[q];   // rebased R2
    }
    const double Sl = LK - Lme;
    const float Th = static_cast<float>(T), Sh = static_cast<float>(Sl), Qh = static_cast<float>(Qoff);
    gsh[r] = make_float4(Th, static_cast<float>(static_cast<double>(Th) - T), Sh,
                         static_cast<float>(static_cast<double>(Sh) - Sl));
    rsc[r] = static_cast<float>(exp2(Lme));
    q1i[r] = make_float2(Qh, static_cast<float>(static_cast<double>(Qh) - Qoff));
}

// whole-ray (J p) of both directions from the GN-mode phase-A segment partials (seg_b_kernel's GN
// combination, in ray order)
template <bool PAIRED>
__device__ __forceinline__ void gn_rout_from_seg(const ProjArgs& A, int canon0, int dir, int r, float* rout)
{
    const int R = A.R, K = A.K;
    const float* part0 = A.segp + static_cast<size_t>(canon0) * kSegFields * R;
    double Lb[5], dLb[5], gq[4], p1q[4], p2q[4], p3q[4], dgq[4];
    Lb[0] = 0.0;
    dLb[0] = 0.0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        gq[q] = p1q[q] = p2q[q] = p3q[q] = dgq[q] = 0.0;
        double sq = 0.0, dsq = 0.0;
        if (q < K) {
            const float* pq = part0 + static_cast<size_t>(dir > 0 ? K - 1 - q : q) * kSegFields * R;
            sq = static_cast<double>(pq[0 * R + r]) - pq[1 * R + r];
            gq[q] = static_cast<double>(pq[2 * R + r]) - pq[3 * R + r];
            if (PAIRED) p2q[q] = pq[7 * R + r];
            dsq = pq[4 * R + r];
            dgq[q] = pq[5 * R + r];
            p1q[q] = pq[6 * R + r];
            p3q[q] = pq[8 * R + r];
        }
        Lb[q + 1] = Lb[q] + sq;
        dLb[q + 1] = dLb[q] + dsq;
    }
    double LK = 0.0, dLK = 0.0;
#pragma unroll
    for (int q = 0; q < 5; ++q)
        if (q == K) { LK = Lb[q]; dLK = dLb[q]; }
    double dG = 0.0, P1 = 0.0, P2 = 0.0, P3 = 0.0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        if (q < K) {
            dG += exp2(Lb[q]) * (dgq[q] - dLb[q] * gq[q]);
            if (PAIRED) {
                const double e = exp2(-Lb[q + 1]);   // rebased R1..R3 (seg_a_kernel)
                P1 += e * p1q[q];
                P2 += e * p2q[q];
                P3 += e * (p3q[q] + dLb[q] * p2q[q]);
            }
        }
    }
    rout[r] = static_cast<float>(A.delta * dG);
    rout[R + r] = PAIRED ? static_cast<float>(A.delta * exp2(LK) * (P1 + P3 - dLK * P2)) : 0.f;
}

// lin walk: the Jacobian entries of every sample of the band into the lane's cache block
// walk_lin, unrolled by two with alternating register roles and unconditional next-sample loads (walk_b)
template <bool PAIRED>
__device__ __forceinline__ void walk_lin(const float2* __restrict__ img, int P, int r0, int r1, int ilo, int64_t dU,
                                         int64_t dV, float cf, float ch, const RayB& rb, int& i, int64_t& u,
                                         int64_t& v, StateB& st, float4* cl, int& k, float2& am)
{
    {
        const int iv = hi32(v);
        if (i < ilo || iv < r0 || iv >= r1) return;
    }
    auto load = [&](SmpB& x, int64_t uu, int64_t vv, bool ok) {
        int o = (hi32(vv) - r0) * P + hi32(uu);
        o = ok ? o : 0;
        PGET_CHECK(o >= 0 && o + P + 1 < (r1 - r0 + 1) * P);
        x.c00 = img[o]; x.c01 = img[o + 1]; x.c10 = img[o + P]; x.c11 = img[o + P + 1];
        x.fu = frac23(uu);
        x.fv = frac23(vv);
    };
    StateB x_ = st;
    auto step = [&](const SmpB& cur, SmpB& nx) -> bool {
        const int i2 = i - 1;
        const int64_t u2 = u - dU, v2 = v - dV;
        const int iv2 = hi32(v2);
        const bool nxt = i2 >= ilo && iv2 >= r0 && iv2 < r1;   // sweep-B bands are a few rows: no band_steps
        load(nx, u2, v2, nxt);
        const float2 x = bilerp2(cur.c00, cur.c01, cur.c10, cur.c11, cur.fu, cur.fv);
        const float arg_hi = fmaf(x.y, ch, x_.s);
        const float E = ex2(arg_hi - x_.sc);
        const float le = x.x * E;
        float4 cv;
        cv.x = rb.kl * E;
        cv.y = rb.km * (((rb.G - x_.q) - (rb.Gc - x_.qc)) - 0.5f * le);
        cv.z = 0.f;
        cv.w = 0.f;
        if constexpr (PAIRED) {
            const float E1 = ex2((rb.Sl - arg_hi) - (rb.Slc - x_.sc));
            const float le1 = x.x * E1;
            cv.z = rb.kl1 * E1;
            cv.w = rb.km1 * ((x_.q1 - x_.q1c) + 0.5f * le1);
            kahan(x_.q1, x_.q1c, le1);
        }
        kahan(x_.q, x_.qc, le);
        kahan(x_.s, x_.sc, x.y * cf);
        __stcs(cl + static_cast<int64_t>(k) * 32, cv);   // streaming store: written once, read 2 x n_cg times
        am.x = fmaxf(am.x, fmaxf(fabsf(cv.x), fabsf(cv.z)));
        am.y = fmaxf(am.y, fmaxf(fabsf(cv.y), fabsf(cv.w)));
        ++k;
        i = i2;
        u = u2;
        v = v2;
        return nxt;
    };
    SmpB sa, sb;
    load(sa, u, v, true);
    while (step(sa, sb) && step(sb, sa)) {
    }
    st = x_;
}

// Cached entries are streamed from HBM: a 4-slot register ring (the entry of sample k+4 is loaded
// into the slot just consumed) plus an L2 prefetch 16 samples ahead keep several loads in flight per
// lane; kend bounds the reads to the lane's cache block.
__device__ __forceinline__ float4 ld_entry(const float4* __restrict__ cl, int k, int kend)
{
    return k < kend ? __ldg(cl + static_cast<int64_t>(k) * 32) : make_float4(0.f, 0.f, 0.f, 0.f);
}
__device__ __forceinline__ void pf_entry(const float4* cl, int k, int kend)
{
    if (k < kend) asm volatile("prefetch.global.L2 [%0];" ::"l"(cl + static_cast<int64_t>(k) * 32));
}

// jvpc walk: (J p) partial sums of the band from staged p = (dlam, dmu) and the cached entries
__device__ __forceinline__ void walk_jvpc(const float2* __restrict__ img, int P, int r0, int r1, int ilo, int64_t dU,
                                          int64_t dV, int& i, int64_t& u, int64_t& v, const float4* __restrict__ cl,
                                          int& k, int kend, float& acc, float& acc1)
{
    const int iv0 = hi32(v);
    if (i < ilo || iv0 < r0 || iv0 >= r1) return;
    float4 c0 = ld_entry(cl, k, kend), c1 = ld_entry(cl, k + 1, kend), c2 = ld_entry(cl, k + 2, kend),
           c3 = ld_entry(cl, k + 3, kend);
    int o = (iv0 - r0) * P + hi32(u);
    float2 q00 = img[o], q01 = img[o + 1], q10 = img[o + P], q11 = img[o + P + 1];
    float fu = frac23(u), fv = frac23(v);
    auto step = [&](float4& c) -> bool {
        const int i2 = i - 1;
        const int64_t u2 = u - dU, v2 = v - dV;
        const int iv2 = hi32(v2);
        const bool nxt = i2 >= ilo && iv2 >= r0 && iv2 < r1;
        float2 n00 = q00, n01 = q01, n10 = q10, n11 = q11;
        int o2 = o;
        if (nxt) {
            o2 = (iv2 - r0) * P + hi32(u2);
            n00 = img[o2]; n01 = img[o2 + 1]; n10 = img[o2 + P]; n11 = img[o2 + P + 1];
        }
        const float2 d = bilerp2(q00, q01, q10, q11, fu, fv);
        acc = fmaf(d.x, c.x, fmaf(d.y, c.y, acc));
        acc1 = fmaf(d.x, c.z, fmaf(d.y, c.w, acc1));
        pf_entry(cl, k + PGET_PF_DIST, kend);
        c = ld_entry(cl, k + 4, kend);
        ++k;
        i = i2;
        u = u2;
        v = v2;
        q00 = n00; q01 = n01; q10 = n10; q11 = n11;
        o = o2;
        fu = frac23(u);
        fv = frac23(v);
        return nxt;
    };
    while (step(c0) && step(c1) && step(c2) && step(c3)) {
    }
}

// gnb walk: scatter w_r (alpha, beta) + w'_r (alpha', beta') of the band's samples (same-cell registers).
// ck points at the lane's next entry; the ring reads up to 4 rows and the prefetch PGET_PF_DIST rows
// past it unchecked (kCachePadRows rows are allocated past the cache).
// INTACC: one block-shared accumulator of 32-bit fixed-point values in two planes (lambda, mu; planar
// so that a warp's adds spread over all 32 banks), added to with native shared
// integer atomics (red.shared.add.u32): a pending cell's four float2 sums are scaled by S (a power of
// two, |value * S| < 2^22 by construction, see gnb_kernel), rounded to integers with the
// 1.5 * 2^23 magic-number FFMA and added.  Integer addition is associative, so the result does not
// depend on the order in which warps and lanes add.
static_assert(PGET_PF_DIST + 4 <= kCachePadRows, "cache read-ahead exceeds the padding");
__device__ __forceinline__ void red_s32(uint32_t addr, int v)
{
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
// The cached scatter's entry stream is read once per product: with PGET_GNB_EF its loads carry an L2 evict-first
// policy, so the stream does not push the CTA-private slot partials (re-read and re-written by every unit's
// flush, then read by the slot reduction) out of L2.
#ifndef PGET_GNB_EF
#define PGET_GNB_EF 0
#endif
__device__ __forceinline__ float4 ldg_entry(const float4* p)
{
#if PGET_GNB_EF
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    float4 v;
    asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p), "l"(pol));
    return v;
#else
    return __ldg(p);
#endif
}
template <bool INTACC>
__device__ __forceinline__ void walk_gnb(float2* __restrict__ acc, int P, int r0, int r1, int ilo,
                                         int64_t dU, int64_t dV, float wr, float wr1, int& i, int64_t& u, int64_t& v,
                                         const float4*& ck, const float4* cend, float2 S, uint32_t planeB, int sP4)
{
    const int sP = P;   // accumulator row of sample row iv: iv - r0
    const int iv0 = hi32(v);
    if (i < ilo || iv0 < r0 || iv0 >= r1) return;
    int n = band_steps(i, ilo, v, dV, r0, r1);
    // byte address of a sample's cell in the shared accumulator: org + iv * sP4 + iu * 4 (INTACC), with
    // org the address of (row 0, col 0) for this band's row mapping (abase + (iv - r0) sP + iu); sP4 =
    // 4 P and planeB come from the kernel parameters (constant-bank operands, nothing rematerialised)
    const uint32_t org = static_cast<uint32_t>(__cvta_generic_to_shared(acc)) - static_cast<uint32_t>(r0 * sP * 4);
    auto cell = [&](int ivv, int iuu) -> uint32_t { return org + static_cast<uint32_t>(ivv * sP4 + iuu * 4); };
    auto rmw = [&](uint32_t a0, float2 a, float2 b, float2 c, float2 d) {
        if constexpr (INTACC) {
            const float2 mg = make_float2(12582912.f, 12582912.f);   // 1.5 * 2^23
            const float2 ta = __ffma2_rn(a, S, mg), tb = __ffma2_rn(b, S, mg);
            const float2 tc = __ffma2_rn(c, S, mg), td = __ffma2_rn(d, S, mg);
            const uint32_t a1 = a0 + static_cast<uint32_t>(sP4);
            red_s32(a0, __float_as_int(ta.x) - 0x4B400000);
            red_s32(a0 + planeB, __float_as_int(ta.y) - 0x4B400000);
            red_s32(a0 + 4, __float_as_int(tb.x) - 0x4B400000);
            red_s32(a0 + 4 + planeB, __float_as_int(tb.y) - 0x4B400000);
            red_s32(a1, __float_as_int(tc.x) - 0x4B400000);
            red_s32(a1 + planeB, __float_as_int(tc.y) - 0x4B400000);
            red_s32(a1 + 4, __float_as_int(td.x) - 0x4B400000);
            red_s32(a1 + 4 + planeB, __float_as_int(td.y) - 0x4B400000);
        } else {
            // element index: cell() counts 4 bytes per element in both layouts
            float2* pa = acc + (static_cast<int>(a0 - static_cast<uint32_t>(__cvta_generic_to_shared(acc))) >> 2);
            const float2 t00 = pa[0], t01 = pa[1], t10 = pa[sP], t11 = pa[sP + 1];
            pa[0] = make_float2(t00.x + a.x, t00.y + a.y);
            pa[1] = make_float2(t01.x + b.x, t01.y + b.y);
            pa[sP] = make_float2(t10.x + c.x, t10.y + c.y);
            pa[sP + 1] = make_float2(t11.x + d.x, t11.y + d.y);
        }
    };
    // the pending cell starts as the first sample's (valid address, zero sums): no first-time test
    uint32_t pa = cell(iv0, hi32(u));
    const float2 z2 = make_float2(0.f, 0.f);
    float2 p00 = z2, p01 = z2, p10 = z2, p11 = z2;
    const float4* const p0 = ck;
    int k = 0;   // entry row of the current sample, relative to p0
    float4 c0 = ldg_entry(p0), c1 = ldg_entry(p0 + 32), c2 = ldg_entry(p0 + 64), c3 = ldg_entry(p0 + 96);
    const float2 w2 = make_float2(wr, wr), w12 = make_float2(wr1, wr1);
    auto step = [&](float4& c) -> bool {
        const int iv = hi32(v);
        const uint32_t aa = cell(iv, hi32r(u));
        PGET_CHECK(hi32(u) >= 0 && hi32(u) + 1 < P && iv >= r0 && iv < r1 && p0 + k * 32 < cend);
        // 1 + the bilinear fractions (exactly): x * f = x * (1 + f) - x in one FMA, bit for bit the
        // product of walk_b, without the two subtractions of 1
        const float gu = frac23p1(u), gv = frac23p1(v);
        const float2 av = __ffma2_rn(w2, make_float2(c.x, c.y), __fmul2_rn(w12, make_float2(c.z, c.w)));
#if PGET_ABLATE == 4   // 4: no entry stream (the first four rows again: cache hits; wrong values, timing only)
        c = __ldg(p0 + (((k + 4) & 3) << 5));
#else
        asm volatile("prefetch.global.L2 [%0];" ::"l"(p0 + ((k + PGET_PF_DIST) << 5)));
        c = ldg_entry(p0 + ((k + 4) << 5));
#endif
        ++k;
        const float2 nav = make_float2(-av.x, -av.y);
        const float2 tv = __ffma2_rn(av, make_float2(gv, gv), nav);     // row j0+1: av * fv
        const float2 bv = __ffma2_rn(tv, make_float2(-1.f, -1.f), av); // row j0
        const float2 c11 = __ffma2_rn(tv, make_float2(gu, gu), make_float2(-tv.x, -tv.y));
        const float2 c10 = __ffma2_rn(c11, make_float2(-1.f, -1.f), tv);
        const float2 c01 = __ffma2_rn(bv, make_float2(gu, gu), make_float2(-bv.x, -bv.y));
        const float2 c00 = __ffma2_rn(c01, make_float2(-1.f, -1.f), bv);
        if (aa != pa) {
            if (PGET_ABLATE != 1 || p00.x == 12345.f) rmw(pa, p00, p01, p10, p11);   // ABLATE 1: no scatter
            pa = aa;
            p00 = c00; p01 = c01; p10 = c10; p11 = c11;
        } else {
            p00 = __fadd2_rn(p00, c00);
            p01 = __fadd2_rn(p01, c01);
            p10 = __fadd2_rn(p10, c10);
            p11 = __fadd2_rn(p11, c11);
        }
        u -= dU;
        v -= dV;
        return true;
    };
    // full rounds of the 4-entry ring without per-sample exit tests, then the 0-3 remaining samples
    for (; n >= 4; n -= 4) {
        step(c0);
        step(c1);
        step(c2);
        step(c3);
    }
    if (n > 0) {
        step(c0);
        if (n > 1) {
            step(c1);
            if (n > 2) step(c2);
        }
    }
    rmw(pa, p00, p01, p10, p11);
    i -= k;
    ck = p0 + (k << 5);
}

// per-unit lane setup shared by the three kernels: the lane's ray of comb group grp, its entry
// sample into the unit's segment and position; false if the lane has no ray
__device__ __forceinline__ bool lane_ray(const ProjArgs& A, const UnitInfo& ui, const RayP* rays, int grp, int lane,
                                         int64_t dU, int64_t dV, int& r, int& ii, int& ilo, int64_t& uu, int64_t& vv)
{
    r = grp < A.n_groups ? A.groups[grp * 32 + lane] : -1;
    ii = -1; ilo = 0; uu = 0; vv = 0;
    if (r < 0) return false;
    const RayP rp = rays[r];
    ii = seg_entry(rp, ui.dir > 0 ? ui.yhi : ui.ylo);
    ilo = rp.ilo;
    uu = rp.U0 + static_cast<int64_t>(ii) * dU;
    vv = rp.V0 + static_cast<int64_t>(ii) * dV;
    return true;
}

// lin_kernel: once per LM iteration.  Stages (lam, mu) bands like seg_b_kernel (same units, groups,
// stage list); needs the segment partials of the VJP-mode phase A.
template <bool PAIRED>
__global__ void __launch_bounds__(512, 1) lin_kernel(ProjArgs A)
{
    pdl_entry();
    const int W = blockDim.x >> 5;
    const int NT = blockDim.x;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* mbar = reinterpret_cast<uint64_t*>(smem);
    unsigned char* const stage0 = smem + 128;
    float4* gsh = reinterpret_cast<float4*>(smem + A.off_gsh);
    float* rsc = reinterpret_cast<float*>(smem + A.off_rsc);
    float2* q1i = reinterpret_cast<float2*>(smem + A.off_q1);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int c = blockIdx.x;
    const int64_t sb0 = A.s_begin[c];
    const int64_t n_stages = A.s_begin[c + 1] - sb0;
    if (n_stages == 0) return;
    const int P = A.P, R = A.R, Rb = A.RbB;
    if (tid == 0) {
        mbar_init(&mbar[0], 1);
        mbar_init(&mbar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0) {
        issue_seg_stage<false>(A, Rb, sb0, stage0, &mbar[0]);
        if (n_stages > 1) issue_seg_stage<false>(A, Rb, sb0 + 1, stage0 + A.stage_bytes, &mbar[1]);
    }
    int64_t s = 0;
    const float cf = A.cf, ch = A.ch;
    for (int u = A.u_begin[c]; u < A.u_begin[c + 1]; ++u) {
        const UnitInfo ui = unit_info(A, u, Rb);
        const RayP* rays = A.rays + static_cast<size_t>(ui.ab) * R;
        const int64_t dU = rays[0].dU, dV = rays[0].dV;
        for (int r = tid; r < R; r += NT) seg_constants<PAIRED>(A, ui, r, gsh, rsc, q1i);
        __syncthreads();
        for (int pass = 0; pass < A.passesB; ++pass) {
            const int grp = pass * W + warp;
            int r, ii, ilo, k = 0;
            int64_t uu, vv;
            RayB rb{0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
            StateB st{0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
            float4* cl = nullptr;
            float2 am = make_float2(0.f, 0.f);
            if (lane_ray(A, ui, rays, grp, lane, dU, dV, r, ii, ilo, uu, vv)) {
                const float sc = rsc[r];
                const float4 G = gsh[r];
                const float2 q1 = q1i[r];
                rb = RayB{A.delta * sc, -A.delta * A.delta * sc, G.x, G.y, A.delta, -A.delta * A.delta, G.z, G.w};
                st.q1 = q1.x;
                st.q1c = q1.y;
                int kend_unused;
                cl = cache_lane(A, ui, grp, lane, &kend_unused);
            }
            for (int j = 0; j < ui.nb; ++j) {
                int r0, r1;
                seg_band(ui, j, Rb, r0, r1);
                const int b = static_cast<int>(s & 1);
                mbar_wait(&mbar[b], static_cast<uint32_t>((s >> 1) & 1));
                const float2* sbuf = reinterpret_cast<const float2*>(stage0 + b * A.stage_bytes);
                walk_lin<PAIRED>(sbuf, P, r0, r1, ilo, dU, dV, cf, ch, rb, ii, uu, vv, st, cl, k, am);
                __syncthreads();   // stage buffer b consumed
                if (tid == 0 && s + 2 < n_stages)
                    issue_seg_stage<false>(A, Rb, sb0 + s + 2, stage0 + b * A.stage_bytes, &mbar[b]);
                ++s;
            }
            entry_bounds(A, ui, am);
        }
        __syncthreads();   // gsh / rsc / q1i are rewritten by the next unit
    }
}

// jvpc_kernel: per CG step, the per-ray (J p) partials of every unit from staged p (float2 bands of
// (dlam, dmu), the same stage list) and the cache.
__global__ void __launch_bounds__(512, 1) jvpc_kernel(ProjArgs A)
{
    pdl_entry();
    const int W = blockDim.x >> 5;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* mbar = reinterpret_cast<uint64_t*>(smem);
    unsigned char* const stage0 = smem + 128;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int c = blockIdx.x;
    const int64_t sb0 = A.s_begin[c];
    const int64_t n_stages = A.s_begin[c + 1] - sb0;
    if (n_stages == 0) return;
    const int P = A.P, R = A.R, Rb = A.RbB;
    if (tid == 0) {
        mbar_init(&mbar[0], 1);
        mbar_init(&mbar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0) {
        issue_seg_stage<false>(A, Rb, sb0, stage0, &mbar[0]);
        if (n_stages > 1) issue_seg_stage<false>(A, Rb, sb0 + 1, stage0 + A.stage_bytes, &mbar[1]);
    }
    int64_t s = 0;
    for (int u = A.u_begin[c]; u < A.u_begin[c + 1]; ++u) {
        const UnitInfo ui = unit_info(A, u, Rb);
        const RayP* rays = A.rays + static_cast<size_t>(ui.ab) * R;
        const int64_t dU = rays[0].dU, dV = rays[0].dV;
        float* jp = A.jp + static_cast<size_t>(ui.canon) * 2 * R;
        for (int pass = 0; pass < A.passesB; ++pass) {
            const int grp = pass * W + warp;
            int r, ii, ilo, k = 0, kend = 0;
            int64_t uu, vv;
            float acc = 0.f, acc1 = 0.f;
            const float4* cl = nullptr;
            if (lane_ray(A, ui, rays, grp, lane, dU, dV, r, ii, ilo, uu, vv)) cl = cache_lane(A, ui, grp, lane, &kend);
            for (int j = 0; j < ui.nb; ++j) {
                int r0, r1;
                seg_band(ui, j, Rb, r0, r1);
                const int b = static_cast<int>(s & 1);
                mbar_wait(&mbar[b], static_cast<uint32_t>((s >> 1) & 1));
                const float2* sbuf = reinterpret_cast<const float2*>(stage0 + b * A.stage_bytes);
                walk_jvpc(sbuf, P, r0, r1, ilo, dU, dV, ii, uu, vv, cl, k, kend, acc, acc1);
                __syncthreads();   // stage buffer b consumed
                if (tid == 0 && s + 2 < n_stages)
                    issue_seg_stage<false>(A, Rb, sb0 + s + 2, stage0 + b * A.stage_bytes, &mbar[b]);
                ++s;
            }
            if (r >= 0) {
                jp[r] = acc;
                jp[R + r] = acc1;
            }
        }
    }
}

// the scatter weights of ray r from the whole-ray (J p) of its angle-bank: w_r = w_j sum_j' w_j' (J p)_{d,j'}
// (both directions; doubled for a duplicate-merged angle-bank)
__device__ __forceinline__ void gn_weights(const ProjArgs& A, const float* rout, int r, float& wr, float& wr1)
{
    const int J = A.J, R = A.R;
    const int d = r / J, j = r - d * J;
    float wd = 0.f, wd1 = 0.f;
    for (int jj = 0; jj < J; ++jj) {
        wd = fmaf(A.w[jj], rout[d * J + jj], wd);
        wd1 = fmaf(A.w[jj], rout[R + d * J + jj], wd1);
    }
    if (A.dup_half) { wd *= 2.f; wd1 *= 2.f; }
    wr = A.w[j] * wd;
    wr1 = A.w[j] * wd1;
}

// gnw_kernel: per CG step and (member, traced angle-bank), the whole-ray (J p) of the GN-mode phase-A
// partials (once, instead of once per segment unit inside gnb_kernel) and the scatter weights, to A.gw
// SINO: the VJP's weights instead, from the sinogram A.win (w_r = w_j (win[d] + win of the duplicate
// angle-bank), w'_r from bank 1 mirrored, as seg_b_kernel forms them): the cached scatter then computes
// the gradient J^T r of the LM iteration from the coefficient cache
template <bool PAIRED, bool SINO = false>
__global__ void __launch_bounds__(256) gnw_kernel(ProjArgs A, const int32_t* __restrict__ tabs, int ntab)
{
    pdl_entry();
    extern __shared__ __align__(128) unsigned char smem[];
    float* rout = reinterpret_cast<float*>(smem);   // [2R]
    const int t = blockIdx.x, m = blockIdx.y;
    const int R = A.R;
    const int ab = tabs[t];
    const int dir = A.rays[static_cast<size_t>(ab) * R].dV > 0 ? 1 : -1;
    const int ct = m * ntab + t;
    if (!SINO)
        for (int r = threadIdx.x; r < R; r += blockDim.x) gn_rout_from_seg<PAIRED>(A, ct * A.K, dir, r, rout);
    __syncthreads();
    float* gw = A.gw + static_cast<size_t>(ct) * 2 * R;
    float wm = 0.f, wm1 = 0.f;
    const size_t wbase = (static_cast<size_t>(m) * A.n_ab + ab) * A.n_det;
    const size_t wbase2 = (static_cast<size_t>(m) * A.n_ab + dup_of(A, ab)) * A.n_det;
    const size_t wpbase = (static_cast<size_t>(m) * A.n_ab + ab + 1) * A.n_det;
    const size_t wpbase2 = (static_cast<size_t>(m) * A.n_ab + dup_of(A, ab + 1)) * A.n_det;
    for (int r = threadIdx.x; r < R; r += blockDim.x) {
        float wr, wr1;
        if constexpr (SINO) {
            const int d = r / A.J, j = r - d * A.J;
            float wd = A.win[wbase + d], wd1 = 0.f;
            if (A.dup_half) wd += A.win[wbase2 + d];
            if (PAIRED) wd1 = A.win[wpbase + A.n_det - 1 - d] + A.win[wpbase2 + A.n_det - 1 - d];
            wr = A.w[j] * wd;
            wr1 = A.w[j] * wd1;
        } else {
            gn_weights(A, rout, r, wr, wr1);
        }
        gw[r] = wr;
        gw[R + r] = wr1;
        wm = fmaxf(wm, fabsf(wr));
        wm1 = fmaxf(wm1, fabsf(wr1));
    }
    if (A.gscale) {   // max |w_r|, |w'_r| of the angle-bank: gscale[ct * 8 + 2, 3]
        __shared__ float red[2][8];
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            wm = fmaxf(wm, __shfl_xor_sync(0xffffffffu, wm, o));
            wm1 = fmaxf(wm1, __shfl_xor_sync(0xffffffffu, wm1, o));
        }
        if ((threadIdx.x & 31) == 0) { red[0][threadIdx.x >> 5] = wm; red[1][threadIdx.x >> 5] = wm1; }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int k = 1; k < static_cast<int>(blockDim.x >> 5); ++k) {
                wm = fmaxf(wm, red[0][k]);
                wm1 = fmaxf(wm1, red[1][k]);
            }
            A.gscale[static_cast<size_t>(ct) * 8 + 2] = wm;
            A.gscale[static_cast<size_t>(ct) * 8 + 3] = wm1;
        }
    }
}

cudaError_t launch_gnw(bool paired, const ProjArgs& A, const int32_t* tabs, int ntab, int B, cudaStream_t s,
                       bool sino)
{
    const size_t sm = 2 * A.R * sizeof(float);
    if (sino) {
        if (paired) launch_k(gnw_kernel<true, true>, dim3(ntab, B), 256, sm, s, A, tabs, ntab);
        else launch_k(gnw_kernel<false, true>, dim3(ntab, B), 256, sm, s, A, tabs, ntab);
    } else {
        if (paired) launch_k(gnw_kernel<true>, dim3(ntab, B), 256, sm, s, A, tabs, ntab);
        else launch_k(gnw_kernel<false>, dim3(ntab, B), 256, sm, s, A, tabs, ntab);
    }
    return cudaGetLastError();
}

// gnb_kernel: per CG step, w_r from the (J p) partials, then the cached scatter into slots (as
// seg_b_kernel; no image staging).
// WIDE: up to 26 warps (one pass over 26 comb groups, configs 3-4) at <= 72 registers; else <= 16 warps
template <bool PAIRED, bool INTACC, bool WIDE = false>
__global__ void __launch_bounds__(WIDE ? 832 : 512, 1) gnb_kernel(ProjArgs A)
{
    pdl_entry();
    const int W = blockDim.x >> 5;
    const int NT = blockDim.x;
    extern __shared__ __align__(128) unsigned char smem[];
    float2* wacc_all = reinterpret_cast<float2*>(smem + A.off_wacc);
    float* rout = reinterpret_cast<float*>(smem + A.off_rout);   // [2R] whole-ray (J p), both directions
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int c = blockIdx.x;
    if (A.u_begin[c] == A.u_begin[c + 1]) return;
    const int P = A.P, R = A.R, K = A.K, Rb = A.RbB;
    const int RB1 = Rb + 1;
    const int NACC = INTACC ? 1 : W;   // INTACC: one shared fixed-point accumulator, else one per warp
    float2* wacc = wacc_all + (INTACC ? 0 : static_cast<size_t>(warp) * RB1 * P);
    {
        float4* z = reinterpret_cast<float4*>(wacc_all);
        const int n4 = NACC * RB1 * P / 2;
        for (int k = tid; k < n4; k += NT) z[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    const size_t plane = static_cast<size_t>(A.N) * A.Ns;
    for (int u = A.u_begin[c]; u < A.u_begin[c + 1]; ++u) {
        const UnitInfo ui = unit_info(A, u, Rb);
        const RayP* rays = A.rays + static_cast<size_t>(ui.ab) * R;
        const int64_t dU = rays[0].dU, dV = rays[0].dV;
        const float* jp0 = A.jp ? A.jp + static_cast<size_t>(ui.canon - ui.seg) * 2 * R : nullptr;
        for (int r = tid; r < R && !A.gw; r += NT) {   // whole-ray (J p) (gw: done by gnw_kernel)
            if (A.jp) {   // the K cached-entry partials of jvpc_kernel, in fixed order
                float a = 0.f, a1 = 0.f;
                for (int q = 0; q < K; ++q) {
                    a += jp0[static_cast<size_t>(q) * 2 * R + r];
                    a1 += jp0[static_cast<size_t>(q) * 2 * R + R + r];
                }
                rout[r] = a;
                rout[R + r] = a1;
            } else {      // the GN-mode phase-A partials (recomputed JVP of p)
                gn_rout_from_seg<PAIRED>(A, ui.canon - ui.seg, ui.dir, r, rout);
            }
        }
        float2* slot = A.slots + static_cast<size_t>(ui.slot) * plane;
        if (ui.first) {
            float4* z = reinterpret_cast<float4*>(slot);
            const size_t z0 = static_cast<size_t>(A.slot_lo[ui.slot]) * A.Ns / 2;
            const size_t z1 = static_cast<size_t>(A.slot_hi[ui.slot]) * A.Ns / 2;
            for (size_t k = z0 + tid; k < z1; k += NT) z[k] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        __syncthreads();
        const RayP rfirst = rays[0], rlast = rays[R - 1];
        const double kuv = static_cast<double>(dU) / static_cast<double>(dV);
        auto ucol = [&](const RayP& rp, double vrow) {
            return (static_cast<double>(rp.U0) + (vrow * 4294967296.0 - static_cast<double>(rp.V0)) * kuv) *
                   (1.0 / 4294967296.0);
        };
        // INTACC fixed-point scales of the unit's angle-bank: a pixel's pending-cell value is at most
        // cellmax samples x (max|w_r| + max|w'_r|) x the entry bound (bilinear weights <= 1); S, a power
        // of two (exact scaling both ways), puts that bound, raised by 2^-10 against rounding in the
        // pending sums, below 2^22, where the magic-number rounding is exact
        float2 S = make_float2(1.f, 1.f), iS = make_float2(1.f, 1.f);
        if constexpr (INTACC) {
            const float* gs = A.gscale + static_cast<size_t>((ui.canon - ui.seg) / K) * 8;
            const float wsum = (gs[2] + gs[3]) * (static_cast<float>(A.cellmax) * (1.f + 0x1p-10f));
            int ex, ey;
            frexpf(wsum * gs[0], &ex);
            frexpf(wsum * gs[1], &ey);
            S = make_float2(ldexpf(1.f, 22 - ex), ldexpf(1.f, 22 - ey));
            iS = make_float2(ldexpf(1.f, ex - 22), ldexpf(1.f, ey - 22));
        }
        for (int pass = 0; pass < A.passesB; ++pass) {
            const int grp = pass * W + warp;
            int r, ii, ilo, kend = 0;
            int64_t uu, vv;
            float wr = 0.f, wr1 = 0.f;
            const float4* cl = nullptr;
            if (lane_ray(A, ui, rays, grp, lane, dU, dV, r, ii, ilo, uu, vv)) {
                if (A.gw) {
                    const float* gw = A.gw + static_cast<size_t>((ui.canon - ui.seg) / K) * 2 * R;
                    wr = gw[r];
                    wr1 = gw[R + r];
                } else {
                    gn_weights(A, rout, r, wr, wr1);
                }
                cl = cache_lane(A, ui, grp, lane, &kend);
            }
            const float4* const cend = cl + static_cast<int64_t>(kend) * 32;
            for (int j = 0; j < ui.nb; ++j) {
                int r0, r1;
                seg_band(ui, j, Rb, r0, r1);
                // the band's accumulator rows are r - r0 (no flipping): the row it shares with the next
                // band is flushed with it, zeroed, and collects the next band's part (slot adds twice)
                if (PGET_ABLATE != 3)   // 3: no walk
                    walk_gnb<INTACC>(wacc, P, r0, r1, ilo, dU, dV, wr, wr1, ii, uu, vv, cl, cend, S,
                                     static_cast<uint32_t>(A.planeB4), A.P4);
                __syncthreads();   // every warp ring complete
                int qlo, qhi;
                {
                    const double a0 = ucol(rfirst, r0 - 1.0), a1 = ucol(rfirst, r1 + 1.0);
                    const double b0 = ucol(rlast, r0 - 1.0), b1 = ucol(rlast, r1 + 1.0);
                    const double umin = fmin(fmin(a0, a1), fmin(b0, b1)), umax = fmax(fmax(a0, a1), fmax(b0, b1));
                    qlo = max(0, static_cast<int>(floor(umin)) - 2) >> 1;
                    qhi = min(P - 1, static_cast<int>(floor(umax)) + 3) >> 1;
                }
                // element (row rw, pair q) is flushed by warp rw mod W, lane q mod 32 in every band: each
                // slot element always by the same thread, in program order (deterministic), without the
                // flat index's division; only the pairs [qlo, qhi] the band's rays can reach
                int rw = r0 + ((warp - r0 % W) % W + W) % W;
                const int qs = qlo + ((lane - qlo % 32) % 32 + 32) % 32;
                for (; rw <= r1 && PGET_ABLATE != 2; rw += W) {   // 2: no flush
                    const int lr = rw - r0;
                    PGET_CHECK(lr >= 0 && lr < RB1);
                    const int ir = rw - kHalo;
                    const bool inrow = ir >= 0 && ir < A.N;
                    for (int q = qs; q <= qhi; q += 32) {
                        float4 sum = make_float4(0.f, 0.f, 0.f, 0.f);
                        if constexpr (INTACC) {
                            int2* el = reinterpret_cast<int2*>(wacc_all) + static_cast<size_t>(lr) * (P / 2) + q;
                            int2* em = el + static_cast<size_t>(RB1) * (P / 2);   // mu plane
                            const int2 xl = *el, xm = *em;
                            *el = make_int2(0, 0);
                            *em = make_int2(0, 0);
                            sum = make_float4(static_cast<float>(xl.x) * iS.x, static_cast<float>(xm.x) * iS.y,
                                              static_cast<float>(xl.y) * iS.x, static_cast<float>(xm.y) * iS.y);
                        } else {
#pragma unroll 4
                            for (int w = 0; w < W; ++w) {
                                float4* el = reinterpret_cast<float4*>(wacc_all + (static_cast<size_t>(w) * RB1 + lr) * P) + q;
                                const float4 x = *el;
                                sum.x += x.x; sum.y += x.y; sum.z += x.z; sum.w += x.w;
                                *el = make_float4(0.f, 0.f, 0.f, 0.f);
                            }
                        }
                        const int ic = 2 * q - kHalo;
                        if (inrow && ic >= 0 && ic < A.Ns)
                            atomicAdd(reinterpret_cast<float4*>(slot + static_cast<size_t>(ir) * A.Ns + ic), sum);
                    }
                }
                __syncthreads();   // rings zeroed before the next band's scatter
            }
        }
    }
}

// ||J s||^2 of the LM wrap's pred from the GN-mode phase-A partials of (u, s) (paired: the two banks
// of a line per traversal; duplicate angle-banks counted twice): each block takes the segment-0
// units of its unit list, i.e. every (member, traced angle-bank) once, and writes that angle-bank's
// sum of squared detector values to sq[canon / K]
template <bool PAIRED>
__global__ void __launch_bounds__(512, 1) jsq_kernel(ProjArgs A, double* sq)
{
    pdl_entry();
    extern __shared__ __align__(128) unsigned char smem[];
    float* rout = reinterpret_cast<float*>(smem + A.off_rout);
    __shared__ double red[32];
    const int tid = threadIdx.x, NT = blockDim.x;
    const int c = blockIdx.x;
    const int R = A.R, J = A.J;
    for (int u = A.u_begin[c]; u < A.u_begin[c + 1]; ++u) {
        if (A.units[u].seg != 0) continue;
        const UnitInfo ui = unit_info(A, u, A.RbB);
        for (int r = tid; r < R; r += NT) gn_rout_from_seg<PAIRED>(A, ui.canon - ui.seg, ui.dir, r, rout);
        __syncthreads();
        double acc = 0.0;
        for (int d = tid; d < A.n_det; d += NT) {
            float yf = 0.f, yr = 0.f;
            for (int j = 0; j < J; ++j) {
                yf = fmaf(A.w[j], rout[d * J + j], yf);
                yr = fmaf(A.w[j], rout[R + d * J + j], yr);
            }
            acc += static_cast<double>(yf) * yf + static_cast<double>(yr) * yr;
        }
        if (A.dup_half) acc *= 2.0;   // the duplicate angle-bank measures the same rays
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
        if ((tid & 31) == 0) red[tid >> 5] = acc;
        __syncthreads();
        if (tid == 0) {
            double t = 0.0;
            for (int w = 0; w < (NT >> 5); ++w) t += red[w];
            sq[ui.canon / A.K] = t;
        }
        __syncthreads();   // rout and red are rewritten by the next unit
    }
}

// per member: the angle-banks' sums in order into partial[m * nblk] (the other nblk - 1 partials 0)
__global__ void jsq_member_kernel(const double* __restrict__ sq, int ntab, int B, int nblk, double* partial)
{
    pdl_entry();
    const int m = blockIdx.x * blockDim.x + threadIdx.x;
    if (m >= B) return;
    double t = 0.0;
    for (int i = 0; i < ntab; ++i) t += sq[static_cast<size_t>(m) * ntab + i];
    partial[static_cast<size_t>(m) * nblk] = t;
    for (int k = 1; k < nblk; ++k) partial[static_cast<size_t>(m) * nblk + k] = 0.0;
}

cudaError_t launch_jsq(bool paired, const ProjArgs& A, double* sq, int grid, int block, size_t smem, cudaStream_t s)
{
    if (paired) launch_k(jsq_kernel<true>, grid, block, smem, s, A, sq);
    else launch_k(jsq_kernel<false>, grid, block, smem, s, A, sq);
    return cudaGetLastError();
}

cudaError_t launch_jsq_member(const double* sq, int ntab, int B, int nblk, double* partial, cudaStream_t s)
{
    launch_k(jsq_member_kernel, (B + 127) / 128, 128, 0, s, sq, ntab, B, nblk, partial);
    return cudaGetLastError();
}

cudaError_t launch_gnc(int phase, bool paired, const ProjArgs& A, int grid, int block, size_t smem, cudaStream_t s)
{
    if (phase == 0) {
        if (paired) launch_k(lin_kernel<true>, grid, block, smem, s, A);
        else launch_k(lin_kernel<false>, grid, block, smem, s, A);
    } else if (phase == 1) {
        launch_k(jvpc_kernel, grid, block, smem, s, A);
    } else {
        if (A.gscale) {
            if (block > 512) {
                if (paired) launch_k(gnb_kernel<true, true, true>, grid, block, smem, s, A);
                else launch_k(gnb_kernel<false, true, true>, grid, block, smem, s, A);
            } else {
                if (paired) launch_k(gnb_kernel<true, true>, grid, block, smem, s, A);
                else launch_k(gnb_kernel<false, true>, grid, block, smem, s, A);
            }
        } else {
            if (paired) launch_k(gnb_kernel<true, false>, grid, block, smem, s, A);
            else launch_k(gnb_kernel<false, false>, grid, block, smem, s, A);
        }
    }
    return cudaGetLastError();
}

// Dynamic shared-memory limits are a per-(device, kernel) process-wide attribute: only ever raised, so a
// handle created later with a smaller configuration never lowers the limit an earlier (larger) handle
// relies on (handles are immutable and usable side by side, include/pget.h).
static std::mutex g_smem_mu;
static std::map<std::pair<int, const void*>, int> g_smem_hw;
template <class F>
static cudaError_t raise_smem(F* fn, int v)
{
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(g_smem_mu);
    int& hw = g_smem_hw[{dev, reinterpret_cast<const void*>(fn)}];
    if (v <= hw) return cudaSuccess;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, v);
    if (e == cudaSuccess) hw = v;
    return e;
}

cudaError_t set_gnc_smem_limit(size_t smem)
{
    const int v = static_cast<int>(smem);
    cudaError_t e;
    if ((e = raise_smem(lin_kernel<true>, v))) return e;
    if ((e = raise_smem(lin_kernel<false>, v))) return e;
    if ((e = raise_smem(jvpc_kernel, v))) return e;
    if ((e = raise_smem(gnb_kernel<true, false>, v))) return e;
    if ((e = raise_smem(gnb_kernel<true, true>, v))) return e;
    if ((e = raise_smem(gnb_kernel<false, true>, v))) return e;
    if ((e = raise_smem(gnb_kernel<true, true, true>, v))) return e;
    if ((e = raise_smem(gnb_kernel<false, true, true>, v))) return e;
    if ((e = raise_smem(jsq_kernel<true>, v))) return e;
    if ((e = raise_smem(jsq_kernel<false>, v))) return e;
    return raise_smem(gnb_kernel<false, false>, v);
}

// ------------------------------------------------------------------------------------------ reduction
// g[m][j][i] = sum over the class-0 slots of member m of slot[j][i] + sum over its class-1 slots of
// slot[i][j] (transposed frame), in fp64, slots in the schedule's fixed order.  Block (tile, m * G + g)
// adds the g-th of G ranges of member m's slot list into part[g][m]; finish_kernel adds the G
// partials in order g = 0..G-1 (deterministic).
__global__ void reduce_slots_kernel(const float2* __restrict__ slots, double2* __restrict__ part, int N, int Ns,
                                    int B, int G, const int32_t* __restrict__ red_off,
                                    const int32_t* __restrict__ red_slot, const int32_t* __restrict__ slot_lo,
                                    const int32_t* __restrict__ slot_hi)
{
    pdl_entry();
    __shared__ double2 tile[32][33];
    const int m = blockIdx.z / G, gq = blockIdx.z - m * G;
    const int tx = threadIdx.x, ty = threadIdx.y;   // 32 x 8
    const int i0 = blockIdx.x * 32, j0 = blockIdx.y * 32;
    const size_t plane = static_cast<size_t>(N) * Ns;
    const int e0 = red_off[2 * m], e1 = red_off[2 * m + 1], e2 = red_off[2 * m + 2];
    const int n = e2 - e0;
    double2 acc[4], accT[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) acc[k] = accT[k] = make_double2(0.0, 0.0);
    // slots in list order; four slots' loads are issued before their (in-order) additions, so each
    // thread keeps 16 loads in flight (the kernel is latency-bound otherwise)
    const int eb = e0 + (gq * n) / G, ee = e0 + ((gq + 1) * n) / G;
    for (int e = eb; e < ee; e += 4) {
        float2 v[4][4];
        int cl[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            cl[t] = -1;
            if (e + t < ee) {
                const int cls = e + t >= e1 ? 1 : 0;
                const int sid = red_slot[e + t];
                // slot rows outside [lo, hi) were never written: skip a slot that misses the tile
                const int t0 = cls ? i0 : j0, lo = slot_lo[sid], hi = slot_hi[sid];
                if (t0 + 32 <= lo || t0 >= hi) continue;
                cl[t] = cls;
                const float2* sl = slots + static_cast<size_t>(sid) * plane;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    // class 0: element (row j, col i) = (j0 + ty + 8k, i0 + tx)
                    // class 1: element (row i, col j) of the transposed slot = (i0 + ty + 8k, j0 + tx)
                    // rows outside [lo, hi) hold stale data (never zeroed, never written): read as 0
                    const int rr = (cls ? i0 : j0) + ty + 8 * k, cc = (cls ? j0 : i0) + tx;
                    v[t][k] = (rr >= lo && rr < hi && cc < N) ? sl[static_cast<size_t>(rr) * Ns + cc]
                                                              : make_float2(0.f, 0.f);
                }
            }
        }
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            if (cl[t] < 0) continue;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                double2& a = cl[t] ? accT[k] : acc[k];
                a.x += v[t][k].x;
                a.y += v[t][k].y;
            }
        }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) tile[ty + 8 * k][tx] = accT[k];   // tile[i - i0][j - j0]
    __syncthreads();
    double2* out = part + (static_cast<size_t>(gq) * B + m) * N * N;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int j = j0 + ty + 8 * k, i = i0 + tx;
        if (j < N && i < N) {
            const double2 t = tile[tx][ty + 8 * k];
            out[static_cast<size_t>(j) * N + i] = make_double2(acc[k].x + t.x, acc[k].y + t.y);
        }
    }
}

// ------------------------------------------------------------------------------------------ launcher
template <int MODE>
static cudaError_t launch_mode(int maxg, bool paired, const ProjArgs& A, int grid, int block, size_t smem,
                               cudaStream_t s)
{
    constexpr bool CP = MODE != MODE_JVP;   // the JVP is never line-paired
    if (A.var_cw) {   // model variant (N3): unpaired only
        if (maxg == 1) launch_k(proj_kernel<MODE, 1, false, true>, grid, block, smem, s, A);
        else launch_k(proj_kernel<MODE, 2, false, true>, grid, block, smem, s, A);
    } else if (paired && CP) {
        if (maxg == 1) launch_k(proj_kernel<MODE, 1, CP>, grid, block, smem, s, A);
        else launch_k(proj_kernel<MODE, 2, CP>, grid, block, smem, s, A);
    } else {
        if (maxg == 1) launch_k(proj_kernel<MODE, 1, false>, grid, block, smem, s, A);
        else launch_k(proj_kernel<MODE, 2, false>, grid, block, smem, s, A);
    }
    return cudaGetLastError();
}

cudaError_t launch_proj(int mode, int maxg, bool paired, const ProjArgs& A, int grid, int block, size_t smem,
                        cudaStream_t s)
{
    if (maxg != 1 && maxg != 2) return cudaErrorInvalidValue;
    switch (mode) {
    case MODE_FWD: return launch_mode<MODE_FWD>(maxg, paired, A, grid, block, smem, s);
    case MODE_JVP: return launch_mode<MODE_JVP>(maxg, paired, A, grid, block, smem, s);
    case MODE_VJP: return launch_mode<MODE_VJP>(maxg, paired, A, grid, block, smem, s);
    case MODE_GN: return launch_mode<MODE_GN>(maxg, paired, A, grid, block, smem, s);
    }
    return cudaErrorInvalidValue;
}

template <int MODE>
static cudaError_t launch_seg_mode(int phase, int maxg, bool paired, const ProjArgs& A, int grid, int block,
                                   size_t smem, cudaStream_t s)
{
    if (phase == 0) {
        if (paired) {
            if (block > 512) launch_k(seg_a_kernel<MODE, 1, true, true>, grid, block, smem, s, A);
            else if (maxg == 1) launch_k(seg_a_kernel<MODE, 1, true>, grid, block, smem, s, A);
            else launch_k(seg_a_kernel<MODE, 2, true>, grid, block, smem, s, A);
        } else {
            if (block > 512) launch_k(seg_a_kernel<MODE, 1, false, true>, grid, block, smem, s, A);
            else if (maxg == 1) launch_k(seg_a_kernel<MODE, 1, false>, grid, block, smem, s, A);
            else launch_k(seg_a_kernel<MODE, 2, false>, grid, block, smem, s, A);
        }
    } else {
        const bool cache = MODE == MODE_VJP && A.cache != nullptr;   // fused cache build (LM wrap)
        if (cache) {
            if (paired) launch_k(seg_b_kernel<MODE, true, MODE == MODE_VJP>, grid, block, smem, s, A);
            else launch_k(seg_b_kernel<MODE, false, MODE == MODE_VJP>, grid, block, smem, s, A);
        } else {
            if (paired) launch_k(seg_b_kernel<MODE, true, false>, grid, block, smem, s, A);
            else launch_k(seg_b_kernel<MODE, false, false>, grid, block, smem, s, A);
        }
    }
    return cudaGetLastError();
}

cudaError_t launch_seg(int phase, int mode, int maxg, bool paired, const ProjArgs& A, int grid, int block,
                       size_t smem, cudaStream_t s)
{
    if (maxg != 1 && maxg != 2) return cudaErrorInvalidValue;
    if (mode == MODE_JVP && phase == 0) {   // the standalone JVP: phase A only, unpaired
        if (block > 512) launch_k(seg_a_kernel<MODE_JVP, 1, false, true>, grid, block, smem, s, A);
        else if (maxg == 1) launch_k(seg_a_kernel<MODE_JVP, 1, false>, grid, block, smem, s, A);
        else launch_k(seg_a_kernel<MODE_JVP, 2, false>, grid, block, smem, s, A);
        return cudaGetLastError();
    }
    if (mode == MODE_FWD && phase == 0) {   // the standalone forward: plain sums, G and (paired) p2 only
        if (paired) {
            if (block > 512) launch_k(seg_a_kernel<MODE_FWD, 1, true, true>, grid, block, smem, s, A);
            else if (maxg == 1) launch_k(seg_a_kernel<MODE_FWD, 1, true>, grid, block, smem, s, A);
            else launch_k(seg_a_kernel<MODE_FWD, 2, true>, grid, block, smem, s, A);
        } else {
            if (block > 512) launch_k(seg_a_kernel<MODE_FWD, 1, false, true>, grid, block, smem, s, A);
            else if (maxg == 1) launch_k(seg_a_kernel<MODE_FWD, 1, false>, grid, block, smem, s, A);
            else launch_k(seg_a_kernel<MODE_FWD, 2, false>, grid, block, smem, s, A);
        }
        return cudaGetLastError();
    }
    if (mode == MODE_VJP) return launch_seg_mode<MODE_VJP>(phase, maxg, paired, A, grid, block, smem, s);
    if (mode == MODE_GN) return launch_seg_mode<MODE_GN>(phase, maxg, paired, A, grid, block, smem, s);
    return cudaErrorInvalidValue;
}

template <int MODE>
static cudaError_t seg_attr_mode(int phase, size_t smem)
{
    const int v = static_cast<int>(smem);
    cudaError_t e;
    if (phase == 0) {
        if ((e = raise_smem(seg_a_kernel<MODE, 1, true>, v))) return e;
        if ((e = raise_smem(seg_a_kernel<MODE, 2, true>, v))) return e;
        if ((e = raise_smem(seg_a_kernel<MODE, 1, true, true>, v))) return e;
        if ((e = raise_smem(seg_a_kernel<MODE, 1, false, true>, v))) return e;
        if ((e = raise_smem(seg_a_kernel<MODE, 1, false>, v))) return e;
        return raise_smem(seg_a_kernel<MODE, 2, false>, v);
    }
    if ((e = raise_smem(seg_b_kernel<MODE, true, false>, v))) return e;
    if ((e = raise_smem(seg_b_kernel<MODE, false, false>, v))) return e;
    if ((e = raise_smem(seg_b_kernel<MODE, true, MODE == MODE_VJP>, v))) return e;
    return raise_smem(seg_b_kernel<MODE, false, MODE == MODE_VJP>, v);
}

cudaError_t set_seg_smem_limit(int phase, int mode, size_t smem)
{
    if (mode == MODE_JVP) {
        const int v = static_cast<int>(smem);
        cudaError_t e = raise_smem(seg_a_kernel<MODE_JVP, 1, false>, v);
        if (e) return e;
        e = raise_smem(seg_a_kernel<MODE_JVP, 1, false, true>, v);
        if (e) return e;
        return raise_smem(seg_a_kernel<MODE_JVP, 2, false>, v);
    }
    if (mode == MODE_FWD && phase == 0) {
        const int v = static_cast<int>(smem);
        cudaError_t e;
        if ((e = raise_smem(seg_a_kernel<MODE_FWD, 1, true>, v))) return e;
        if ((e = raise_smem(seg_a_kernel<MODE_FWD, 2, true>, v))) return e;
        if ((e = raise_smem(seg_a_kernel<MODE_FWD, 1, true, true>, v))) return e;
        if ((e = raise_smem(seg_a_kernel<MODE_FWD, 1, false, true>, v))) return e;
        if ((e = raise_smem(seg_a_kernel<MODE_FWD, 1, false>, v))) return e;
        return raise_smem(seg_a_kernel<MODE_FWD, 2, false>, v);
    }
    if (mode == MODE_VJP) return seg_attr_mode<MODE_VJP>(phase, smem);
    if (mode == MODE_GN) return seg_attr_mode<MODE_GN>(phase, smem);
    return cudaErrorInvalidValue;
}

int proj_warps(int mode) { return (mode == MODE_VJP || mode == MODE_GN) ? 16 : 8; }   // the most
int proj_ctas_per_sm(int mode) { return mode == MODE_FWD ? 3 : (mode == MODE_JVP ? 2 : 1); }

template <int MODE>
static cudaError_t attr_mode(size_t smem)
{
    constexpr bool CP = MODE != MODE_JVP;
    const int v = static_cast<int>(smem);
    cudaError_t e;
    if ((e = raise_smem(proj_kernel<MODE, 1, false>, v))) return e;
    if ((e = raise_smem(proj_kernel<MODE, 2, false>, v))) return e;
    if ((e = raise_smem(proj_kernel<MODE, 1, CP>, v))) return e;
    if ((e = raise_smem(proj_kernel<MODE, 1, false, true>, v))) return e;
    if ((e = raise_smem(proj_kernel<MODE, 2, false, true>, v))) return e;
    return raise_smem(proj_kernel<MODE, 2, CP>, v);
}

cudaError_t set_proj_smem_limit(int mode, size_t smem)
{
    switch (mode) {
    case MODE_FWD: return attr_mode<MODE_FWD>(smem);
    case MODE_JVP: return attr_mode<MODE_JVP>(smem);
    case MODE_VJP: return attr_mode<MODE_VJP>(smem);
    case MODE_GN: return attr_mode<MODE_GN>(smem);
    }
    return cudaErrorInvalidValue;
}

}  // namespace pget
