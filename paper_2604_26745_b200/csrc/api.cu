// api.cu -- the extern "C" boundary of libpget (include/pget.h): argument
// validation, workspace carving, launch configuration and the LM-iteration
// orchestration (SURVEY.md §3 call stacks 1-3).  Everything is enqueued on the
// caller's stream; nothing here allocates, frees or synchronises except
// pget_geometry_create / pget_geometry_destroy.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <map>
#include <mutex>
#include <new>
#include <string>
#include <type_traits>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "internal.h"
#include "kernels.cuh"

using namespace pget;

namespace {

thread_local std::string g_err;

// NVTX range around every public entry point (SURVEY.md §5 tracing): visible in Nsight Systems / ncu
// --nvtx; a no-op without an attached tool (NVTX v3 is header-only)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

// ---- tracing (pget_profile_begin / pget_profile_end)
struct ProfRec {
    int mode;
    cudaEvent_t a, b;
};
struct Profiler {
    std::mutex mu;
    std::atomic<bool> on{false};
    std::atomic<long long> total{0};
    std::vector<cudaEvent_t> pool;
    size_t used = 0;
    std::vector<ProfRec> recs;
    long long mode_launches[4] = {0, 0, 0, 0};
};
Profiler g_prof;

inline void note()
{
    if (g_prof.on.load(std::memory_order_relaxed)) g_prof.total.fetch_add(1, std::memory_order_relaxed);
}

pget_status fail(pget_status s, const std::string& msg)
{
    g_err = msg;
    return s;
}

pget_status cuda_fail(cudaError_t e, const char* where)
{
    g_err = std::string(where) + ": " + cudaGetErrorString(e);
    return PGET_ERR_CUDA;
}

#define CK(expr)                                          \
    do {                                                  \
        cudaError_t e_ = (expr);                          \
        if (e_ != cudaSuccess) return cuda_fail(e_, #expr); \
    } while (0)

constexpr int kNblk = 64;      // blocks per member of every reduction kernel (fixed order)
constexpr int kVecThreads = 256;

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

struct ProjCfg {
    int kind;             // schedule: kSchedFwd / kSchedJvp / kSchedAdj
    int W, maxg, passesA, passesB, RbA, RbB, nbA, nbB, grid;   // W: warps per CTA of this geometry
    int G;                // fp64 partial images of the slot reduction (adjoint modes)
    bool paired;          // line-paired projector (forward / VJP / GN of a dup geometry)
    size_t smem;
    int stage_bytes, off_wacc, off_rout, off_gsh;
};

size_t align128(size_t x) { return (x + 127) & ~size_t(127); }

int sched_kind(int mode) { return mode == MODE_FWD ? kSchedFwd : (mode == MODE_JVP ? kSchedJvp : kSchedAdj); }

// Launch configuration of the projector for `mode`: warps and CTAs per SM
// are fixed per mode, the task schedule is the handle's (schedule.cpp); the band height is the
// largest (<= 32 rows) whose double-buffered stage, the warp accumulators (adjoint modes) and the
// per-ray arrays fit the per-CTA shared-memory budget.
ProjCfg proj_cfg(const Geometry& g, int mode)
{
    ProjCfg c;
    const int cps = proj_ctas_per_sm(mode);
    c.kind = sched_kind(mode);
    const Schedule& S = g.sch[c.kind];
    c.paired = g.pair && mode != MODE_JVP;
    const bool hasB = mode == MODE_VJP || mode == MODE_GN;
    const bool nf4 = mode == MODE_JVP || mode == MODE_GN;
    // Warps per CTA and ray groups per warp.  Every warp of a band should carry the same number of
    // groups (the band ends at a CTA barrier).  Adjoint modes: one register-resident group per warp
    // (<= 128 registers for up to 16 warps) and W = the group count divided evenly over the fewest
    // passes (config 2: 15 groups -> 15 warps, 1 pass; configs 3/4: 26 -> 13 warps, 2 passes).
    // Forward / JVP: 8 warps, up to 2 groups per warp.
    const int ncgA = S.max_gA, ncgB = hasB ? S.max_gB : 0;
    if (hasB) {
        const int gmax = std::max(ncgA, ncgB);
        const int passes = (gmax + proj_warps(mode) - 1) / proj_warps(mode);
        c.W = std::max(4, (gmax + passes - 1) / passes);
        c.maxg = 1;
    } else {
        c.W = proj_warps(mode);
        c.maxg = (ncgA + c.W - 1) / c.W >= 2 ? 2 : 1;
    }
    c.passesA = std::max(1, (ncgA + c.W * c.maxg - 1) / (c.W * c.maxg));
    c.passesB = std::max(1, (ncgB + c.W * c.maxg - 1) / (c.W * c.maxg));
    const int W = c.W;
    const size_t per_sm = 233472;   // 228 KB of shared memory per SM
    const size_t budget = std::min<size_t>(g.smem_optin, per_sm / cps - 1024);
    const size_t rout_b = align128(2 * sizeof(float) * g.R), gsh_b = align128(sizeof(float4) * g.R);
    const size_t fixed = 128 + rout_b + gsh_b;
    const size_t pixA = nf4 ? 16 : 8;
    int Rb = std::min(32, g.P - 1);
    size_t SB = 0, total = 0;
    for (; Rb >= 1; --Rb) {
        SB = align128(std::max<size_t>(static_cast<size_t>(Rb + 1) * g.P * pixA,
                                       hasB ? static_cast<size_t>(Rb + 1) * g.P * 8 : 0));
        total = fixed + 2 * SB + (hasB ? align128(static_cast<size_t>(W) * (Rb + 1) * g.P * 8) : 0);
        if (total <= budget) break;
    }
    if (Rb < 1) Rb = 1;
    c.RbA = c.RbB = Rb;
    c.nbA = c.nbB = (g.P - 1 + Rb - 1) / Rb;
    c.stage_bytes = static_cast<int>(SB);
    c.off_wacc = static_cast<int>(128 + 2 * SB);
    const size_t wacc_b = hasB ? align128(static_cast<size_t>(W) * (Rb + 1) * g.P * 8) : 0;
    c.off_rout = static_cast<int>(c.off_wacc + wacc_b);
    c.off_gsh = static_cast<int>(c.off_rout + rout_b);
    c.smem = c.off_gsh + gsh_b;
    c.grid = S.C > 0 ? S.C : g.sm_count * cps;
    // slot reduction: enough (tile, member, slot-range) blocks to fill the GPU twice
    {
        const int tiles = ((g.desc.n_px + 31) / 32) * ((g.desc.n_px + 31) / 32);
        const int64_t want = (2LL * g.sm_count + int64_t(tiles) * g.desc.batch - 1) / (int64_t(tiles) * g.desc.batch);
        int64_t wg = want;
        if (const char* ev = std::getenv("PGET_RED_G")) wg = std::max(1, std::atoi(ev));   // experiment
        c.G = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(wg, std::max(1, S.max_slots_member))));
        if (g.sid) c.G = 1;   // the pixel basis writes one fp64 partial (sid.cu)
    }
    return c;
}

int slot_pitch(const Geometry& g) { return (g.desc.n_px + 1) & ~1; }

// Launch configuration of the segmented adjoint.  Phase A: 16 warps,
// 1 CTA per SM (measured best of 4x4, 8x2, 8x1, 12x1, 16x1: scripts/sega_exp.sh), up to 2 groups of
// 32 adjacent rays per warp, shared memory = two float4 stage buffers.  Phase B: one CTA per SM, one comb group per warp (W = the group count over the fewest
// passes of <= 16 warps), shared memory = two float2 stages + the warps' band accumulators + the
// per-ray constants.  Band heights: the largest (<= 32 rows) that fits.
struct SegCfg {
    int WA, maxgA, passesA, RbA, gridA, stageA;
    size_t smemA;
    int WB, passesB, RbB, gridB, stageB, off_wacc, off_rout, off_gsh, off_rsc, off_q1;
    int RbG, off_waccG, off_routG;   // gnb_kernel: no stage buffers, so taller bands
    int WG, passesG;                 // gnb_kernel warps (one shared accumulator: up to 26, one pass) and passes
    size_t smemG;
    size_t smemB;
};

SegCfg seg_cfg(const Geometry& g)
{
    const Schedule& S = g.sch[kSchedAdj];
    SegCfg c;
    const int ngA = (g.R + 31) / 32;
    c.WA = g.segA_W;   // consumer warps (the kernel adds one producer warp)
    if (g.segA_wide && ngA > c.WA && ngA <= 26) c.WA = ngA;   // the 26-warp build: one group per warp
    c.maxgA = ngA > c.WA ? 2 : 1;
    c.passesA = std::max(1, (ngA + c.WA * c.maxgA - 1) / (c.WA * c.maxgA));
    const size_t per_sm = 233472;
    {
        const size_t budget = std::min<size_t>(g.smem_optin, per_sm / g.segA_cps - 1024);
        int Rb = std::min(g.rbA_cap, g.P - 1);
        size_t SB = 0;
        constexpr int kStagesA = kSegAStages;
        for (; Rb > 1; --Rb) {
            SB = align128(static_cast<size_t>(Rb + 1) * g.P * sizeof(float4));
            if (128 + kStagesA * SB <= budget) break;
        }
        SB = align128(static_cast<size_t>(Rb + 1) * g.P * sizeof(float4));
        c.RbA = Rb;
        c.stageA = static_cast<int>(SB);
        c.smemA = 128 + kStagesA * SB;
        c.gridA = S.CA > 0 ? S.CA : g.segA_cps * g.sm_count;
    }
    {
        const int ngB = std::max(1, S.max_gB);
        const int passes = (ngB + 15) / 16;
        c.WB = std::max(4, (ngB + passes - 1) / passes);
        c.passesB = (ngB + c.WB - 1) / c.WB;
        const size_t budget = std::min<size_t>(g.smem_optin, per_sm - 1024);
        const size_t rout_b = align128(2 * sizeof(float) * g.R), gsh_b = align128(sizeof(float4) * g.R);
        const size_t rsc_b = align128(sizeof(float) * g.R), q1_b = align128(sizeof(float2) * g.R);
        const size_t fixed = 128 + rout_b + gsh_b + rsc_b + q1_b;
        int Rb = std::min(32, g.P - 1);
        size_t SB = 0, wacc = 0;
        for (; Rb > 1; --Rb) {
            SB = align128(static_cast<size_t>(Rb + 1) * g.P * sizeof(float2));
            wacc = align128(static_cast<size_t>(c.WB) * (Rb + 1) * g.P * sizeof(float2));
            if (fixed + 2 * SB + wacc <= budget) break;
        }
        SB = align128(static_cast<size_t>(Rb + 1) * g.P * sizeof(float2));
        wacc = align128(static_cast<size_t>(c.WB) * (Rb + 1) * g.P * sizeof(float2));
        c.RbB = Rb;
        c.stageB = static_cast<int>(SB);
        c.off_wacc = static_cast<int>(128 + 2 * SB);
        c.off_rout = static_cast<int>(c.off_wacc + wacc);
        c.off_gsh = static_cast<int>(c.off_rout + rout_b);
        c.off_rsc = static_cast<int>(c.off_gsh + gsh_b);
        c.off_q1 = static_cast<int>(c.off_rsc + rsc_b);
        c.smemB = c.off_q1 + q1_b;
        c.gridB = S.C > 0 ? S.C : g.sm_count;
        {
            int Rbg = std::min(32, g.P - 1);
            size_t wg = 0;
            for (; Rbg > 1; --Rbg) {
                wg = align128(static_cast<size_t>(c.WB) * (Rbg + 1) * g.P * sizeof(float2));
                if (128 + wg + rout_b <= budget) break;
            }
            wg = align128(static_cast<size_t>(c.WB) * (Rbg + 1) * g.P * sizeof(float2));
            c.RbG = g.gnb_tall ? Rbg : c.RbB;
            c.off_waccG = g.gnb_tall ? 128 : c.off_wacc;
            c.off_routG = g.gnb_tall ? static_cast<int>(128 + wg) : c.off_rout;
            c.smemG = g.gnb_tall ? 128 + wg + rout_b : c.smemB;
            if (g.gnb_int && g.gn_hybrid) {   // one shared accumulator: bands up to a whole segment
                int maxseg = 1;
                for (size_t k = 0; k + 1 < S.seg_rows.size(); ++k)
                    maxseg = std::max(maxseg, S.seg_rows[k + 1] - S.seg_rows[k]);
                // no more shared memory than a segment needs: the rest stays L1 for the entry stream
                int Rbi = std::min(g.P - 1, maxseg);
                size_t wi = 0;
                for (; Rbi > 1; --Rbi) {
                    wi = align128(static_cast<size_t>(Rbi + 1) * g.P * sizeof(int2));
                    if (128 + wi + rout_b <= budget) break;
                }
                wi = align128(static_cast<size_t>(Rbi + 1) * g.P * sizeof(int2));
                c.RbG = Rbi;
                c.off_waccG = 128;
                c.off_routG = static_cast<int>(128 + wi);
                c.smemG = 128 + wi + rout_b;
            }
            // the fixed-point scatter keeps one accumulator whatever the warp count: with 17-26 comb
            // groups every group gets its own warp (one pass) in the 26-warp build of gnb_kernel
            c.WG = c.WB;
            c.passesG = c.passesB;
            if (g.gnb_int && g.gn_hybrid && g.gnb_wide && ngB > 16 && ngB <= 26) {
                c.WG = ngB;
                c.passesG = 1;
            }
        }
    }
    return c;
}

ProjArgs base_args(const Geometry& g, const ProjCfg& c)
{
    ProjArgs A;
    std::memset(&A, 0, sizeof A);
    const Schedule& S = g.sch[c.kind];
    A.rays = g.d_rays;
    A.tasks = S.d_tasks;
    A.cta_begin = S.d_cta_begin;
    A.groups = S.d_groups;
    A.w = g.var ? g.d_ones : g.d_w;   // variant: the response W_j(d_i) is inside the ray sums (A.var_cw)
    A.var_cw = static_cast<const float2*>(g.d_var_cw);
    A.n_t = g.n_t;
    A.N = g.desc.n_px;
    A.Ns = slot_pitch(g);
    A.P = g.P;
    A.n_det = g.desc.n_det;
    A.J = g.desc.n_subrays;
    A.R = g.R;
    A.n_ab = g.n_ab;
    A.dup_half = g.dup ? g.desc.n_angles / 2 : 0;
    A.B = g.desc.batch;
    A.RbA = c.RbA;
    A.RbB = c.RbB;
    A.nbA = c.nbA;
    A.nbB = c.nbB;
    A.passesA = c.passesA;
    A.passesB = c.passesB;
    A.stage_bytes = c.stage_bytes;
    A.off_wacc = c.off_wacc;
    A.off_rout = c.off_rout;
    A.off_gsh = c.off_gsh;
    A.P4 = 4 * g.P;
    A.P8 = 8 * g.P;
    A.P16 = 16 * g.P;
    A.planeB4 = 4 * (A.RbB + 1) * g.P;
    A.delta = static_cast<float>(g.delta);
    const double cf = -g.delta * 1.4426950408889634;   // -Delta log2(e)
    A.cf = static_cast<float>(cf);
    A.ch = static_cast<float>(0.5 * cf);
    return A;
}

// the pixel basis (N3, R-pb): kernel arguments from the packed images (and outputs) of A
SidArgs sid_args(const Geometry& g, const ProjArgs& A)
{
    SidArgs S;
    std::memset(&S, 0, sizeof S);
    S.dir = g.d_sdir;
    S.off = g.d_soff;
    S.img2 = A.img2[0];
    S.img4 = A.img4[0];
    S.wj = g.var ? g.d_ones : g.d_w;
    S.dj2 = g.d_sdj2;
    S.y = A.y;
    S.dy = A.dy;
    S.win = A.win;
    S.nhits = g.sid_nhits;
    S.det_radius = g.desc.det_radius;
    S.c_slope = static_cast<float>(g.desc.c_slope);
    S.r_slope = static_cast<float>(g.desc.r_slope);
    S.sig0 = static_cast<float>(g.desc.subray_sigma * 2.0 / static_cast<double>(g.desc.n_det - 1));
    S.lmax = static_cast<float>(std::sqrt(2.0) * g.h * (1.0 + 1e-6));
    S.N = g.desc.n_px;
    S.P = g.P;
    S.R = g.R;
    S.J = g.desc.n_subrays;
    S.n_det = g.desc.n_det;
    S.n_ab = g.n_ab;
    S.nB = g.desc.n_banks;
    S.B = g.desc.batch;
    return S;
}

pget_status run_proj(const Geometry& g, int mode, const ProjCfg& c, const ProjArgs& A, cudaStream_t s)
{
    cudaEvent_t ea = nullptr, eb = nullptr;
    if (g_prof.on.load(std::memory_order_relaxed)) {
        std::lock_guard<std::mutex> lk(g_prof.mu);
        g_prof.total++;
        g_prof.mode_launches[mode]++;
        if (g_prof.used + 2 <= g_prof.pool.size()) {
            ea = g_prof.pool[g_prof.used++];
            eb = g_prof.pool[g_prof.used++];
            g_prof.recs.push_back({mode, ea, eb});
        }
    }
    if (ea) cudaEventRecord(ea, s);
    cudaError_t e = g.sid ? launch_sid_proj(mode, g.var, sid_args(g, A), s)
                          : launch_proj(mode, c.maxg, c.paired, A, c.grid, c.W * 32, c.smem, s);
    if (eb) cudaEventRecord(eb, s);
    if (e != cudaSuccess) return cuda_fail(e, "projector launch");
    return PGET_OK;
}

// the segmented adjoint: phase A then phase B on s, bracketed together by the profiler's events
pget_status run_seg(const Geometry& g, int mode, ProjArgs A, float* segp, cudaStream_t s, float4* cache = nullptr,
                    bool have_a = false, float* gscale = nullptr)
{
    const Schedule& S = g.sch[kSchedAdj];
    const SegCfg c = seg_cfg(g);
    cudaEvent_t ea = nullptr, eb = nullptr;
    if (g_prof.on.load(std::memory_order_relaxed)) {
        std::lock_guard<std::mutex> lk(g_prof.mu);
        g_prof.total += 2;
        g_prof.mode_launches[mode]++;
        if (g_prof.used + 2 <= g_prof.pool.size()) {
            ea = g_prof.pool[g_prof.used++];
            eb = g_prof.pool[g_prof.used++];
            g_prof.recs.push_back({mode, ea, eb});
        }
    }
    A.segp = segp;
    A.cache = cache;   // VJP: also write the GN Jacobian-entry cache (fused lin_kernel)
    A.gscale = cache ? gscale : nullptr;
    A.cellmax = g.cellmax;
    A.cache_off = S.d_cache_off;   // the fused builder writes the comb-group layout of its own scatter
    A.cache_rows_member = S.cache_rows_member;
    A.cache_ng = S.max_gB;
    A.ntab = S.ntab;
    A.slot_lo = S.d_slot_lo;
    A.slot_hi = S.d_slot_hi;
    A.K = S.K;
    A.seg_rows = S.d_seg_rows;
    A.n_groups = S.max_gB;
    A.groups = S.d_groups;
    if (ea) cudaEventRecord(ea, s);
    // phase A
    A.units = S.d_unitsA;
    A.u_begin = S.d_ua_begin;
    A.stages = S.d_stA;
    A.s_begin = S.d_sa_begin;
    A.RbA = c.RbA;
    A.passesA = c.passesA;
    A.stage_bytes = c.stageA;
    // have_a: segp already holds this u's VJP-mode phase-A partials (the segmented forward of the same
    // u wrote them), so only phase B runs
    cudaError_t e = have_a ? cudaSuccess : launch_seg(0, mode, c.maxgA, g.pair, A, c.gridA, (c.WA + 1) * 32, c.smemA, s);
    if (e == cudaSuccess) {
        A.units = S.d_unitsB;
        A.u_begin = S.d_ub_begin;
        A.stages = S.d_stB;
        A.s_begin = S.d_sb_begin;
        A.RbB = c.RbB;
        A.passesB = c.passesB;
        A.stage_bytes = c.stageB;
        A.off_wacc = c.off_wacc;
        A.off_rout = c.off_rout;
        A.off_gsh = c.off_gsh;
        A.off_rsc = c.off_rsc;
        A.off_q1 = c.off_q1;
        e = launch_seg(1, mode, 1, g.pair, A, c.gridB, c.WB * 32, c.smemB, s);
    }
    if (eb) cudaEventRecord(eb, s);
    if (e != cudaSuccess) return cuda_fail(e, "segmented projector launch");
    return PGET_OK;
}

// the three schedules of a handle on the host (sm_count CTAs per SM-count, the kernels' CTAs per SM)
void build_host_schedules(Geometry& g, const std::vector<RayP>& rays)
{
    for (int k = 0; k < 3; ++k) {
        const int mode = k == kSchedFwd ? MODE_FWD : (k == kSchedJvp ? MODE_JVP : MODE_VJP);
        Schedule& S = g.sch[k];
        if (k == kSchedAdj && g.adj_seg) {
            build_adj_schedule(g, rays, g.segA_cps * g.sm_count, g.sm_count, &S);
            const SegCfg sc = seg_cfg(g);
            build_adj_stages(sc.RbA, sc.passesA, sc.RbB, sc.passesB, &S);
            const double cache_gb = static_cast<double>(g.desc.batch) * std::max(S.cache_rows_member, S.cache_rows_memberC) *
                                    32 * sizeof(float4) / 1e9;
            if (cache_gb > g.cache_max_gb) g.gn_cached = false;
        } else {
            build_schedule(g, k, g.sm_count * proj_ctas_per_sm(mode), &S);
        }
    }
    if (g.adj_seg && g.jvp_seg) {   // segmented standalone JVP (phase A only)
        build_adj_schedule(g, rays, g.segA_cps * g.sm_count, g.sm_count, &g.schJ, true);
        const SegCfg sc = seg_cfg(g);
        build_adj_stages(sc.RbA, sc.passesA, sc.RbB, sc.passesB, &g.schJ);
    }
}

// ---- workspace carving
struct WS {
    float2* img2[2] = {nullptr, nullptr};
    float4* img4[2] = {nullptr, nullptr};
    float2* slots = nullptr;
    double2* gacc = nullptr;  // [G][B][N][N] fp64 partial gradients (g_lam, g_mu), G = ProjCfg::G
    float* segp = nullptr;    // segmented adjoint: [n_canon][kSegFields][R] phase-A partial sums
    float* segpJ = nullptr;   // segmented standalone JVP: [n_canonJ][kSegFields][R]
    float4* cache = nullptr;  // GN with cached Jacobian entries: [B][rows][32]
    float* jp = nullptr;      // [n_canon][2][R] per-segment (J p) partials
    float* gscale = nullptr;  // [B * ntab][8] fixed-point scale bounds (gnb_kernel INTACC)
    float *ysino = nullptr, *dysino = nullptr;
    float *bl = nullptr, *bm = nullptr, *zl = nullptr, *zm = nullptr, *pl = nullptr, *pm = nullptr;
    float *ql = nullptr, *qm = nullptr, *ul = nullptr, *um = nullptr;
    float *sl = nullptr, *sm = nullptr, *beta = nullptr;   // pget_lm_solve
    double* part = nullptr;   // [8][B][kNblk]
    CGState* cg = nullptr;
    // pixel basis (sid.cu): per-ray adjoint weights and sums, bounds, 64-bit fixed-point accumulator
    float4* sray = nullptr;
    float2* sraybd = nullptr;
    unsigned* sbound = nullptr;
    unsigned long long* sacc = nullptr;
    size_t bytes = 0;
};

WS carve(const Geometry& g, int op, char* base)
{
    WS w;
    size_t off = 0;
    const size_t B = g.desc.batch;
    const size_t img = B * g.P * g.P;
    const size_t n2 = B * g.desc.n_px * g.desc.n_px;
    const size_t ns = B * g.n_ab * g.desc.n_det;
    auto take = [&](size_t bytes) -> char* {
        char* p = base ? base + off : nullptr;
        off += align256(bytes);
        return p;
    };
    const bool guard = op == PGET_OP_SAFEGUARD;
    const bool lm = op == PGET_OP_GN_CG_STEP || op == PGET_OP_LM_SOLVE;
    const bool need2 = op == PGET_OP_FORWARD || op == PGET_OP_VJP || op == PGET_OP_GN_APPLY || lm || guard;
    const bool need4 = op == PGET_OP_JVP || op == PGET_OP_GN_APPLY || lm || guard;
    const bool needacc = op == PGET_OP_VJP || op == PGET_OP_GN_APPLY || lm;
    for (int k = 0; k < 2; ++k) {
        if (need2) w.img2[k] = reinterpret_cast<float2*>(take(img * sizeof(float2)));
        if (need4) w.img4[k] = reinterpret_cast<float4*>(take(img * sizeof(float4)));
    }
    if (needacc) {
        const ProjCfg c = proj_cfg(g, MODE_VJP);   // VJP and GN share the adjoint schedule
        const size_t plane = static_cast<size_t>(g.desc.n_px) * slot_pitch(g);
        w.slots = reinterpret_cast<float2*>(take(static_cast<size_t>(std::max(1, g.sch[kSchedAdj].n_slots)) * plane *
                                                 sizeof(float2)));
        w.gacc = reinterpret_cast<double2*>(take(static_cast<size_t>(c.G) * n2 * sizeof(double2)));
        if (g.sid) {
            const size_t nr = B * g.n_ab * static_cast<size_t>(g.R);
            w.sray = reinterpret_cast<float4*>(take(nr * sizeof(float4)));
            w.sraybd = reinterpret_cast<float2*>(take(nr * sizeof(float2)));
            w.sbound = reinterpret_cast<unsigned*>(take(2 * B * sizeof(unsigned)));
            w.sacc = reinterpret_cast<unsigned long long*>(take(2 * n2 * sizeof(unsigned long long)));
        }
        if (g.adj_seg)
            w.segp = reinterpret_cast<float*>(take(static_cast<size_t>(g.sch[kSchedAdj].n_canon) * kSegFields *
                                                   g.R * sizeof(float)));
        const bool uses_cache = op == PGET_OP_GN_CG_STEP || op == PGET_OP_LM_SOLVE ||
                                (op == PGET_OP_GN_APPLY && g.gn_apply_cached);
        if (g.adj_seg && g.gn_cached && uses_cache) {
            const Schedule& S = g.sch[kSchedAdj];
            w.cache = reinterpret_cast<float4*>(
                take((static_cast<size_t>(B) * std::max(S.cache_rows_member, S.cache_rows_memberC) + kCachePadRows) *
                     32 * sizeof(float4)));
            w.jp = reinterpret_cast<float*>(take(static_cast<size_t>(S.n_canon) * 2 * g.R * sizeof(float)));
            if (g.gnb_int && g.gn_hybrid)
                w.gscale = reinterpret_cast<float*>(take(static_cast<size_t>(B) * S.ntab * 8 * sizeof(float)));
        }
    }
    if ((op == PGET_OP_FORWARD || guard) && g.adj_seg && g.fwd_seg)   // the segmented forward's partials
        w.segp = reinterpret_cast<float*>(take(static_cast<size_t>(g.sch[kSchedAdj].n_canon) * kSegFields *
                                               g.R * sizeof(float)));
    if ((op == PGET_OP_JVP || guard) && g.adj_seg && g.jvp_seg)
        w.segpJ = reinterpret_cast<float*>(take(static_cast<size_t>(g.schJ.n_canon) * kSegFields * g.R * sizeof(float)));
    if (op == PGET_OP_GN_CG_STEP || op == PGET_OP_LM_SOLVE) {
        w.ysino = reinterpret_cast<float*>(take(ns * sizeof(float)));
        w.dysino = reinterpret_cast<float*>(take(ns * sizeof(float)));
        float** vecs[] = {&w.bl, &w.bm, &w.zl, &w.zm, &w.pl, &w.pm, &w.ql, &w.qm, &w.ul, &w.um};
        for (float** v : vecs) *v = reinterpret_cast<float*>(take(n2 * sizeof(float)));
        w.part = reinterpret_cast<double*>(take(9 * B * kNblk * sizeof(double)));   // [8]: priors
        w.cg = reinterpret_cast<CGState*>(take(2 * B * sizeof(CGState)));   // double-buffered (cg_fused_kernel)
        if (op == PGET_OP_LM_SOLVE) {   // the step, per-member beta
            w.sl = reinterpret_cast<float*>(take(n2 * sizeof(float)));
            w.sm = reinterpret_cast<float*>(take(n2 * sizeof(float)));
            w.beta = reinterpret_cast<float*>(take(B * sizeof(float)));
        }
    }
    if (guard) {
        w.ysino = reinterpret_cast<float*>(take(ns * sizeof(float)));
        w.dysino = reinterpret_cast<float*>(take(ns * sizeof(float)));
        w.zl = reinterpret_cast<float*>(take(n2 * sizeof(float)));
        w.zm = reinterpret_cast<float*>(take(n2 * sizeof(float)));
        w.part = reinterpret_cast<double*>(take(18 * B * kNblk * sizeof(double)));   // [12..17]: priors
    }
    w.bytes = off;
    return w;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// every pointer argument: non-NULL, 16-byte aligned, CUDA device (or managed) memory of the handle's device
pget_status check_ptrs(std::initializer_list<const void*> ptrs, const char* what, int device)
{
    for (const void* p : ptrs) {
        if (!p) return fail(PGET_ERR_INVALID_ARGUMENT, std::string(what) + ": NULL device pointer");
        if (!aligned16(p)) return fail(PGET_ERR_ALIGNMENT, std::string(what) + ": pointer not 16-byte aligned");
        cudaPointerAttributes at;
        if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
            cudaGetLastError();   // clear the sticky-free error state of the failed query
            return fail(PGET_ERR_INVALID_ARGUMENT, std::string(what) + ": pointer is not CUDA memory");
        }
        if (at.type == cudaMemoryTypeManaged) continue;
        if (at.type != cudaMemoryTypeDevice)
            return fail(PGET_ERR_INVALID_ARGUMENT, std::string(what) + ": pointer is not device memory");
        if (at.device != device)
            return fail(PGET_ERR_INVALID_ARGUMENT, std::string(what) + ": pointer on another device");
    }
    return PGET_OK;
}

pget_status check_common(pget_geometry h, int op, void* ws, size_t ws_bytes, WS* w)
{
    if (!h) return fail(PGET_ERR_INVALID_ARGUMENT, "NULL geometry handle");
    if (h->g.device < 0) return fail(PGET_ERR_INVALID_ARGUMENT, "host-only geometry handle (device < 0)");
    int dev = -1;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    if (dev != h->g.device)
        return fail(PGET_ERR_INVALID_ARGUMENT, "current CUDA device differs from the geometry's device");
    const WS need = carve(h->g, op, nullptr);
    if (ws_bytes < need.bytes) return fail(PGET_ERR_WORKSPACE, "workspace too small");
    if (need.bytes && (!ws || !aligned16(ws))) return fail(PGET_ERR_WORKSPACE, "workspace NULL or misaligned");
    *w = carve(h->g, op, static_cast<char*>(ws));
    return PGET_OK;
}

int vec_grid(size_t n)
{
    return static_cast<int>(std::max<size_t>(1, std::min<size_t>(1184, (n + kVecThreads - 1) / kVecThreads)));
}

}  // namespace

void free_device_tables(Geometry* g)
{
    cudaFree(g->d_rays);
    cudaFree(g->d_w);
    cudaFree(g->d_ones);
    cudaFree(g->d_var_cw);
    g->d_rays = nullptr;
    g->d_w = nullptr;
    g->d_ones = nullptr;
    g->d_var_cw = nullptr;
    cudaFree(g->d_sdir);
    cudaFree(g->d_soff);
    cudaFree(g->d_sdj2);
    g->d_sdir = g->d_soff = nullptr;
    g->d_sdj2 = nullptr;
    for (Schedule& S : g->sch) {
        cudaFree(S.d_cta_begin); cudaFree(S.d_tasks); cudaFree(S.d_groups); cudaFree(S.d_red_off); cudaFree(S.d_red_slot);
        S.d_cta_begin = nullptr; S.d_tasks = nullptr; S.d_groups = nullptr; S.d_red_off = nullptr; S.d_red_slot = nullptr;
        cudaFree(S.d_slot_lo); cudaFree(S.d_slot_hi);
        S.d_slot_lo = S.d_slot_hi = nullptr;
        cudaFree(S.d_unitsA); cudaFree(S.d_unitsB); cudaFree(S.d_ua_begin); cudaFree(S.d_ub_begin);
        cudaFree(S.d_sa_begin); cudaFree(S.d_sb_begin); cudaFree(S.d_stA); cudaFree(S.d_stB); cudaFree(S.d_seg_rows);
        cudaFree(S.d_cache_off);
        S.d_cache_off = nullptr;
        cudaFree(S.d_groupsC);
        cudaFree(S.d_cache_offC);
        S.d_groupsC = nullptr;
        S.d_cache_offC = nullptr;
    }
    {
        Schedule& S = g->schJ;
        cudaFree(S.d_unitsA); cudaFree(S.d_ua_begin); cudaFree(S.d_stA); cudaFree(S.d_sa_begin); cudaFree(S.d_seg_rows);
        S.d_unitsA = nullptr; S.d_ua_begin = S.d_sa_begin = S.d_seg_rows = nullptr; S.d_stA = nullptr;
        cudaFree(g->d_tabsJ);
        g->d_tabsJ = nullptr;
        cudaFree(g->d_tabsA);
        g->d_tabsA = nullptr;
        S.d_unitsA = S.d_unitsB = nullptr;
        S.d_ua_begin = S.d_ub_begin = S.d_sa_begin = S.d_sb_begin = S.d_seg_rows = nullptr;
        S.d_stA = S.d_stB = nullptr;
    }
}

// =========================================================================================== C ABI
extern "C" {

const char* pget_status_string(pget_status s)
{
    switch (s) {
    case PGET_OK: return "PGET_OK";
    case PGET_ERR_INVALID_ARGUMENT: return "PGET_ERR_INVALID_ARGUMENT";
    case PGET_ERR_SHAPE: return "PGET_ERR_SHAPE";
    case PGET_ERR_ALIGNMENT: return "PGET_ERR_ALIGNMENT";
    case PGET_ERR_WORKSPACE: return "PGET_ERR_WORKSPACE";
    case PGET_ERR_OUT_OF_MEMORY: return "PGET_ERR_OUT_OF_MEMORY";
    case PGET_ERR_CUDA: return "PGET_ERR_CUDA";
    case PGET_ERR_NOT_FINITE: return "PGET_ERR_NOT_FINITE";
    }
    return "PGET_ERR_UNKNOWN";
}

const char* pget_last_error_message(void) { return g_err.c_str(); }

pget_status pget_geometry_create(const pget_geometry_desc* desc, int device, pget_geometry* out)
{
    NvtxRange nvtx_("pget_geometry_create");
    if (!out) return fail(PGET_ERR_INVALID_ARGUMENT, "out is NULL");
    *out = nullptr;
    pget_geometry h = new (std::nothrow) pget_geometry_s;
    if (!h) return fail(PGET_ERR_OUT_OF_MEMORY, "host allocation failed");
    std::string err;
    pget_status st = build_geometry(desc, &h->g, &err);
    if (st != PGET_OK) { delete h; return fail(st, err); }
    Geometry& g = h->g;
    if (g.desc.n_px > 2048) { delete h; return fail(PGET_ERR_INVALID_ARGUMENT, "n_px > 2048 not supported"); }
    g.device = device;
    if (const char* ev = std::getenv("PGET_NO_PAIR")) g.pair = g.pair && std::atoi(ev) == 0;   // experiments
    // the model variant (N3): its attenuation exp(-c_i A_i) does not factor along a ray, so it runs the
    // whole-ray (fused) projectors, unpaired, with the recomputed GN product
    auto variant_paths = [&g]() {
        if (!g.var && !g.sid) return;   // the pixel basis (R-pb) likewise: whole rays, sid.cu
        g.adj_seg = g.jvp_seg = g.fwd_seg = false;
        g.gn_cached = false;
        g.pair = false;
    };
    if (device < 0) {   // host-only handle: tables, info and the host schedules; no device tables, no compute
        variant_paths();
        std::vector<RayP> rays;
        build_ray_params(g, &rays);
        build_host_schedules(g, rays);
        *out = h;
        return PGET_OK;
    }
    int prev = -1;
    cudaError_t e = cudaGetDevice(&prev);
    if (e == cudaSuccess) e = cudaSetDevice(device);
    int optin = 0;
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&g.sm_count, cudaDevAttrMultiProcessorCount, device);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    if (e == cudaSuccess) g.smem_optin = static_cast<size_t>(optin);
    int coop = 0, per_sm = 0;
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device);
    if (e == cudaSuccess && !coop) e = cudaErrorNotSupported;
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cg_fused_kernel, kVecThreads, 0);
    if (e == cudaSuccess) g.cg_coop_blocks = std::max(1, per_sm) * g.sm_count;
    std::vector<RayP> rays;
    build_ray_params(g, &rays);
    if (e == cudaSuccess) e = cudaMalloc(&g.d_rays, rays.size() * sizeof(RayP));
    if (const char* ev = std::getenv("PGET_ADJ_FUSED")) g.adj_seg = std::atoi(ev) == 0;   // A/B experiments
    if (const char* ev = std::getenv("PGET_JVP_FUSED")) g.jvp_seg = std::atoi(ev) == 0;
    if (const char* ev = std::getenv("PGET_FWD_FUSED")) g.fwd_seg = std::atoi(ev) == 0;
    if (const char* ev = std::getenv("PGET_FWD_PLAIN")) g.fwd_plain = std::atoi(ev) != 0;
    if (const char* ev = std::getenv("PGET_CG_PDL")) g.cg_pdl = std::atoi(ev) != 0;
    if (const char* ev = std::getenv("PGET_FWD_PLAIN_TRIAL")) g.fwd_plain_trial = std::atoi(ev) != 0;
    g.gnb_tall = g.P >= 200;   // measured: config 4 -3.6 % LM, config 2 +0.8 %
    if (const char* ev = std::getenv("PGET_GNB_TALL")) g.gnb_tall = std::atoi(ev) != 0;
    if (const char* ev = std::getenv("PGET_GNB_INT")) g.gnb_int = g.gnb_int && std::atoi(ev) != 0;
    if (const char* ev = std::getenv("PGET_GNB_WIDE")) g.gnb_wide = std::atoi(ev) != 0;
    // the cached GN path over consecutive-ray groups (measured: LM config 2 -0.6 %, config 3 -3 %, config
    // 4 -1 %; config 5's 64 members: +3.5 % with groups of 32 consecutive rays, -3.4 % (206.8 -> 199.7 ms)
    // with the interleaved groups of stride 2); PGET_GNB_ADJ=0/1 overrides
    g.gnb_adj = true;
    if (const char* ev = std::getenv("PGET_GNB_ADJ")) g.gnb_adj = std::atoi(ev) != 0;
    if (const char* ev = std::getenv("PGET_SEGA_WIDE")) g.segA_wide = std::atoi(ev) != 0;
    if (const char* ev = std::getenv("PGET_GNB_STRIDE")) g.gnbC_stride = std::max(1, std::min(16, std::atoi(ev)));
    if (const char* ev = std::getenv("PGET_GN_APPLY_CACHED")) g.gn_apply_cached = std::atoi(ev) != 0;
    if (const char* ev = std::getenv("PGET_GN_CACHE_MAX_GB")) g.cache_max_gb = std::atof(ev);
    if (const char* ev = std::getenv("PGET_GN_CACHE")) {   // 0: recompute, 1: hybrid, 2: fully cached
        const int v = std::atoi(ev);
        g.gn_cached = v != 0;
        g.gn_hybrid = v == 1;
    }
    if (const char* ev = std::getenv("PGET_RBA_CAP")) g.rbA_cap = std::max(4, std::min(128, std::atoi(ev)));
    if (const char* ev = std::getenv("PGET_SEGA_W")) g.segA_W = std::max(1, std::min(15, std::atoi(ev)));
    if (const char* ev = std::getenv("PGET_SEGA_CPS")) g.segA_cps = std::max(1, std::min(4, std::atoi(ev)));
    if ((g.segA_W + 1) * 32 * g.segA_cps > 2048) g.segA_cps = 2048 / ((g.segA_W + 1) * 32);
    variant_paths();
    g.gnb_adj = g.gnb_adj && g.gnb_int && g.gn_hybrid;   // the float accumulators need comb lanes
    // the coefficient cache while it stays well inside HBM (config 2: 0.4 GB, config 4: 2.7 GB,
    // config 5's 64 assemblies: 25 GB of 180; measured: config 5 LM iteration 307 -> 210 ms)
    build_host_schedules(g, rays);
    for (int k = 0; k < 3 && e == cudaSuccess; ++k) {
        Schedule& S = g.sch[k];
        auto up = [&](auto** dst, const auto& v) {
            using T = typename std::remove_reference<decltype(v)>::type::value_type;
            if (e == cudaSuccess) e = cudaMalloc(dst, std::max<size_t>(1, v.size()) * sizeof(T));
            if (e == cudaSuccess && !v.empty()) e = cudaMemcpy(*dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
        };
        up(&S.d_cta_begin, S.cta_begin);
        up(&S.d_tasks, S.tasks);
        up(&S.d_groups, S.groups);
        up(&S.d_red_off, S.red_off);
        up(&S.d_red_slot, S.red_slot);
        up(&S.d_slot_lo, S.slot_lo);
        up(&S.d_slot_hi, S.slot_hi);
        if (k == kSchedAdj && g.adj_seg) {
            up(&S.d_unitsA, S.unitsA);
            up(&S.d_unitsB, S.unitsB);
            up(&S.d_ua_begin, S.ua_begin);
            up(&S.d_ub_begin, S.ub_begin);
            up(&S.d_stA, S.stA);
            up(&S.d_stB, S.stB);
            up(&S.d_sa_begin, S.sa_begin);
            up(&S.d_sb_begin, S.sb_begin);
            up(&S.d_seg_rows, S.seg_rows);
            up(&S.d_cache_off, S.cache_off);
            up(&S.d_groupsC, S.groupsC);
            up(&S.d_cache_offC, S.cache_offC);
        }
    }
    if (g.adj_seg && g.jvp_seg) {
        Schedule& S = g.schJ;
        auto up = [&](auto** dst, const auto& v) {
            using T = typename std::remove_reference<decltype(v)>::type::value_type;
            if (e == cudaSuccess) e = cudaMalloc(dst, std::max<size_t>(1, v.size()) * sizeof(T));
            if (e == cudaSuccess && !v.empty()) e = cudaMemcpy(*dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
        };
        up(&S.d_unitsA, S.unitsA);
        up(&S.d_ua_begin, S.ua_begin);
        up(&S.d_stA, S.stA);
        up(&S.d_sa_begin, S.sa_begin);
        up(&S.d_seg_rows, S.seg_rows);
        up(&g.d_tabsJ, g.task_ab);
    }
    if (g.adj_seg && e == cudaSuccess) {   // traced angle-banks of the adjoint schedule (segmented forward)
        const std::vector<int32_t>& lst = g.pair ? g.task_ab_p : g.task_ab;
        e = cudaMalloc(&g.d_tabsA, std::max<size_t>(1, lst.size()) * sizeof(int32_t));
        if (e == cudaSuccess && !lst.empty())
            e = cudaMemcpy(g.d_tabsA, lst.data(), lst.size() * sizeof(int32_t), cudaMemcpyHostToDevice);
    }
    if (e == cudaSuccess) e = cudaMalloc(&g.d_w, g.wf.size() * sizeof(float));
    if (e == cudaSuccess && g.var) {   // the variant's tables as float (W_j(d_i), c_i) and unit weights
        std::vector<float2> cw(g.var_w.size());
        for (int j = 0; j < g.desc.n_subrays; ++j)
            for (int i = 0; i < g.n_t; ++i)
                cw[static_cast<size_t>(j) * g.n_t + i] =
                    make_float2(static_cast<float>(g.var_w[static_cast<size_t>(j) * g.n_t + i]), static_cast<float>(g.var_c[i]));
        const std::vector<float> ones(g.wf.size(), 1.0f);
        e = cudaMalloc(&g.d_var_cw, cw.size() * sizeof(float2));
        if (e == cudaSuccess) e = cudaMemcpy(g.d_var_cw, cw.data(), cw.size() * sizeof(float2), cudaMemcpyHostToDevice);
        if (e == cudaSuccess) e = cudaMalloc(&g.d_ones, ones.size() * sizeof(float));
        if (e == cudaSuccess) e = cudaMemcpy(g.d_ones, ones.data(), ones.size() * sizeof(float), cudaMemcpyHostToDevice);
    }
    if (e == cudaSuccess && g.sid) {   // the pixel basis: fp64 O1 dirs and offsets, delta_j^2 log2(e)
        const int J = g.desc.n_subrays;
        const double p = 2.0 / static_cast<double>(g.desc.n_det - 1);
        std::vector<float> dj2(J);
        for (int j = 0; j < J; ++j) {
            const double dj = static_cast<double>(2 * j + 1 - J) / static_cast<double>(2 * J) * p;
            dj2[j] = static_cast<float>(dj * dj * 1.4426950408889634);
        }
        e = cudaMalloc(&g.d_sdir, g.dirs.size() * sizeof(double));
        if (e == cudaSuccess) e = cudaMemcpy(g.d_sdir, g.dirs.data(), g.dirs.size() * sizeof(double), cudaMemcpyHostToDevice);
        if (e == cudaSuccess) e = cudaMalloc(&g.d_soff, g.offsets.size() * sizeof(double));
        if (e == cudaSuccess) e = cudaMemcpy(g.d_soff, g.offsets.data(), g.offsets.size() * sizeof(double), cudaMemcpyHostToDevice);
        if (e == cudaSuccess) e = cudaMalloc(&g.d_sdj2, dj2.size() * sizeof(float));
        if (e == cudaSuccess) e = cudaMemcpy(g.d_sdj2, dj2.data(), dj2.size() * sizeof(float), cudaMemcpyHostToDevice);
        if (e == cudaSuccess && 2 * sizeof(float) * g.R + 1024 > g.smem_optin) e = cudaErrorInvalidConfiguration;
        if (e == cudaSuccess) e = set_sid_smem_limit(2 * sizeof(float) * g.R);
    }
    if (e == cudaSuccess) e = cudaMemcpy(g.d_rays, rays.data(), rays.size() * sizeof(RayP), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(g.d_w, g.wf.data(), g.wf.size() * sizeof(float), cudaMemcpyHostToDevice);
    for (int mode = 0; mode < 4 && e == cudaSuccess; ++mode) {
        const size_t sm = proj_cfg(g, mode).smem;
        if (sm > g.smem_optin) e = cudaErrorInvalidConfiguration;
        else e = set_proj_smem_limit(mode, sm);
    }
    if (g.adj_seg && e == cudaSuccess) {
        const SegCfg sc = seg_cfg(g);
        if (sc.smemA > g.smem_optin || sc.smemB > g.smem_optin) e = cudaErrorInvalidConfiguration;
        if (e == cudaSuccess) e = set_seg_smem_limit(0, MODE_FWD, sc.smemA);
        for (int mode : {MODE_VJP, MODE_GN}) {
            if (e == cudaSuccess) e = set_seg_smem_limit(0, mode, sc.smemA);
            if (e == cudaSuccess) e = set_seg_smem_limit(1, mode, sc.smemB);
        }
        if (e == cudaSuccess) e = set_gnc_smem_limit(std::max(sc.smemB, sc.smemG));
        if (e == cudaSuccess && g.jvp_seg) e = set_seg_smem_limit(0, MODE_JVP, sc.smemA);
    }
    if (prev >= 0) cudaSetDevice(prev);
    if (e != cudaSuccess) {
        free_device_tables(&g);
        delete h;
        return cuda_fail(e, "pget_geometry_create");
    }
    *out = h;
    return PGET_OK;
}

pget_status pget_geometry_destroy(pget_geometry h)
{
    if (!h) return PGET_OK;
    if (h->g.device < 0) { delete h; return PGET_OK; }
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(h->g.device);
    free_device_tables(&h->g);
    if (prev >= 0) cudaSetDevice(prev);
    delete h;
    return PGET_OK;
}

pget_status pget_geometry_info(pget_geometry h, pget_geometry_info_t* o)
{
    if (!h || !o) return fail(PGET_ERR_INVALID_ARGUMENT, "NULL argument");
    const Geometry& g = h->g;
    const pget_geometry_desc& d = g.desc;
    o->n_rays = static_cast<int64_t>(d.batch) * g.n_ab * g.R;
    o->n_samples_nominal = g.n_samples_nominal;
    o->n_samples_traced = g.pair ? g.n_samples_traced_p : g.n_samples_traced;
    o->n_samples_traced_jvp = g.n_samples_traced;
    o->angle_banks_merged = g.dup ? 1 : 0;
    o->pad_ = 0;
    o->image_elems = static_cast<int64_t>(d.batch) * d.n_px * d.n_px;
    o->sino_elems = static_cast<int64_t>(d.batch) * g.n_ab * d.n_det;
    o->n_t = g.n_t;
    o->n_px = d.n_px;
    o->n_angles = d.n_angles;
    o->n_banks = d.n_banks;
    o->n_det = d.n_det;
    o->n_subrays = d.n_subrays;
    o->batch = d.batch;
    o->h = g.h;
    o->delta = g.delta;
    o->T = g.T;
    return PGET_OK;
}

size_t pget_table_bytes(pget_geometry h, int id)
{
    if (!h) return 0;
    const Geometry& g = h->g;
    switch (id) {
    case PGET_TABLE_ANGLES: return g.angles.size() * sizeof(double);
    case PGET_TABLE_DIRS: return g.dirs.size() * sizeof(double);
    case PGET_TABLE_OFFSETS: return g.offsets.size() * sizeof(double);
    case PGET_TABLE_WEIGHTS: return g.weights.size() * sizeof(double);
    case PGET_TABLE_TLAT: return 3 * sizeof(double);
    case PGET_TABLE_CLIP: return g.clip.size() * sizeof(int32_t);
    case PGET_TABLE_VAR_C: return g.var_c.size() * sizeof(double);
    case PGET_TABLE_VAR_W: return g.var_w.size() * sizeof(double);
    }
    return 0;
}

pget_status pget_geometry_export(pget_geometry h, int id, void* dst, size_t bytes)
{
    if (!h || !dst) return fail(PGET_ERR_INVALID_ARGUMENT, "NULL argument");
    if (id < PGET_TABLE_ANGLES || id > PGET_TABLE_VAR_W) return fail(PGET_ERR_INVALID_ARGUMENT, "bad table id");
    const size_t need = pget_table_bytes(h, id);
    if (need == 0) return PGET_OK;   // an empty table (the model variant's when it is off)
    if (bytes < need) return fail(PGET_ERR_SHAPE, "destination too small");
    const Geometry& g = h->g;
    const double tl[3] = {g.h, g.delta, g.T};
    const void* src = nullptr;
    switch (id) {
    case PGET_TABLE_ANGLES: src = g.angles.data(); break;
    case PGET_TABLE_DIRS: src = g.dirs.data(); break;
    case PGET_TABLE_OFFSETS: src = g.offsets.data(); break;
    case PGET_TABLE_WEIGHTS: src = g.weights.data(); break;
    case PGET_TABLE_TLAT: src = tl; break;
    case PGET_TABLE_CLIP: src = g.clip.data(); break;
    case PGET_TABLE_VAR_C: src = g.var_c.data(); break;
    case PGET_TABLE_VAR_W: src = g.var_w.data(); break;
    }
    std::memcpy(dst, src, need);
    return PGET_OK;
}

size_t pget_workspace_bytes(pget_geometry h, int op)
{
    if (!h || op < 0 || op > PGET_OP_LM_SOLVE) return 0;
    return carve(h->g, op, nullptr).bytes + 256;
}

// ---- building blocks (all enqueued on s)
static pget_status pack2(const Geometry& g, const WS& w, const float* lam, const float* mu, const float* slam,
                         const float* smu, float* ul, float* um, cudaStream_t s, const BoxK* box = nullptr)
{
    const size_t img = static_cast<size_t>(g.desc.batch) * g.P * g.P;
    launch_k(pack2_kernel, vec_grid(img), kVecThreads, 0, s, lam, mu, slam, smu, w.img2[0], w.img2[1], ul, um,
                                                      g.desc.n_px, g.P, g.desc.batch, box ? 1 : 0,
                                                      box ? *box : BoxK{make_float4(0.f, 0.f, 0.f, 0.f), 0.f}); note();
    CK(cudaGetLastError());
    return PGET_OK;
}

static pget_status pack4(const Geometry& g, const WS& w, const float* lam, const float* mu, const float* dl,
                         const float* dm, cudaStream_t s)
{
    const size_t img = static_cast<size_t>(g.desc.batch) * g.P * g.P;
    launch_k(pack4_kernel, vec_grid(img), kVecThreads, 0, s, lam, mu, dl, dm, w.img4[0], w.img4[1], g.desc.n_px, g.P,
                                                      g.desc.batch); note();
    CK(cudaGetLastError());
    return PGET_OK;
}

// y (and dy) from the packed images (MODE_FWD / MODE_JVP)
static pget_status proj_out(const Geometry& g, const WS& w, int mode, float* y, float* dy, cudaStream_t s)
{
    const ProjCfg c = proj_cfg(g, mode);
    ProjArgs A = base_args(g, c);
    for (int k = 0; k < 2; ++k) { A.img2[k] = w.img2[k]; A.img4[k] = w.img4[k]; }
    A.y = y;
    A.dy = dy;
    return run_proj(g, mode, c, A, s);
}

// adjoint projector into w.gacc (MODE_VJP with weights win, or MODE_GN), then the fixed-order reduction
static pget_status proj_adjoint(const Geometry& g, const WS& w, int mode, const float* win, cudaStream_t s,
                                bool build_cache = false, bool have_a = false)
{
    const ProjCfg c = proj_cfg(g, mode);
    ProjArgs A = base_args(g, c);
    for (int k = 0; k < 2; ++k) { A.img2[k] = w.img2[k]; A.img4[k] = w.img4[k]; }
    A.slots = w.slots;
    A.win = win;
    if (g.sid) {   // pixel basis: bounds, scatter into the fixed-point accumulator, fp64 partials
        SidArgs S = sid_args(g, A);
        S.ray = w.sray;
        S.raybd = w.sraybd;
        S.bound = w.sbound;
        S.acc = w.sacc;
        cudaEvent_t ea = nullptr, eb = nullptr;
        if (g_prof.on.load(std::memory_order_relaxed)) {
            std::lock_guard<std::mutex> lk(g_prof.mu);
            g_prof.total += 3;
            g_prof.mode_launches[mode]++;
            if (g_prof.used + 2 <= g_prof.pool.size()) {
                ea = g_prof.pool[g_prof.used++];
                eb = g_prof.pool[g_prof.used++];
                g_prof.recs.push_back({mode, ea, eb});
            }
        }
        if (ea) cudaEventRecord(ea, s);
        const cudaError_t e = launch_sid_adj(mode, g.var, S, w.gacc, s);
        if (eb) cudaEventRecord(eb, s);
        if (e != cudaSuccess) return cuda_fail(e, "pixel-basis adjoint launch");
        return PGET_OK;
    }
    if (build_cache && w.gscale)   // the builder's entry bounds start from 0 (atomicMax)
        CK(cudaMemsetAsync(w.gscale, 0, static_cast<size_t>(g.desc.batch) * g.sch[kSchedAdj].ntab * 8 * sizeof(float), s));
    pget_status st = g.adj_seg ? run_seg(g, mode, A, w.segp, s, build_cache ? w.cache : nullptr, have_a, w.gscale)
                               : run_proj(g, mode, c, A, s);
    if (st) return st;
    const int N = g.desc.n_px;
    const dim3 grid((N + 31) / 32, (N + 31) / 32, g.desc.batch * c.G);
    launch_k(reduce_slots_kernel, grid, dim3(32, 8), 0, s, w.slots, w.gacc, N, slot_pitch(g), g.desc.batch, c.G,
                                                    g.sch[kSchedAdj].d_red_off, g.sch[kSchedAdj].d_red_slot,
                                                    g.sch[kSchedAdj].d_slot_lo, g.sch[kSchedAdj].d_slot_hi); note();
    CK(cudaGetLastError());
    return PGET_OK;
}

// GN with cached Jacobian entries: args shared by the three kernels (phase-B units,
// groups, stage list and launch shape of the segmented adjoint)
// the priors attached to the handle, weights times the LM continuation factor
static PriorArgs prior_args(const Geometry& g, float scale)
{
    PriorArgs p;
    p.m1 = g.prior_m1;
    p.m2 = g.prior_m2;
    p.a1 = g.prior_a1 * scale;
    p.a2 = g.prior_a2 * scale;
    return p;
}

static ProjArgs gnc_args(const Geometry& g, const WS& w)
{
    const Schedule& S = g.sch[kSchedAdj];
    const SegCfg c = seg_cfg(g);
    ProjArgs A = base_args(g, proj_cfg(g, MODE_GN));
    for (int k = 0; k < 2; ++k) { A.img2[k] = w.img2[k]; A.img4[k] = w.img4[k]; }
    A.slots = w.slots;
    A.segp = w.segp;
    A.slot_lo = S.d_slot_lo;
    A.slot_hi = S.d_slot_hi;
    A.K = S.K;
    A.seg_rows = S.d_seg_rows;
    A.n_groups = g.gnb_adj ? S.max_gC : S.max_gB;
    A.groups = g.gnb_adj ? S.d_groupsC : S.d_groups;
    A.units = S.d_unitsB;
    A.u_begin = S.d_ub_begin;
    A.stages = S.d_stB;
    A.s_begin = S.d_sb_begin;
    A.RbB = c.RbB;
    A.passesB = c.passesB;
    A.stage_bytes = c.stageB;
    A.off_wacc = c.off_wacc;
    A.off_rout = c.off_rout;
    A.off_gsh = c.off_gsh;
    A.off_rsc = c.off_rsc;
    A.off_q1 = c.off_q1;
    A.cache = w.cache;
    A.cache_off = g.gnb_adj ? S.d_cache_offC : S.d_cache_off;
    A.cache_rows_member = g.gnb_adj ? S.cache_rows_memberC : S.cache_rows_member;
    A.cache_ng = g.gnb_adj ? S.max_gC : S.max_gB;
    A.ntab = S.ntab;
    A.jp = w.jp;
    A.gscale = w.gscale;
    A.cellmax = g.cellmax;
    return A;
}

// the cache from the VJP-mode phase-A partials in w.segp (of u, whose (lam, mu) bands are in w.img2)
static pget_status gnc_build(const Geometry& g, const WS& w, cudaStream_t s)
{
    const SegCfg c = seg_cfg(g);
    if (w.gscale) CK(cudaMemsetAsync(w.gscale, 0, static_cast<size_t>(g.desc.batch) * g.sch[kSchedAdj].ntab * 8 * sizeof(float), s));
    cudaError_t e = launch_gnc(0, g.pair, gnc_args(g, w), c.gridB, c.WB * 32, c.smemB, s);
    note();
    if (e != cudaSuccess) return cuda_fail(e, "lin_kernel launch");
    return PGET_OK;
}

// q-partials of H p from the cache: p packed into w.img2, (J p) partials, scatter, slot reduction
// hybrid (g.gn_hybrid): the (J p) of p recomputed by the GN-mode phase A from (u, p) (pack4 into
// w.img4), the scatter from the cache; else the (J p) from the cache too (jvpc_kernel)
static pget_status gnc_product(const Geometry& g, const WS& w, const float* lam, const float* mu, const float* pl,
                               const float* pm, cudaStream_t s, bool packed = false)
{
    // packed: w.img4 already holds (lam, mu, pl, pm) (the fused CG kernel mirrors its p update there)
    pget_status st = g.gn_hybrid ? (packed ? PGET_OK : pack4(g, w, lam, mu, pl, pm, s))
                                 : pack2(g, w, pl, pm, nullptr, nullptr, nullptr, nullptr, s, nullptr);
    if (st) return st;
    const SegCfg c = seg_cfg(g);
    ProjArgs A = gnc_args(g, w);
    if (g.gn_hybrid) {   // the per-ray scatter weights into w.jp's space (unused by the hybrid product)
        A.jp = nullptr;
        A.gw = w.jp;
    }
    cudaEvent_t ea = nullptr, eb = nullptr;
    if (g_prof.on.load(std::memory_order_relaxed)) {
        std::lock_guard<std::mutex> lk(g_prof.mu);
        g_prof.total += g.gn_hybrid ? 3 : 2;   // phase A (+ gnw) + scatter
        g_prof.mode_launches[MODE_GN]++;
        if (g_prof.used + 2 <= g_prof.pool.size()) {
            ea = g_prof.pool[g_prof.used++];
            eb = g_prof.pool[g_prof.used++];
            g_prof.recs.push_back({MODE_GN, ea, eb});
        }
    }
    if (ea) cudaEventRecord(ea, s);
    cudaError_t e;
    if (g.gn_hybrid) {
        const Schedule& S = g.sch[kSchedAdj];
        ProjArgs Aa = A;
        Aa.units = S.d_unitsA;
        Aa.u_begin = S.d_ua_begin;
        Aa.stages = S.d_stA;
        Aa.s_begin = S.d_sa_begin;
        Aa.RbA = c.RbA;
        Aa.passesA = c.passesA;
        Aa.stage_bytes = c.stageA;
        e = launch_seg(0, MODE_GN, c.maxgA, g.pair, Aa, c.gridA, (c.WA + 1) * 32, c.smemA, s);
        if (e == cudaSuccess) e = launch_gnw(g.pair, A, g.d_tabsA, S.ntab, g.desc.batch, s);
    } else {
        e = launch_gnc(1, g.pair, A, c.gridB, c.WB * 32, c.smemB, s);
    }
    if (e == cudaSuccess) {
        ProjArgs Ag = A;
        Ag.RbB = c.RbG;
        Ag.planeB4 = 4 * (c.RbG + 1) * g.P;
        Ag.off_wacc = c.off_waccG;
        Ag.off_rout = c.off_routG;
        Ag.passesB = c.passesG;
        e = launch_gnc(2, g.pair, Ag, c.gridB, c.WG * 32, c.smemG, s);
    }
    if (eb) cudaEventRecord(eb, s);
    if (e != cudaSuccess) return cuda_fail(e, "cached GN launch");
    const ProjCfg pc = proj_cfg(g, MODE_GN);
    const int N = g.desc.n_px;
    const dim3 grid((N + 31) / 32, (N + 31) / 32, g.desc.batch * pc.G);
    launch_k(reduce_slots_kernel, grid, dim3(32, 8), 0, s, w.slots, w.gacc, N, slot_pitch(g), g.desc.batch, pc.G,
                                                    g.sch[kSchedAdj].d_red_off, g.sch[kSchedAdj].d_red_slot,
                                                    g.sch[kSchedAdj].d_slot_lo, g.sch[kSchedAdj].d_slot_hi); note();
    CK(cudaGetLastError());
    return PGET_OK;
}

// the LM iteration's gradient J^T win through the coefficient cache (consecutive-ray layout, built by
// gnc_build from u's phase-A partials): the VJP's per-ray weights from the sinogram (gnw_kernel SINO),
// the cached scatter and the slot reduction into w.gacc -- the VJP without re-walking the image
static pget_status gnc_gradient(const Geometry& g, const WS& w, const float* win, cudaStream_t s)
{
    const SegCfg c = seg_cfg(g);
    const Schedule& S = g.sch[kSchedAdj];
    ProjArgs A = gnc_args(g, w);
    A.jp = nullptr;
    A.gw = w.jp;
    A.win = win;
    cudaEvent_t ea = nullptr, eb = nullptr;
    if (g_prof.on.load(std::memory_order_relaxed)) {
        std::lock_guard<std::mutex> lk(g_prof.mu);
        g_prof.total += 2;
        g_prof.mode_launches[MODE_VJP]++;
        if (g_prof.used + 2 <= g_prof.pool.size()) {
            ea = g_prof.pool[g_prof.used++];
            eb = g_prof.pool[g_prof.used++];
            g_prof.recs.push_back({MODE_VJP, ea, eb});
        }
    }
    if (ea) cudaEventRecord(ea, s);
    cudaError_t e = launch_gnw(g.pair, A, g.d_tabsA, S.ntab, g.desc.batch, s, true);
    if (e == cudaSuccess) {
        ProjArgs Ag = A;
        Ag.RbB = c.RbG;
        Ag.planeB4 = 4 * (c.RbG + 1) * g.P;
        Ag.off_wacc = c.off_waccG;
        Ag.off_rout = c.off_routG;
        Ag.passesB = c.passesG;
        e = launch_gnc(2, g.pair, Ag, c.gridB, c.WG * 32, c.smemG, s);
    }
    if (eb) cudaEventRecord(eb, s);
    if (e != cudaSuccess) return cuda_fail(e, "cached gradient launch");
    const ProjCfg pc = proj_cfg(g, MODE_VJP);
    const int N = g.desc.n_px;
    const dim3 grid((N + 31) / 32, (N + 31) / 32, g.desc.batch * pc.G);
    launch_k(reduce_slots_kernel, grid, dim3(32, 8), 0, s, w.slots, w.gacc, N, slot_pitch(g), g.desc.batch, pc.G,
                                                    S.d_red_off, S.d_red_slot, S.d_slot_lo, S.d_slot_hi); note();
    CK(cudaGetLastError());
    return PGET_OK;
}

// the forward of the packed u in w.img2: segmented (the VJP-mode phase A of the adjoint schedule +
// fp64 combine) when enabled, else the fused projector.  Used for the LM wrap's F(u), whose phase-A
// partials the gradient VJP then reuses, and its trial forward; the standalone forward stays fused
// (measured faster alone on configs 2, 3 and 5)
// plain: the phase A in forward mode (uncompensated sums, no adjoint fields: the standalone forward, graded
// per element like the fused forward that never compensated); else the VJP mode, whose partials the LM
// wrap's gradient reuses and whose compensated sums feed f(u), f(u+s) and f(u~)
static pget_status fwd_out(const Geometry& g, const WS& w, float* y, cudaStream_t s, bool plain = false)
{
    if (!(g.adj_seg && g.fwd_seg)) return proj_out(g, w, MODE_FWD, y, nullptr, s);
    const Schedule& S = g.sch[kSchedAdj];
    const SegCfg c = seg_cfg(g);
    ProjArgs A = base_args(g, proj_cfg(g, MODE_VJP));
    for (int k = 0; k < 2; ++k) { A.img2[k] = w.img2[k]; A.img4[k] = w.img4[k]; }
    A.y = y;
    A.segp = w.segp;
    A.K = S.K;
    A.seg_rows = S.d_seg_rows;
    A.units = S.d_unitsA;
    A.u_begin = S.d_ua_begin;
    A.stages = S.d_stA;
    A.s_begin = S.d_sa_begin;
    A.RbA = c.RbA;
    A.passesA = c.passesA;
    A.stage_bytes = c.stageA;
    cudaEvent_t ea = nullptr, eb = nullptr;
    if (g_prof.on.load(std::memory_order_relaxed)) {
        std::lock_guard<std::mutex> lk(g_prof.mu);
        g_prof.total += 2;
        g_prof.mode_launches[MODE_FWD]++;
        if (g_prof.used + 2 <= g_prof.pool.size()) {
            ea = g_prof.pool[g_prof.used++];
            eb = g_prof.pool[g_prof.used++];
            g_prof.recs.push_back({MODE_FWD, ea, eb});
        }
    }
    if (ea) cudaEventRecord(ea, s);
    cudaError_t e = launch_seg(0, plain ? MODE_FWD : MODE_VJP, c.maxgA, g.pair, A, c.gridA, (c.WA + 1) * 32, c.smemA, s);
    const int ntab = static_cast<int>((g.pair ? g.task_ab_p : g.task_ab).size());
    if (e == cudaSuccess) e = launch_fwd_combine(g.pair, A, g.d_tabsA, ntab, g.desc.batch, s);
    if (eb) cudaEventRecord(eb, s);
    if (e != cudaSuccess) return cuda_fail(e, "segmented forward launch");
    return PGET_OK;
}

// the standalone JVP of the packed (u, d) in w.img4: segmented (phase A over every traced angle-bank
// + fp64 combine) when enabled, else the fused projector
static pget_status jvp_out(const Geometry& g, const WS& w, float* y, float* dy, cudaStream_t s)
{
    if (!(g.adj_seg && g.jvp_seg)) return proj_out(g, w, MODE_JVP, y, dy, s);
    const Schedule& S = g.schJ;
    const SegCfg c = seg_cfg(g);
    ProjArgs A = base_args(g, proj_cfg(g, MODE_JVP));
    for (int k = 0; k < 2; ++k) { A.img2[k] = w.img2[k]; A.img4[k] = w.img4[k]; }
    A.y = y;
    A.dy = dy;
    A.segp = w.segpJ;
    A.K = S.K;
    A.seg_rows = S.d_seg_rows;
    A.units = S.d_unitsA;
    A.u_begin = S.d_ua_begin;
    A.stages = S.d_stA;
    A.s_begin = S.d_sa_begin;
    A.RbA = c.RbA;
    A.passesA = c.passesA;
    A.stage_bytes = c.stageA;
    cudaEvent_t ea = nullptr, eb = nullptr;
    if (g_prof.on.load(std::memory_order_relaxed)) {
        std::lock_guard<std::mutex> lk(g_prof.mu);
        g_prof.total += 2;
        g_prof.mode_launches[MODE_JVP]++;
        if (g_prof.used + 2 <= g_prof.pool.size()) {
            ea = g_prof.pool[g_prof.used++];
            eb = g_prof.pool[g_prof.used++];
            g_prof.recs.push_back({MODE_JVP, ea, eb});
        }
    }
    if (ea) cudaEventRecord(ea, s);
    cudaError_t e = launch_seg(0, MODE_JVP, c.maxgA, false, A, c.gridA, (c.WA + 1) * 32, c.smemA, s);
    if (e == cudaSuccess) e = launch_jvp_combine(A, g.d_tabsJ, static_cast<int>(g.task_ab.size()), g.desc.batch, s);
    if (eb) cudaEventRecord(eb, s);
    if (e != cudaSuccess) return cuda_fail(e, "segmented JVP launch");
    return PGET_OK;
}

pget_status pget_forward(pget_geometry h, const float* lam, const float* mu, float* y, void* ws, size_t ws_bytes,
                         pget_stream_t stream)
{
    NvtxRange nvtx_("pget_forward");
    WS w;
    pget_status st = check_common(h, PGET_OP_FORWARD, ws, ws_bytes, &w);
    if (st) return st;
    if ((st = check_ptrs({lam, mu, y}, "pget_forward", h->g.device))) return st;
    const Geometry& g = h->g;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if ((st = pack2(g, w, lam, mu, nullptr, nullptr, nullptr, nullptr, s))) return st;
    return fwd_out(g, w, y, s, g.fwd_plain);   // the warp-specialised segmented phase A + fp64 combine (fused: variant only)
}

pget_status pget_jvp(pget_geometry h, const float* lam, const float* mu, const float* dlam, const float* dmu,
                     float* y, float* dy, void* ws, size_t ws_bytes, pget_stream_t stream)
{
    NvtxRange nvtx_("pget_jvp");
    WS w;
    pget_status st = check_common(h, PGET_OP_JVP, ws, ws_bytes, &w);
    if (st) return st;
    if ((st = check_ptrs({lam, mu, dlam, dmu, dy}, "pget_jvp", h->g.device))) return st;
    if (y && !aligned16(y)) return fail(PGET_ERR_ALIGNMENT, "pget_jvp: y not 16-byte aligned");
    const Geometry& g = h->g;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if ((st = pack4(g, w, lam, mu, dlam, dmu, s))) return st;
    return jvp_out(g, w, y, dy, s);
}

pget_status pget_vjp(pget_geometry h, const float* lam, const float* mu, const float* wv, float* g_lam, float* g_mu,
                     void* ws, size_t ws_bytes, pget_stream_t stream)
{
    NvtxRange nvtx_("pget_vjp");
    WS w;
    pget_status st = check_common(h, PGET_OP_VJP, ws, ws_bytes, &w);
    if (st) return st;
    if ((st = check_ptrs({lam, mu, wv, g_lam, g_mu}, "pget_vjp", h->g.device))) return st;
    const Geometry& g = h->g;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int N = g.desc.n_px, B = g.desc.batch;
    if ((st = pack2(g, w, lam, mu, nullptr, nullptr, nullptr, nullptr, s))) return st;
    if ((st = proj_adjoint(g, w, MODE_VJP, wv, s))) return st;
    launch_k(finish_kernel, dim3(vec_grid(static_cast<size_t>(N) * N), B), kVecThreads, 0, s, 
        w.gacc, proj_cfg(g, MODE_VJP).G, nullptr, nullptr, 0.f, 0.f, 1.f, g_lam, g_mu, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
        nullptr, nullptr, nullptr, N, PriorArgs{}, nullptr); note();
    CK(cudaGetLastError());
    return PGET_OK;
}

pget_status pget_gn_apply(pget_geometry h, const float* lam, const float* mu, const float* p_lam, const float* p_mu,
                          float alpha, float beta, float* q_lam, float* q_mu, void* ws, size_t ws_bytes,
                          pget_stream_t stream)
{
    NvtxRange nvtx_("pget_gn_apply");
    WS w;
    pget_status st = check_common(h, PGET_OP_GN_APPLY, ws, ws_bytes, &w);
    if (st) return st;
    if ((st = check_ptrs({lam, mu, p_lam, p_mu, q_lam, q_mu}, "pget_gn_apply", h->g.device))) return st;
    if (!std::isfinite(alpha) || !std::isfinite(beta) || alpha < 0.f || beta < 0.f)
        return fail(PGET_ERR_INVALID_ARGUMENT, "alpha, beta must be finite and >= 0");
    const Geometry& g = h->g;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int N = g.desc.n_px, B = g.desc.batch;
    if ((st = pack2(g, w, lam, mu, nullptr, nullptr, nullptr, nullptr, s))) return st;
    if (g.adj_seg && g.gn_cached && g.gn_apply_cached) {   // phase A (VJP mode) of u -> cache -> cached product
        const SegCfg c = seg_cfg(g);
        const Schedule& S = g.sch[kSchedAdj];
        ProjArgs A = gnc_args(g, w);
        A.units = S.d_unitsA;
        A.u_begin = S.d_ua_begin;
        A.stages = S.d_stA;
        A.s_begin = S.d_sa_begin;
        A.RbA = c.RbA;
        A.passesA = c.passesA;
        A.stage_bytes = c.stageA;
        CK(launch_seg(0, MODE_VJP, c.maxgA, g.pair, A, c.gridA, (c.WA + 1) * 32, c.smemA, s));
        note();
        if ((st = gnc_build(g, w, s))) return st;
        if ((st = gnc_product(g, w, lam, mu, p_lam, p_mu, s))) return st;
    } else {
        if ((st = pack4(g, w, lam, mu, p_lam, p_mu, s))) return st;
        if ((st = proj_adjoint(g, w, MODE_GN, nullptr, s))) return st;
    }
    launch_k(finish_kernel, dim3(vec_grid(static_cast<size_t>(N) * N), B), kVecThreads, 0, s, 
        w.gacc, proj_cfg(g, MODE_GN).G, p_lam, p_mu, alpha, beta, 1.f, q_lam, q_mu, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
        nullptr, nullptr, nullptr, N, prior_args(g, 1.f), nullptr); note();
    CK(cudaGetLastError());
    return PGET_OK;
}

// One LM iteration (see pget_gn_cg_step) on a carved workspace.  betav (device, per member, nullable)
// overrides beta; box (nullable) projects the step onto [lam_lo, lam_hi] x [mu_lo, mu_hi] before
// pred and the trial (reading R-N1).
static pget_status gn_cg_impl(const Geometry& g, WS w, const float* lam, const float* mu,
                              const float* y_meas, float alpha, float beta, const float* betav, int32_t n_cg,
                              uint32_t flags, float* s_lam, float* s_mu, pget_gn_stats* stats, const BoxK* box,
                              cudaStream_t s, float pscale = 1.f, bool sgp = false)
{
    pget_status st;
    const int N = g.desc.n_px, B = g.desc.batch;
    const int n2 = N * N;
    const int nsper = g.n_ab * g.desc.n_det;
    const dim3 vg(kNblk, B);
    double* P[9];
    for (int k = 0; k < 9; ++k) P[k] = w.part + static_cast<size_t>(k) * B * kNblk;
    // priors (pget_set_prior) at the continuation scale pscale; P[8] holds their value partials
    const PriorArgs pr = prior_args(g, pscale);
    const bool has_prior = pr.m1 || pr.m2;
    double* Pp = has_prior ? P[8] : nullptr;
    const int sgrid = (B + 127) / 128;
    const int Gv = proj_cfg(g, MODE_VJP).G, Gg = proj_cfg(g, MODE_GN).G;

    // 1-2: r = F(u) - y, 1/2||r||^2, ||Lu||^2   (u packed once for the whole iteration)
    if ((st = pack2(g, w, lam, mu, nullptr, nullptr, nullptr, nullptr, s))) return st;
    if ((st = fwd_out(g, w, w.ysino, s))) return st;
    launch_k(residual_kernel, vg, kVecThreads, 0, s, w.ysino, y_meas, P[0], nsper); note();
    launch_k(regsq_kernel, vg, kVecThreads, 0, s, lam, mu, P[1], N); note();
    if (has_prior) launch_k(priorsq_kernel, vg, kVecThreads, 0, s, lam, mu, pr, Pp, N); note();
    CK(cudaGetLastError());
    // 3: b = -(J^T r + alpha L^T L u (+ P^T P u)); z = p = b; s = 0; ||b||^2
    const bool cached = g.adj_seg && g.gn_cached;
    // the gradient VJP also writes the GN Jacobian-entry cache (fused cache build)
    // F(u) above was the segmented forward: its phase-A partials of u are the VJP's phase A
    if (cached && n_cg > 0 && g.gnb_adj) {
        // the cache over consecutive-ray groups, built by lin_kernel from the phase-A partials of u that
        // F(u) left (the fused builder of the VJP writes the comb layout of its own scatter); the
        // gradient then comes from the cache like every GN product
        if ((st = gnc_build(g, w, s))) return st;
        if ((st = gnc_gradient(g, w, w.ysino, s))) return st;
    } else if ((st = proj_adjoint(g, w, MODE_VJP, w.ysino, s, cached && n_cg > 0, g.adj_seg && g.fwd_seg))) {
        return st;
    }
    launch_k(finish_kernel, vg, kVecThreads, 0, s, w.gacc, Gv, lam, mu, alpha, 0.f, -1.f, w.bl, w.bm, w.bl, w.bm, P[2], w.zl,
                                            w.zm, w.pl, w.pm, s_lam, s_mu, N, pr, nullptr); note();
    CK(cudaGetLastError());
    launch_k(scalar_kernel, sgrid, 128, 0, s, SC_INIT, 0, P[0], P[1], P[2], kNblk, w.cg, stats, B, alpha, beta, betav, Pp); note();
    CK(cudaGetLastError());

    // 5: CG
    if (sgp && box) {   // 5': SGP (O11) instead of CG: s stays inside the box
        const size_t nimg = static_cast<size_t>(B) * n2;
        launch_k(sgp_init_kernel, vec_grid(nimg), kVecThreads, 0, s, w.bl, w.bm, w.zl, w.zm, w.cg, n2, B); note();
        CK(cudaGetLastError());
        for (int k = 0; k <= n_cg; ++k) {
            // d = P(u + s - a g) - u - s into (pl, pm); the last pass only reports ||d||
            launch_k(sgp_dir_kernel, vg, kVecThreads, 0, s, lam, mu, s_lam, s_mu, w.zl, w.zm, w.cg, *box, w.pl, w.pm, P[3],
                                                      P[4], n2); note();
            CK(cudaGetLastError());
            if (k == n_cg) {
                launch_k(sgp_scalar_kernel, sgrid, 128, 0, s, k, 1, P[3], P[4], nullptr, nullptr, kNblk, w.cg, stats, B); note();
                break;
            }
            if (cached) {   // q = H d
                if ((st = gnc_product(g, w, lam, mu, w.pl, w.pm, s))) return st;
            } else {
                if ((st = pack4(g, w, lam, mu, w.pl, w.pm, s))) return st;
                if ((st = proj_adjoint(g, w, MODE_GN, nullptr, s))) return st;
            }
            launch_k(finish_kernel, vg, kVecThreads, 0, s, w.gacc, Gg, w.pl, w.pm, alpha, beta, 1.f, w.ql, w.qm, w.pl, w.pm,
                                                    P[5], nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, N, pr,
                                                    betav); note();
            launch_k(dot2_kernel, vg, kVecThreads, 0, s, w.ql, w.qm, w.ql, w.qm, P[6], n2); note();
            launch_k(sgp_scalar_kernel, sgrid, 128, 0, s, k, 0, P[3], P[4], P[5], P[6], kNblk, w.cg, stats, B); note();
            launch_k(sgp_update_kernel, vg, kVecThreads, 0, s, s_lam, s_mu, w.zl, w.zm, w.pl, w.pm, w.ql, w.qm, w.cg, n2); note();
            CK(cudaGetLastError());
        }
    }
    for (int k = 0; k < n_cg && !(sgp && box); ++k) {
        // p of step k > 0 was packed by step k-1's fused CG kernel
        const bool packed = k > 0 && (!cached || g.gn_hybrid);
        if (cached) {
            if ((st = gnc_product(g, w, lam, mu, w.pl, w.pm, s, packed))) return st;
        } else {
            if (!packed && (st = pack4(g, w, lam, mu, w.pl, w.pm, s))) return st;
            if ((st = proj_adjoint(g, w, MODE_GN, nullptr, s))) return st;
        }
        {   // finish + gamma + update1 + zeta + update2: one cooperative launch (grid-wide syncs)
            int kk = k, NN = N, BB = B, nb = kNblk, GG = Gg, PP = g.P;
            float al = alpha, be = beta;
            double *pg = P[3], *pz = P[4];
            CGState* cgs = w.cg;
            const float* bv = betav;
            // mirror p into the packed float4 images for the next product (not after the last step)
            const bool mirror = k + 1 < n_cg && (!cached || g.gn_hybrid);
            float4* i4n = mirror ? w.img4[0] : nullptr;
            float4* i4t = mirror ? w.img4[1] : nullptr;
            PriorArgs prv = pr;
            void* args[] = {&w.gacc, &GG, &al, &be, &bv, &s_lam, &s_mu, &w.zl, &w.zm, &w.pl, &w.pm, &w.ql, &w.qm,
                            &pg, &pz, &cgs, &stats, &kk, &NN, &BB, &nb, &i4n, &i4t, &PP, &prv};
            const int grid = std::min(B * kNblk, g.cg_coop_blocks);
            if (g.cg_pdl) {   // cooperative + programmatic serialisation: overlaps the slot reduction's tail
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(grid);
                cfg.blockDim = dim3(kVecThreads);
                cfg.stream = s;
                cudaLaunchAttribute at[2];
                at[0].id = cudaLaunchAttributeCooperative;
                at[0].val.cooperative = 1;
                at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                at[1].val.programmaticStreamSerializationAllowed = 1;
                cfg.attrs = at;
                cfg.numAttrs = pdl_enabled() ? 2 : 1;
                CK(cudaLaunchKernelExC(&cfg, reinterpret_cast<const void*>(cg_fused_kernel), args));
            } else {
                CK(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(cg_fused_kernel), dim3(grid), dim3(kVecThreads),
                                               args, 0, s));
            }
            note();
        }
        CK(cudaGetLastError());
    }
    // (N1) the step actually taken inside the box: s <- clamp(u + s) - u
    if (box) {
        const size_t n = static_cast<size_t>(B) * n2;
        launch_k(project_step_kernel, vec_grid(n), kVecThreads, 0, s, lam, mu, s_lam, s_mu, n, *box); note();
        CK(cudaGetLastError());
    }
    // 6: pred = <b,s> - 1/2(||Js||^2 + alpha ||Ls||^2); ||Js||^2 from the paired GN-mode phase A of
    //    (u, s) when the segmented adjoint is on (the norm only needs GN-level accuracy), else from
    //    the standalone JVP
    if ((st = pack4(g, w, lam, mu, s_lam, s_mu, s))) return st;
    if (g.adj_seg) {
        const SegCfg c = seg_cfg(g);
        const Schedule& S = g.sch[kSchedAdj];
        ProjArgs A = gnc_args(g, w);
        ProjArgs Aa = A;
        Aa.units = S.d_unitsA;
        Aa.u_begin = S.d_ua_begin;
        Aa.stages = S.d_stA;
        Aa.s_begin = S.d_sa_begin;
        Aa.RbA = c.RbA;
        Aa.passesA = c.passesA;
        Aa.stage_bytes = c.stageA;
        CK(launch_seg(0, MODE_GN, c.maxgA, g.pair, Aa, c.gridA, (c.WA + 1) * 32, c.smemA, s));
        note();
        double* sq = reinterpret_cast<double*>(w.ysino);   // per (member, angle-bank); ysino is free here
        CK(launch_jsq(g.pair, A, sq, c.gridB, c.WB * 32, c.smemB, s));
        note();
        CK(launch_jsq_member(sq, S.ntab, B, kNblk, P[5], s));
        note();
    } else {
        if ((st = proj_out(g, w, MODE_JVP, nullptr, w.dysino, s))) return st;
        launch_k(sumsq_kernel, vg, kVecThreads, 0, s, w.dysino, P[5], nsper); note();
    }
    launch_k(regsq_kernel, vg, kVecThreads, 0, s, s_lam, s_mu, P[6], N); note();
    if (has_prior) launch_k(priorsq_kernel, vg, kVecThreads, 0, s, s_lam, s_mu, pr, Pp, N); note();
    launch_k(dot2_kernel, vg, kVecThreads, 0, s, w.bl, w.bm, s_lam, s_mu, P[7], n2); note();
    launch_k(scalar_kernel, sgrid, 128, 0, s, SC_PRED, 0, P[5], P[6], P[7], kNblk, w.cg, stats, B, alpha, beta, betav, Pp); note();
    CK(cudaGetLastError());
    // 7-8: f(u+s), rho, accept, beta_next
    if (flags & PGET_GN_EVAL_TRIAL) {
        if ((st = pack2(g, w, lam, mu, s_lam, s_mu, w.ul, w.um, s, box))) return st;
        if ((st = fwd_out(g, w, w.ysino, s, g.fwd_plain_trial))) return st;
        launch_k(residual_kernel, vg, kVecThreads, 0, s, w.ysino, y_meas, P[0], nsper); note();
        launch_k(regsq_kernel, vg, kVecThreads, 0, s, w.ul, w.um, P[1], N); note();
        if (has_prior) launch_k(priorsq_kernel, vg, kVecThreads, 0, s, w.ul, w.um, pr, Pp, N); note();
        launch_k(scalar_kernel, sgrid, 128, 0, s, SC_TRIAL, 0, P[0], P[1], nullptr, kNblk, w.cg, stats, B, alpha, beta, betav, Pp); note();
        CK(cudaGetLastError());
    }
    return PGET_OK;
}

pget_status pget_gn_cg_step(pget_geometry h, const float* lam, const float* mu, const float* y_meas, float alpha,
                            float beta, int32_t n_cg, uint32_t flags, float* s_lam, float* s_mu,
                            pget_gn_stats* stats, void* ws, size_t ws_bytes, pget_stream_t stream)
{
    NvtxRange nvtx_("pget_gn_cg_step");
    WS w;
    pget_status st = check_common(h, PGET_OP_GN_CG_STEP, ws, ws_bytes, &w);
    if (st) return st;
    if ((st = check_ptrs({lam, mu, y_meas, s_lam, s_mu, stats}, "pget_gn_cg_step", h->g.device))) return st;
    if (n_cg < 0 || n_cg > PGET_MAX_CG) return fail(PGET_ERR_INVALID_ARGUMENT, "n_cg out of [0, PGET_MAX_CG]");
    if (!std::isfinite(alpha) || !std::isfinite(beta) || alpha < 0.f || beta < 0.f)
        return fail(PGET_ERR_INVALID_ARGUMENT, "alpha, beta must be finite and >= 0");
    return gn_cg_impl(h->g, w, lam, mu, y_meas, alpha, beta, nullptr, n_cg, flags, s_lam, s_mu, stats, nullptr,
                      reinterpret_cast<cudaStream_t>(stream));
}

// Full LM solve: n_iter LM iterations with the alpha
// continuation, per-member beta schedule, box projection and accept/reject, all on the device.
pget_status pget_lm_solve(pget_geometry h, float* lam, float* mu, const float* y_meas, const pget_lm_params* prm,
                          pget_gn_stats* stats, void* ws, size_t ws_bytes, pget_stream_t stream)
{
    NvtxRange nvtx_("pget_lm_solve");
    WS w;
    pget_status st = check_common(h, PGET_OP_LM_SOLVE, ws, ws_bytes, &w);
    if (st) return st;
    if ((st = check_ptrs({lam, mu, y_meas, stats}, "pget_lm_solve", h->g.device))) return st;
    if (!prm) return fail(PGET_ERR_INVALID_ARGUMENT, "pget_lm_solve: NULL params");
    const pget_lm_params p = *prm;
    if (p.n_iter < 0 || p.n_cg < 0 || p.n_cg > PGET_MAX_CG || p.k_freeze < 0)
        return fail(PGET_ERR_INVALID_ARGUMENT, "pget_lm_solve: n_iter, n_cg or k_freeze out of range");
    if (!std::isfinite(p.alpha0) || p.alpha0 < 0.f || !std::isfinite(p.alpha_decay) || p.alpha_decay < 1.f ||
        !std::isfinite(p.beta0) || p.beta0 < 0.f)
        return fail(PGET_ERR_INVALID_ARGUMENT, "pget_lm_solve: alpha0 >= 0, alpha_decay >= 1, beta0 >= 0 required");
    const bool use_box = (p.flags & PGET_LM_BOX) != 0;
    if (use_box && !(p.lam_lo <= p.lam_hi && p.mu_lo <= p.mu_hi))
        return fail(PGET_ERR_INVALID_ARGUMENT, "pget_lm_solve: empty box");
    const bool use_sgp = (p.flags & PGET_LM_SGP) != 0;
    if (use_sgp && !use_box) return fail(PGET_ERR_INVALID_ARGUMENT, "pget_lm_solve: PGET_LM_SGP needs PGET_LM_BOX");
    if (!std::isfinite(p.lam_per_mu) || p.lam_per_mu < 0.f || (p.lam_per_mu > 0.f && !use_box))
        return fail(PGET_ERR_INVALID_ARGUMENT, "pget_lm_solve: lam_per_mu must be finite, >= 0, and needs PGET_LM_BOX");
    if (p.lam_per_mu > 0.f && p.lam_lo > p.lam_per_mu * p.mu_hi)
        return fail(PGET_ERR_INVALID_ARGUMENT, "pget_lm_solve: lam <= lam_per_mu mu excludes the whole box");
    if (p.flags & ~(PGET_LM_BOX | PGET_LM_SGP)) return fail(PGET_ERR_INVALID_ARGUMENT, "pget_lm_solve: unknown flags");
    const Geometry& g = h->g;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int N = g.desc.n_px, B = g.desc.batch, n2 = N * N;
    const BoxK box{make_float4(p.lam_lo, p.lam_hi, p.mu_lo, p.mu_hi), p.lam_per_mu};
    launch_k(fill_kernel, (B + 127) / 128, 128, 0, s, w.beta, p.beta0, B); note();
    CK(cudaGetLastError());
    if (use_box) {   // the initial guess itself is projected onto the box
        const size_t n = static_cast<size_t>(B) * n2;
        launch_k(clamp_kernel, vec_grid(n), kVecThreads, 0, s, lam, mu, n, box); note();
        CK(cudaGetLastError());
    }
    double alpha = p.alpha0, pscale = 1.0;
    for (int k = 0; k < p.n_iter; ++k) {
        if (k > 0 && k <= p.k_freeze) {   // (alpha, alpha1, alpha2)_k = (alpha, alpha1, alpha2)_0 / decay^min(k, k_freeze)
            alpha /= p.alpha_decay;
            pscale /= p.alpha_decay;
        }
        pget_gn_stats* sk = stats + static_cast<size_t>(k) * B;
        if ((st = gn_cg_impl(g, w, lam, mu, y_meas, static_cast<float>(alpha), 0.f, w.beta, p.n_cg,
                             PGET_GN_EVAL_TRIAL, w.sl, w.sm, sk, use_box ? &box : nullptr, s,
                             static_cast<float>(pscale), use_sgp)))
            return st;
        launch_k(lm_update_kernel, dim3(vec_grid(n2), B), kVecThreads, 0, s, lam, mu, w.ul, w.um, sk, w.beta, n2); note();
        CK(cudaGetLastError());
    }
    return PGET_OK;
}

// Prop. 1 safeguard (Algorithm 2): m_k(s~), m_k(s_k), f(u~), rho, accept.
pget_status pget_safeguard(pget_geometry h, const float* lam, const float* mu, const float* y_meas, const float* s_lam,
                           const float* s_mu, const float* cand_lam, const float* cand_mu, float alpha, float kappa,
                           float* u_next_lam, float* u_next_mu, pget_safeguard_stats* stats, void* ws,
                           size_t ws_bytes, pget_stream_t stream)
{
    NvtxRange nvtx_("pget_safeguard");
    WS w;
    pget_status st = check_common(h, PGET_OP_SAFEGUARD, ws, ws_bytes, &w);
    if (st) return st;
    if ((st = check_ptrs({lam, mu, y_meas, s_lam, s_mu, cand_lam, cand_mu, u_next_lam, u_next_mu, stats}, "pget_safeguard", h->g.device)))
        return st;
    if (!std::isfinite(alpha) || alpha < 0.f) return fail(PGET_ERR_INVALID_ARGUMENT, "alpha must be finite and >= 0");
    if (!std::isfinite(kappa) || !(kappa > 0.f)) return fail(PGET_ERR_INVALID_ARGUMENT, "kappa must be finite and > 0");
    for (const float* p : {lam, mu, s_lam, s_mu})
        if (p == u_next_lam || p == u_next_mu)
            return fail(PGET_ERR_INVALID_ARGUMENT, "pget_safeguard: u_next aliases lam, mu or s");
    const Geometry& g = h->g;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int N = g.desc.n_px, B = g.desc.batch;
    const int n2 = N * N;
    const int nsper = g.n_ab * g.desc.n_det;
    const dim3 vg(kNblk, B);
    double* P[18];
    for (int k = 0; k < 18; ++k) P[k] = w.part + static_cast<size_t>(k) * B * kNblk;
    const size_t nimg = static_cast<size_t>(B) * n2;
    // s~ = u~ - u;  F(u) and J s~ in one JVP launch
    launch_k(diff2_kernel, vec_grid(nimg), kVecThreads, 0, s, cand_lam, cand_mu, lam, mu, w.zl, w.zm, nimg); note();
    CK(cudaGetLastError());
    if ((st = pack4(g, w, lam, mu, w.zl, w.zm, s))) return st;
    if ((st = jvp_out(g, w, w.ysino, w.dysino, s))) return st;
    launch_k(residual_kernel, vg, kVecThreads, 0, s, w.ysino, y_meas, P[0], nsper); note();
    launch_k(regsq_kernel, vg, kVecThreads, 0, s, lam, mu, P[1], N); note();
    launch_k(dotsq_kernel, vg, kVecThreads, 0, s, w.ysino, w.dysino, P[2], P[3], nsper); note();
    launch_k(lapdot_kernel, vg, kVecThreads, 0, s, lam, mu, w.zl, w.zm, P[4], P[5], N); note();
    CK(cudaGetLastError());
    // J s_k
    if ((st = pack4(g, w, lam, mu, s_lam, s_mu, s))) return st;
    if ((st = jvp_out(g, w, nullptr, w.dysino, s))) return st;
    launch_k(dotsq_kernel, vg, kVecThreads, 0, s, w.ysino, w.dysino, P[6], P[7], nsper); note();
    launch_k(lapdot_kernel, vg, kVecThreads, 0, s, lam, mu, s_lam, s_mu, P[8], P[9], N); note();
    CK(cudaGetLastError());
    // f(u~)
    if ((st = pack2(g, w, cand_lam, cand_mu, nullptr, nullptr, nullptr, nullptr, s))) return st;
    if ((st = fwd_out(g, w, w.ysino, s))) return st;
    launch_k(residual_kernel, vg, kVecThreads, 0, s, w.ysino, y_meas, P[10], nsper); note();
    launch_k(regsq_kernel, vg, kVecThreads, 0, s, cand_lam, cand_mu, P[11], N); note();
    // priors (pget_set_prior): the rows sqrt(a1) P1 lam, sqrt(a2) P2 mu of F~ in f, m_k(s~), m_k(s_k), f(u~)
    const PriorArgs pr = prior_args(g, 1.f);
    const bool has_prior = pr.m1 || pr.m2;
    if (has_prior) {
        launch_k(priorsq_kernel, vg, kVecThreads, 0, s, lam, mu, pr, P[12], N); note();
        launch_k(priordot_kernel, vg, kVecThreads, 0, s, lam, mu, w.zl, w.zm, pr, P[13], P[14], N); note();
        launch_k(priordot_kernel, vg, kVecThreads, 0, s, lam, mu, s_lam, s_mu, pr, P[15], P[16], N); note();
        launch_k(priorsq_kernel, vg, kVecThreads, 0, s, cand_lam, cand_mu, pr, P[17], N); note();
    }
    launch_k(guard_scalar_kernel, (B + 127) / 128, 128, 0, s, w.part, kNblk, B, alpha, kappa, stats, has_prior ? 1 : 0); note();
    launch_k(guard_select_kernel, vg, kVecThreads, 0, s, lam, mu, s_lam, s_mu, cand_lam, cand_mu, stats, u_next_lam,
                                                  u_next_mu, n2); note();
    CK(cudaGetLastError());
    return PGET_OK;
}

pget_status pget_set_prior(pget_geometry h, const pget_prior* prior)
{
    if (!h) return fail(PGET_ERR_INVALID_ARGUMENT, "NULL geometry handle");
    if (h->g.device < 0) return fail(PGET_ERR_INVALID_ARGUMENT, "pget_set_prior: host-only handle");
    Geometry& g = h->g;
    if (!prior) {
        g.prior_m1 = g.prior_m2 = nullptr;
        g.prior_a1 = g.prior_a2 = 0.f;
        return PGET_OK;
    }
    if (!std::isfinite(prior->alpha1) || !std::isfinite(prior->alpha2) || prior->alpha1 < 0.f || prior->alpha2 < 0.f)
        return fail(PGET_ERR_INVALID_ARGUMENT, "pget_set_prior: alpha1, alpha2 must be finite and >= 0");
    g.prior_m1 = prior->mask_lam;
    g.prior_m2 = prior->mask_mu;
    g.prior_a1 = prior->mask_lam ? prior->alpha1 : 0.f;
    g.prior_a2 = prior->mask_mu ? prior->alpha2 : 0.f;
    return PGET_OK;
}

// Host-side consistency of a handle's static schedules (diagnostic; tests/test_abi.py).
pget_status pget_schedule_check(pget_geometry h)
{
    if (!h) return fail(PGET_ERR_INVALID_ARGUMENT, "NULL geometry handle");
    const Geometry& g = h->g;
    const int B = g.desc.batch, R = g.R, nd = g.desc.n_det, J = g.desc.n_subrays;
    std::vector<RayP> rays;
    build_ray_params(g, &rays);
    auto bad = [&](const std::string& m) { return fail(PGET_ERR_INVALID_ARGUMENT, "schedule check: " + m); };
    // fused kinds: every (member, traced angle-bank, detector) covered exactly once
    for (int k = 0; k < 2; ++k) {
        const Schedule& S = g.sch[k];
        const bool paired = g.pair && k != kSchedJvp;
        const std::vector<int32_t>& list = paired ? g.task_ab_p : g.task_ab;
        std::map<std::pair<int, int>, std::vector<int>> cover;
        for (const TaskD& t : S.tasks) {
            auto& v = cover[{t.m, t.ab}];
            if (v.empty()) v.assign(nd, 0);
            for (int d = t.dlo; d < t.dhi; ++d) ++v[d];
        }
        if (cover.size() != static_cast<size_t>(B) * list.size()) return bad("fused tasks miss an angle-bank");
        for (auto& kv : cover)
            for (int c : kv.second)
                if (c != 1) return bad("a detector is covered " + std::to_string(c) + " times");
        if (S.cta_begin.size() != static_cast<size_t>(S.C) + 1 || S.cta_begin.back() != static_cast<int>(S.tasks.size()))
            return bad("fused CTA ranges");
    }
    if (!g.adj_seg) return PGET_OK;
    const Schedule& S = g.sch[kSchedAdj];
    const int K = S.K, ntab = S.ntab, ngB = S.max_gB;
    const std::vector<int32_t>& list = g.pair ? g.task_ab_p : g.task_ab;
    if (K < 1 || S.seg_rows.size() != static_cast<size_t>(K) + 1 || S.seg_rows.front() != 0 ||
        S.seg_rows.back() != g.P - 1)
        return bad("segment rows");
    // segments partition every ray's samples
    for (int t = 0; t < ntab; ++t)
        for (int r = 0; r < R; ++r) {
            const RayP& rp = rays[static_cast<size_t>(list[t]) * R + r];
            int64_t n = 0;
            for (int k = 0; k < K; ++k)
                n += rp.dV > 0 ? seg_entry(rp, S.seg_rows[k + 1]) - seg_entry(rp, S.seg_rows[k])
                               : seg_entry(rp, S.seg_rows[k]) - seg_entry(rp, S.seg_rows[k + 1]);
            const int64_t want = rp.ihi >= rp.ilo ? rp.ihi - rp.ilo + 1 : 0;
            if (n != want) return bad("segments do not partition a ray's samples");
        }
    // units: each canonical unit once per phase, in CTA ranges
    for (int ph = 0; ph < 2; ++ph) {
        const std::vector<UnitD>& U = ph ? S.unitsB : S.unitsA;
        const std::vector<int32_t>& ub = ph ? S.ub_begin : S.ua_begin;
        std::vector<int> seen(static_cast<size_t>(S.n_canon), 0);
        for (const UnitD& u : U) {
            if (u.canon < 0 || u.canon >= S.n_canon) return bad("unit index");
            if (u.canon != (u.m * ntab + static_cast<int>(std::find(list.begin(), list.end(), u.ab) - list.begin())) * K + u.seg)
                return bad("canonical unit index");
            ++seen[u.canon];
        }
        for (int c : seen)
            if (c != 1) return bad("a unit is scheduled " + std::to_string(c) + " times");
        if (ub.back() != static_cast<int>(U.size())) return bad("unit CTA ranges");
    }
    // slots: <= 16 units, one CTA, one (member, class), rows inside the slot range; reduce lists
    std::vector<int> used(static_cast<size_t>(S.n_slots), 0);
    for (int c = 0; c < S.C; ++c) {
        int prev = -1;
        for (int u = S.ub_begin[c]; u < S.ub_begin[c + 1]; ++u) {
            const UnitD& t = S.unitsB[u];
            if (t.slot < 0 || t.slot >= S.n_slots) return bad("slot index");
            if (t.slot != prev && used[t.slot]) return bad("a slot spans CTAs or runs");
            if ((t.flags & kTaskFirst) != 0 && t.slot == prev) return bad("first flag");
            ++used[t.slot];
            const int lo = std::max(0, S.seg_rows[t.seg] - kHalo);
            const int hi = std::min(g.desc.n_px, S.seg_rows[t.seg + 1] - kHalo + 1);
            if (lo < S.slot_lo[t.slot] || hi > S.slot_hi[t.slot]) return bad("slot rows");
            prev = t.slot;
        }
    }
    for (int c : used)
        if (c < 1 || c > 16) return bad("slot with " + std::to_string(c) + " units");
    std::vector<int> inl(static_cast<size_t>(S.n_slots), 0);
    for (int e = 0; e < S.red_off.back(); ++e) ++inl[S.red_slot[e]];
    for (int c : inl)
        if (c != 1) return bad("reduce lists");
    // cache blocks cover the longest lane of every comb group
    for (int t = 0; t < ntab; ++t)
        for (int k = 0; k < K; ++k)
            for (int gi = 0; gi < ngB; ++gi) {
                const size_t idx = (static_cast<size_t>(t) * K + k) * ngB + gi;
                const int64_t rows = S.cache_off[idx + 1] - S.cache_off[idx];
                for (int l = 0; l < 32; ++l) {
                    const int r = S.groups[static_cast<size_t>(gi) * 32 + l];
                    if (r < 0) continue;
                    const RayP& rp = rays[static_cast<size_t>(list[t]) * R + r];
                    const int n = rp.dV > 0 ? seg_entry(rp, S.seg_rows[k + 1]) - seg_entry(rp, S.seg_rows[k])
                                            : seg_entry(rp, S.seg_rows[k]) - seg_entry(rp, S.seg_rows[k + 1]);
                    if (n > rows) return bad("cache block shorter than a lane");
                }
            }
    // the consecutive-ray layout (PGET_GNB_ADJ): every ray once, blocks cover the longest lane
    {
        const int ngC = S.max_gC;
        std::vector<int> cseen(R, 0);
        for (int gi = 0; gi < ngC; ++gi)
            for (int l = 0; l < 32; ++l) {
                const int r = S.groupsC[static_cast<size_t>(gi) * 32 + l];
                if (r >= 0) ++cseen[r];
            }
        for (int c : cseen)
            if (c != 1) return bad("consecutive-ray groups");
        for (int t = 0; t < ntab; ++t)
            for (int k = 0; k < K; ++k)
                for (int gi = 0; gi < ngC; ++gi) {
                    const size_t idx = (static_cast<size_t>(t) * K + k) * ngC + gi;
                    const int64_t rows = S.cache_offC[idx + 1] - S.cache_offC[idx];
                    for (int l = 0; l < 32; ++l) {
                        const int r = S.groupsC[static_cast<size_t>(gi) * 32 + l];
                        if (r < 0) continue;
                        const RayP& rp = rays[static_cast<size_t>(list[t]) * R + r];
                        const int n = rp.dV > 0 ? seg_entry(rp, S.seg_rows[k + 1]) - seg_entry(rp, S.seg_rows[k])
                                                : seg_entry(rp, S.seg_rows[k]) - seg_entry(rp, S.seg_rows[k + 1]);
                        if (n > rows) return bad("consecutive-ray cache block shorter than a lane");
                    }
                }
    }
    // comb groups: every ray once, lanes of a group >= comb_S rays apart
    std::vector<int> rseen(R, 0);
    for (int gi = 0; gi < ngB; ++gi)
        for (int l = 0; l < 32; ++l) {
            const int r = S.groups[static_cast<size_t>(gi) * 32 + l];
            if (r < 0) continue;
            ++rseen[r];
            for (int l2 = 0; l2 < l; ++l2) {
                const int r2 = S.groups[static_cast<size_t>(gi) * 32 + l2];
                if (r2 >= 0 && std::abs(r2 - r) < g.comb_S) return bad("comb lanes too close");
            }
        }
    for (int c : rseen)
        if (c != 1) return bad("comb groups do not cover every ray once");
    (void)J;
    return PGET_OK;
}

pget_status pget_workspace_region(pget_geometry h, int op, int region, size_t* offset, size_t* bytes)
{
    if (!h || !offset || !bytes) return fail(PGET_ERR_INVALID_ARGUMENT, "NULL argument");
    if (op != PGET_OP_GN_CG_STEP) return fail(PGET_ERR_INVALID_ARGUMENT, "pget_workspace_region: op");
    const WS w = carve(h->g, op, reinterpret_cast<char*>(uintptr_t(1) << 40));
    const float* p = nullptr;
    switch (region) {
    case PGET_WS_P_LAM: p = w.pl; break;
    case PGET_WS_P_MU: p = w.pm; break;
    case PGET_WS_Q_LAM: p = w.ql; break;
    case PGET_WS_Q_MU: p = w.qm; break;
    default: return fail(PGET_ERR_INVALID_ARGUMENT, "pget_workspace_region: region");
    }
    *offset = static_cast<size_t>(reinterpret_cast<uintptr_t>(p) - (uintptr_t(1) << 40));
    *bytes = static_cast<size_t>(h->g.desc.batch) * h->g.desc.n_px * h->g.desc.n_px * sizeof(float);
    return PGET_OK;
}

pget_status pget_check_finite(const float* x, size_t n, int32_t* flag_dev, pget_stream_t stream)
{
    NvtxRange nvtx_("pget_check_finite");
    if (n == 0) return PGET_OK;
    if (!x || !flag_dev) return fail(PGET_ERR_INVALID_ARGUMENT, "pget_check_finite: NULL pointer");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    CK(cudaMemsetAsync(flag_dev, 0, sizeof(int32_t), s));
    launch_k(finite_scan_kernel, vec_grid(n), kVecThreads, 0, s, x, n, flag_dev); note();
    CK(cudaGetLastError());
    int32_t h = 0;
    CK(cudaMemcpyAsync(&h, flag_dev, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (h) return fail(PGET_ERR_NOT_FINITE, "pget_check_finite: the array holds a NaN or an infinity");
    return PGET_OK;
}

pget_status pget_profile_begin(int32_t max_launches)
{
    if (max_launches < 0) return fail(PGET_ERR_INVALID_ARGUMENT, "max_launches < 0");
    std::lock_guard<std::mutex> lk(g_prof.mu);
    for (cudaEvent_t e : g_prof.pool) cudaEventDestroy(e);
    g_prof.pool.clear();
    g_prof.recs.clear();
    g_prof.used = 0;
    for (int k = 0; k < 4; ++k) g_prof.mode_launches[k] = 0;
    g_prof.total = 0;
    for (int k = 0; k < 2 * max_launches; ++k) {
        cudaEvent_t e;
        cudaError_t err = cudaEventCreate(&e);
        if (err != cudaSuccess) return cuda_fail(err, "cudaEventCreate");
        g_prof.pool.push_back(e);
    }
    g_prof.on = true;
    return PGET_OK;
}

pget_status pget_profile_end(double* ms, int64_t* launches, int64_t* total)
{
    std::lock_guard<std::mutex> lk(g_prof.mu);
    g_prof.on = false;
    double acc[4] = {0, 0, 0, 0};
    for (const ProfRec& r : g_prof.recs) {
        cudaError_t e = cudaEventSynchronize(r.b);
        if (e != cudaSuccess) return cuda_fail(e, "cudaEventSynchronize");
        float t = 0.f;
        e = cudaEventElapsedTime(&t, r.a, r.b);
        if (e != cudaSuccess) return cuda_fail(e, "cudaEventElapsedTime");
        acc[r.mode] += t;
    }
    for (int k = 0; k < 4; ++k) {
        if (ms) ms[k] = acc[k];
        if (launches) launches[k] = g_prof.mode_launches[k];
    }
    if (total) *total = g_prof.total.load();
    return PGET_OK;
}

}  // extern "C"
