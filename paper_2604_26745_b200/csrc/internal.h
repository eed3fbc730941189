// internal.h -- library-private types shared by the host geometry builder and the
// CUDA kernels of libpget.  Not part of the C ABI (see include/pget.h).
#pragma once
#include <stdint.h>
#include <stddef.h>

#include <string>
#include <vector>

#include "../../include/pget.h"

namespace pget {

constexpr int kHalo = 2;          // zero halo (pixels) around the padded images
constexpr int kFracBits = 32;     // fixed-point fraction bits of sample positions
constexpr int kMaxSubrays = 64;

// Per-ray sample parametrisation in padded pixel coordinates, 32.32 fixed point:
//   u_i = U0 + i*dU, v_i = V0 + i*dV   (u = (x+1)/h - 1/2 + kHalo, v likewise)
// in the angle-bank's oriented frame: for orientation class 1 (|dU| > |dV|) u and v are
// swapped, i.e. the ray samples the transposed image.
// U0/V0 carry a +2^-24 px rounding bias so that (low word >> 9) rounds the
// fraction to nearest at 23 bits (see kernels.cu, frac23()).
struct RayP {
    int64_t U0, V0;
    int64_t dU, dV;
    int32_t ilo, ihi;   // nominal clip; empty: ilo > ihi
};
static_assert(sizeof(RayP) == 40, "RayP layout");

// One projector task (device table entry): member, traced angle-bank, detector range, the comb
// groups (sweep B lane sets) of that range, and the partial slot of the adjoint kind.
enum { kTaskClass1 = 1, kTaskFirst = 2 };
struct TaskD {
    int32_t m, ab;        // batch member, traced angle-bank
    int32_t dlo, dhi;     // detectors [dlo, dhi)
    int32_t gbeg, gend;   // comb groups [gbeg, gend) in Schedule::groups
    int32_t slot;         // partial-gradient slot (adjoint kind), -1 otherwise
    int32_t flags;        // kTaskClass1: orientation class 1; kTaskFirst: first task of its slot in its CTA
};
static_assert(sizeof(TaskD) == 32, "TaskD layout");

// Segmented adjoint (VJP / GN): a unit is (member, traced angle-bank, row segment k of K) over all
// detectors.  Phase A traces every ray of the unit through the segment's rows and stores per-ray
// partial sums; phase B combines the K partials of each ray (optical depth before the segment, the
// tail of G, ...) and scatters the segment's adjoint.  Rows are those of the oriented frame
// (padded); segment k covers sample rows [seg_rows[k], seg_rows[k+1]).
struct UnitD {
    int32_t m, ab;        // batch member, traced angle-bank
    int32_t seg;          // row segment
    int32_t canon;        // (m * n_tab + tab) * K + seg: index of the unit's partials
    int32_t slot;         // phase B: partial-gradient slot
    int32_t flags;        // kTaskClass1; kTaskFirst: first unit of its slot (the slot is zeroed first)
    int32_t pad0, pad1;
};
static_assert(sizeof(UnitD) == 32, "UnitD layout");

// One staged band of a phase: unit (index into the phase's unit list) and band j of the unit in
// processing order.
struct StageD {
    int32_t unit, j;
};

// Sample-row entry of a segment: the largest sample index i <= ihi whose row lies inside the
// segment when the ray is walked from its detector end (dV > 0: rows decrease with i, so the bound
// is the exclusive top row `rtop`; dV < 0: the inclusive bottom row `rbot`).  May be < ilo (empty).
#ifdef __CUDACC__
#define PGET_HD __host__ __device__
#else
#define PGET_HD
#endif
PGET_HD inline int64_t pget_floordiv(int64_t a, int64_t b)   // b > 0
{
    const int64_t q = a / b;
    return (a % b != 0 && a < 0) ? q - 1 : q;
}
PGET_HD inline int seg_entry(const RayP& rp, int rtop_or_rbot)
{
    const int64_t bound = static_cast<int64_t>(rtop_or_rbot) << 32;
    int64_t i;
    if (rp.dV > 0) i = pget_floordiv(bound - 1 - rp.V0, rp.dV);   // V0 + i dV <= bound - 1
    else i = pget_floordiv(rp.V0 - bound, -rp.dV);               // V0 + i dV >= bound
    if (i > rp.ihi) i = rp.ihi;
    if (i < static_cast<int64_t>(rp.ilo) - 1) i = static_cast<int64_t>(rp.ilo) - 1;
    return static_cast<int>(i);
}

enum { kSchedFwd = 0, kSchedJvp = 1, kSchedAdj = 2 };
struct Schedule {
    int C = 0;                        // persistent CTAs (grid size)
    std::vector<int32_t> cta_begin;   // [C + 1]: CTA c runs tasks [cta_begin[c], cta_begin[c+1])
    std::vector<TaskD> tasks;
    std::vector<int32_t> groups;      // [n][32] comb groups, ray index in the angle-bank, -1 = idle lane
    int n_slots = 0;                  // adjoint kind: partial slots
    std::vector<int32_t> red_off;     // [2B + 1]: slots of (member m, class c) are red_slot[red_off[2m+c] ..)
    std::vector<int32_t> red_slot;
    int max_slots_member = 0;
    std::vector<int32_t> slot_lo, slot_hi;   // [n_slots] rows [lo, hi) of a slot that can be nonzero
    int32_t *d_slot_lo = nullptr, *d_slot_hi = nullptr;
    int max_gA = 1, max_gB = 1;       // most sweep-A (32 adjacent rays) / sweep-B (comb) groups of a task
    // segmented adjoint (kind kSchedAdj): K row segments, units and stage lists of phases A and B
    int K = 0;
    std::vector<int32_t> seg_rows;    // [K + 1]
    int CA = 0;                       // phase-A CTAs (phase B uses C)
    std::vector<UnitD> unitsA, unitsB;
    std::vector<int32_t> ua_begin, ub_begin;   // [CA + 1], [C + 1]
    std::vector<StageD> stA, stB;
    std::vector<int32_t> sa_begin, sb_begin;   // [CA + 1], [C + 1]
    int64_t n_canon = 0;
    UnitD* d_unitsA = nullptr;
    UnitD* d_unitsB = nullptr;
    int32_t *d_ua_begin = nullptr, *d_ub_begin = nullptr, *d_sa_begin = nullptr, *d_sb_begin = nullptr;
    StageD *d_stA = nullptr, *d_stB = nullptr;
    int32_t* d_seg_rows = nullptr;
    // GN coefficient cache layout: rows of 32 lanes x float4 at cache_off[(t * K + k) * ngB + g]
    // (+ m * cache_rows_member), t = traced angle-bank index, k = segment, g = comb group
    int ntab = 0;
    std::vector<int64_t> cache_off;
    int64_t cache_rows_member = 0;
    int64_t* d_cache_off = nullptr;
    // the same cache over groups of 32 consecutive rays (the cached GN path's builder and scatter:
    // integer atomics need no comb spacing, and neighbouring rays have similar chords)
    std::vector<int32_t> groupsC;
    int max_gC = 1;
    std::vector<int64_t> cache_offC;
    int64_t cache_rows_memberC = 0;
    int32_t* d_groupsC = nullptr;
    int64_t* d_cache_offC = nullptr;
    int32_t* d_cta_begin = nullptr;
    TaskD* d_tasks = nullptr;
    int32_t* d_groups = nullptr;
    int32_t* d_red_off = nullptr;
    int32_t* d_red_slot = nullptr;
};

// Host-side geometry (fp64 tables built per O1, bit-exact with the oracle's
// formulas) plus the device copies the kernels read.
struct Geometry {
    pget_geometry_desc desc;
    int device;
    // O1 tables (host)
    double h, delta, T;
    int n_t;
    std::vector<double> angles, dirs, offsets, weights;
    std::vector<int32_t> clip;
    // model variant (N3, reading R-N3; desc.det_radius > 0): c_i [n_t], W_j(d_i) [J][n_t]
    bool var = false;
    std::vector<double> var_c, var_w;
    // pixel basis (N3, reading R-pb; desc.pixel_basis): exact intersection lengths (sid.cu), unpaired,
    // every angle-bank traced; sid_nhits bounds the rays through one pixel (the fixed-point scale)
    bool sid = false;
    double sid_nhits = 0.0;
    double* d_sdir = nullptr;     // [n_ab][2] dirs
    double* d_soff = nullptr;     // [n_banks][R] offsets
    float* d_sdj2 = nullptr;      // [J] delta_j^2 log2(e)
    int64_t n_samples_nominal;
    int64_t n_samples_traced = 0;
    // launch geometry
    int R;        // rays per angle-bank = n_det * J
    int n_ab;     // n_angles * n_banks
    // Duplicate angle-banks: with an even number of angles, two banks and no bank-1 shift, the rays of
    // (a + n_A/2, bank 1 - b) are those of (a, b) (phi differs by 2 pi; offsets equal), so only the
    // angle-banks with a < n_A/2 are traced and their results are written / their weights merged
    // for both.  dup == false traces every angle-bank.
    bool dup = false;
    int n_tab;    // angle-banks traced per batch member (n_ab / 2 when dup, else n_ab)
    // Line pairing (with dup): bank 1 of angle a traces the lines of bank 0 of angle a in the opposite
    // direction (phi + pi, mirrored offsets), so the forward, VJP and GN projectors trace only the
    // bank-0 angle-banks with a < n_A/2 and evaluate both directions per traversal.
    // pair == false (PGET_NO_PAIR=1, or a model variant whose opposite-direction attenuation does not
    // factor, N3) keeps the duplicate merging but traces both banks of every traced angle separately
    bool pair = false;
    std::vector<int32_t> task_ab_p;   // bank-0 traced angle-banks (class 0, then class 1); empty without dup
    int n_class0_p = 0;
    int64_t n_samples_traced_p = 0;
    int P;        // padded image side (rows = cols = P, even): N + 2 kHalo rounded up to even
    // orientation classes: class 0 = |dV| >= |dU| (image used as is), class 1 = transposed image
    std::vector<int8_t> orient;   // [n_ab]
    std::vector<int32_t> task_ab; // [n_tab] traced angle-banks in processing order: class 0, then class 1
    int n_class0 = 0;
    // comb stride: rays >= comb_S apart (>= 2 sqrt2 px) have disjoint bilinear footprints
    int comb_S = 1;
    // the cached GN path's ray groups (PGET_GNB_ADJ): blocks of 32 x gnbC_stride consecutive rays, each split
    // into gnbC_stride groups of every gnbC_stride-th ray (~1 px apart: neighbouring lanes rarely share a
    // cell, so fewer same-address atomics; chords still similar)
    int gnbC_stride = 1;
    // device tables
    RayP* d_rays = nullptr;       // [n_ab][R] oriented frame
    float* d_w = nullptr;         // [J] float weights
    float* d_ones = nullptr;      // [J] ones: the variant's response sits inside the ray sums
    void* d_var_cw = nullptr;     // [J][n_t] float2 (W_j(d_i), c_i) (model variant)
    std::vector<float> wf;        // host copy of the float weights
    int sm_count = 148;
    int cg_coop_blocks = 148;   // co-resident blocks of cg_fused_kernel (cooperative launch bound)
    size_t smem_optin = 227 * 1024;
    Schedule sch[3];   // kSchedFwd, kSchedJvp, kSchedAdj (schedule.cpp), device copies owned here
    // segmented standalone JVP: phase-A units over every traced angle-bank (unpaired) + a combine
    Schedule schJ;
    bool jvp_seg = true;
    int32_t* d_tabsJ = nullptr;   // [ntab] traced angle-banks of schJ (task_ab)
    bool fwd_seg = true;          // forward as the segmented VJP-mode phase A + combine
    bool fwd_plain = true;        // standalone forward: forward-mode phase A (plain sums); trial f(u+s) too if fwd_plain_trial
    bool fwd_plain_trial = false;
    bool cg_pdl = true;           // the fused CG kernel launched cooperative + programmatic (PGET_CG_PDL=0: plain cooperative)
    int32_t* d_tabsA = nullptr;   // traced angle-banks of the adjoint schedule (task_ab_p or task_ab)
    bool adj_seg = true;   // adjoint (VJP / GN) as the segmented two-phase projector (else the fused one)
    bool gnb_tall = true;   // gnb_kernel with its own (taller) bands: no stage buffers to fit
    // gnb_kernel with one shared 32-bit fixed-point accumulator (native shared integer atomics):
    // requires every pixel's per-unit sum below 2^31 at the scale that keeps a pending cell below
    // 2^22, i.e. (samples near a pixel) / cellmax < 512 (geometry.cpp)
    bool gnb_int = true;
    bool gnb_wide = true;   // cached scatter with one warp per comb group for 17-26 groups (PGET_GNB_WIDE=0: <= 16)
    bool gnb_adj = false;   // cached GN path over consecutive-ray groups (lin_kernel builds the cache; batch 1, PGET_GNB_ADJ)
    bool segA_wide = true;  // phase A with one consumer warp per 32-ray group for 16-26 groups (PGET_SEGA_WIDE=0: 15 warps)
    // pget_gn_apply through the cache too (one product per call: building the cache costs more than
    // it saves; tests set PGET_GN_APPLY_CACHED=1 to pin the cached product at the operator tolerance)
    bool gn_apply_cached = false;
    // geometry priors attached by pget_set_prior (caller-owned device masks; null = off)
    const float* prior_m1 = nullptr;
    const float* prior_m2 = nullptr;
    float prior_a1 = 0.f, prior_a2 = 0.f;
    int cellmax = 1;        // max consecutive samples of one ray inside one pixel cell
    double cache_max_gb = 48.0;   // larger caches fall back to the recomputing GN product (config 5: 25 GB)
    bool gn_hybrid = true;   // cached scatter with the recomputed (J p) (PGET_GN_CACHE=1)
    bool gn_cached = true;   // GN product from the per-LM-iteration Jacobian-entry cache (PGET_GN_CACHE=0: recompute)
    int segA_W = 15, segA_cps = 1;
    int rbA_cap = 64;   // segmented phase A: most rows per band (64 vs 32: GN cfg2 -0.7 %, scripts/rba_exp.sh)   // segmented phase A: warps per CTA, CTAs per SM (scripts/sega_exp.sh)
};

}  // namespace pget

struct pget_geometry_s {
    pget::Geometry g;
};

namespace pget {
// geometry.cpp
pget_status build_geometry(const pget_geometry_desc* d, Geometry* g, std::string* err);
void build_ray_params(const Geometry& g, std::vector<RayP>* rays);
void build_schedule(const Geometry& g, int kind, int C, Schedule* S);
// segmented adjoint schedule: units over CA phase-A CTAs and C phase-B CTAs, slots, comb groups;
// then (once the band heights are known) the stage lists of both phases
void build_adj_schedule(const Geometry& g, const std::vector<RayP>& rays, int CA, int C, Schedule* S,
                        bool unpaired = false);
void build_adj_stages(int RbA, int passesA, int RbB, int passesB, Schedule* S);
}  // namespace pget
