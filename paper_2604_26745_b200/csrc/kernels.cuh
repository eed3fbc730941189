// kernels.cuh -- kernel argument blocks and declarations (library-private).
#pragma once
#include <utility>
#include <cuda_runtime.h>

#include "internal.h"

namespace pget {

// ---- programmatic dependent launch (PDL).  Every library kernel is launched with programmatic stream
// serialisation (launch_k; env PGET_PDL=0 turns it off) and starts with pdl_entry(): it lets its own
// dependent grid be scheduled at once, then waits until its predecessor grid has completed and its
// memory is visible -- stream order is unchanged, but the next kernel's launch overlaps the tail of
// the previous one (both in direct launches and in captured CUDA graphs).
__device__ __forceinline__ void pdl_entry()
{
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
}
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    if (pdl_enabled()) {
        cfg.attrs = at;
        cfg.numAttrs = 1;
    }
    return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

enum { MODE_FWD = 0, MODE_JVP = 1, MODE_VJP = 2, MODE_GN = 3 };
enum { SC_INIT = 0, SC_GAMMA = 1, SC_ZETA = 2, SC_PRED = 3, SC_TRIAL = 4 };

struct ProjArgs {
    const RayP* rays;       // [n_ab][R] oriented-frame fixed-point ray parameters
    const TaskD* tasks;     // schedule (schedule.cpp): CTA c runs tasks [cta_begin[c], cta_begin[c+1])
    const int32_t* cta_begin;
    const int32_t* groups;  // [n][32] comb groups of the schedule (-1 = idle lane)
    const float* w;         // [J] sub-ray weights (float)
    const float2* img2[2];  // [B][P][P] (lam, mu): normal / transposed, zero halo
    const float4* img4[2];  // [B][P][P] (lam, mu, dlam, dmu)
    float2* slots;          // [n_slots][N][Ns] fp32 partial gradients (g_lam, g_mu)
    const float* win;       // [B][n_ab][n_det] VJP weights
    float* y;               // [B][n_ab][n_det]
    float* dy;              // [B][n_ab][n_det]
    int N, Ns, P, n_det, J, R, n_ab, B;
    int P8, P16;            // 8 P and 16 P: byte row pitches of the staged float2 / float4 bands (walk_a; constant-bank operands)
    int P4, planeB4;        // 4 P and 4 (RbB + 1) P: byte strides of the cached scatter's accumulator (constant-bank operands)
    int dup_half;           // n_angles / 2 when duplicate angle-banks are merged (geometry dup), else 0
    int RbA, RbB, nbA, nbB, passesA, passesB;   // sweep A: 32 adjacent rays per warp; sweep B: comb groups
    int stage_bytes, off_wacc, off_rout, off_gsh;   // dynamic shared memory layout (bytes)
    float delta;            // Delta
    float cf, ch;           // -Delta log2(e), -Delta log2(e) / 2
    // segmented adjoint (seg_a_kernel / seg_b_kernel): the phase's units and stage lists per CTA,
    // the K row segments, the per-(unit, ray) partial sums of phase A
    const UnitD* units;
    const int32_t* u_begin;
    const StageD* stages;
    const int32_t* s_begin;
    const int32_t* seg_rows;
    int K, n_groups, off_rsc, off_q1;
    const int32_t* slot_lo;  // [n_slots] rows [slot_lo, slot_hi) a slot's units can write (zeroed by the first)
    const int32_t* slot_hi;
    // GN with cached Jacobian coefficients (lin_kernel / jvpc_kernel / gnb_kernel)
    float4* cache;           // rows of 32 lanes: (alpha, beta, alpha', beta') per sample
    const int64_t* cache_off;
    int64_t cache_rows_member;
    int cache_ng;            // groups per (angle-bank, segment) of the cache layout (comb or consecutive-ray groups)
    int ntab;
    float* jp;               // [n_canon][2][R] per-ray JVP partials of a segment (both directions)
    float* segp;            // [n_canon][kSegFields][R]
    float* gw;              // [B * ntab][2][R] GN scatter weights (w_r, w'_r) of gnw_kernel, or null
    float* gscale;          // [B * ntab][8] fixed-point scale bounds of the cached scatter (null: float path)
    int cellmax;            // max consecutive samples of a ray in one pixel cell
    const float2* var_cw;   // model variant (N3): [J][n_t] (W_j(d_i), c_i), null when off
    int n_t;
};

// pixel-basis model variant (N3, reading R-pb; sid.cu): one CTA per (angle-bank, member)
struct SidArgs {
    const double* dir;      // [n_ab][2] (cos phi, sin phi), the O1 table
    const double* off;      // [n_banks][R] offsets sigma, the O1 table
    const float2* img2;     // [B][P][P] (lam, mu), normal orientation, zero halo
    const float4* img4;     // [B][P][P] (lam, mu, dlam, dmu)
    const float* wj;        // [J] sub-ray weights outside the ray sums (ones with the response)
    const float* dj2;       // [J] delta_j^2 log2(e) (response)
    float* y;               // [B][n_ab][n_det]
    float* dy;
    const float* win;       // VJP weights [B][n_ab][n_det]
    float4* ray;            // [B][n_ab][R] adjoint pass 1: (w_r, G, Gc, -)
    float2* raybd;          // [B][n_ab][R] (sum r E, sum r |lam| c E)
    unsigned* bound;        // [B][2] float bits: per-member magnitude bounds (lam, mu planes)
    unsigned long long* acc;   // [B][2][N][N] 64-bit fixed-point adjoint (lam plane, mu plane)
    double nhits;           // rays through one pixel, at most (all angle-banks)
    double det_radius;
    float c_slope, r_slope, sig0, lmax;
    int N, P, R, J, n_det, n_ab, nB, B;
    int dpc, nch;           // detectors per CTA, CTAs per angle-bank (set by the launchers)
};
cudaError_t launch_sid_proj(int mode, bool var, const SidArgs& A, cudaStream_t s);
cudaError_t launch_sid_adj(int mode, bool var, const SidArgs& A, double2* gacc, cudaStream_t s);
cudaError_t set_sid_smem_limit(size_t bytes);

constexpr int kSegFields = 9;
// rows of 32 entries allocated past the end of the GN coefficient cache: gnb_kernel's entry ring and
// L2 prefetch read ahead of a lane's last sample without bounds checks (the values are never used)
constexpr int kCachePadRows = 16;
// stage buffers of the warp-specialised phase A.  Two (double buffering) leave bands half again as tall as three
// in the same shared memory (config 4: 26 rows instead of 17), and the per-band costs (band_steps, fold_a, the
// barrier hand-over) weigh more than the third buffer's slack: config 4 forward 0.252 -> 0.242 ms, JVP 0.689 ->
// 0.663 ms, LM 22.16 -> 21.87 ms; four: 0.256 / 0.696 / 22.24 ms (profiles/ab_r02nn_stages.txt)
#ifndef PGET_SEGA_STAGES
#define PGET_SEGA_STAGES 2
#endif
constexpr int kSegAStages = PGET_SEGA_STAGES;   // kSegFields: s, sc, g, gc, ds, dg, p1, p2, p3 (see seg_a_kernel)

struct CGState {
    double zeta, a, bcg;
    int stop, pad_;
};


// geometry priors P1, P2 (pget_set_prior): weights already scaled by the LM continuation; a null mask
// switches its term off
// the LM solve's feasible set (N1): box (lam_lo, lam_hi, mu_lo, mu_hi) and, for c > 0, lam <= c mu
struct BoxK {
    float4 b;
    float c;
};

struct PriorArgs {
    const float* m1;
    const float* m2;
    float a1, a2;
};

__global__ void pack2_kernel(const float* lam, const float* mu, const float* slam, const float* smu, float2* out,
                             float2* outT, float* ut_lam, float* ut_mu, int N, int P, int B, int has_box,
                             BoxK box);
__global__ void project_step_kernel(const float* ul, const float* um, float* sl, float* sm, size_t n, BoxK box);
__global__ void lm_update_kernel(float* ul, float* um, const float* tl, const float* tm, const pget_gn_stats* stats,
                                 float* betav, int n2);
__global__ void fill_kernel(float* x, float v, int n);
__global__ void clamp_kernel(float* ul, float* um, size_t n, BoxK box);
__global__ void pack4_kernel(const float* lam, const float* mu, const float* dl, const float* dm, float4* out,
                             float4* outT, int N, int P, int B);
__global__ void reduce_slots_kernel(const float2* slots, double2* part, int N, int Ns, int B, int G,
                                    const int32_t* red_off, const int32_t* red_slot, const int32_t* slot_lo,
                                    const int32_t* slot_hi);
__global__ void finish_kernel(const double2* part, int G, const float* xl, const float* xm, float alpha, float beta,
                              float sign, float* outl, float* outm, const float* dotl, const float* dotm,
                              double* partial, float* copy1l, float* copy1m, float* copy2l, float* copy2m,
                              float* zerol, float* zerom, int N, PriorArgs pr, const float* betav = nullptr);
__global__ void residual_kernel(float* y, const float* ymeas, double* partial, int nper);
__global__ void sumsq_kernel(const float* x, double* partial, int nper);
__global__ void regsq_kernel(const float* xl, const float* xm, double* partial, int N);
// SGP inner solver (O11): CGState carries a = the Barzilai-Borwein length, bcg = the line-search step
__global__ void sgp_init_kernel(const float* bl, const float* bm, float* gl, float* gm, CGState* st, int n2, int B);
__global__ void sgp_dir_kernel(const float* ul, const float* um, const float* sl, const float* sm, const float* gl,
                               const float* gm, const CGState* st, BoxK box, float* dl, float* dm, double* pgd,
                               double* pdd, int n2);
__global__ void sgp_scalar_kernel(int k, int final_, const double* pgd, const double* pdd, const double* pdhd,
                                  const double* pqq, int nblk, CGState* st, pget_gn_stats* stats, int B);
__global__ void sgp_update_kernel(float* sl, float* sm, float* gl, float* gm, const float* dl, const float* dm,
                                  const float* ql, const float* qm, const CGState* st, int n2);
__global__ void priorsq_kernel(const float* xl, const float* xm, PriorArgs pr, double* partial, int N);
__global__ void priordot_kernel(const float* ul, const float* um, const float* sl, const float* sm, PriorArgs pr,
                                double* pdot, double* psq, int N);
__global__ void dot2_kernel(const float* al, const float* am, const float* bl, const float* bm, double* partial,
                            int n2);
__global__ void cg_update1_kernel(float* sl, float* sm, float* zl, float* zm, const float* pl, const float* pm,
                                  const float* ql, const float* qm, const CGState* st, double* partial, int n2);
__global__ void cg_update2_kernel(const float* zl, const float* zm, float* pl, float* pm, const CGState* st,
                                  int n2);
__global__ void cg_fused_kernel(const double2* part, int G, float alpha, float beta_h, const float* betav, float* sl,
                                float* sm, float* zl, float* zm, float* pl, float* pm, float* ql, float* qm,
                                double* pg, double* pz, CGState* st, pget_gn_stats* stats, int k, int N, int B,
                                int nblk, float4* img4n, float4* img4t, int P, PriorArgs pr);
__global__ void dotsq_kernel(const float* a, const float* b, double* pdot, double* psq, int nper);
__global__ void lapdot_kernel(const float* ul, const float* um, const float* sl, const float* sm, double* pdot,
                              double* psq, int N);
__global__ void diff2_kernel(const float* al, const float* am, const float* bl, const float* bm, float* ol,
                             float* om, size_t n);
__global__ void guard_scalar_kernel(const double* P, int nblk, int B, double alpha, double kappa,
                                    pget_safeguard_stats* out, int has_prior);
__global__ void guard_select_kernel(const float* ul, const float* um, const float* sl, const float* sm,
                                    const float* cl, const float* cm, const pget_safeguard_stats* st, float* ol,
                                    float* om, int n2);
__global__ void scalar_kernel(int op, int k, const double* p0, const double* p1, const double* p2, int nblk,
                              CGState* st, pget_gn_stats* stats, int B, double alpha, double beta_h,
                              const float* betav, const double* pp = nullptr);

}  // namespace pget

namespace pget {
cudaError_t launch_proj(int mode, int maxg, bool paired, const ProjArgs& A, int grid, int block, size_t smem,
                        cudaStream_t s);
cudaError_t set_proj_smem_limit(int mode, size_t smem);
cudaError_t launch_seg(int phase, int mode, int maxg, bool paired, const ProjArgs& A, int grid, int block,
                       size_t smem, cudaStream_t s);
cudaError_t set_seg_smem_limit(int phase, int mode, size_t smem);
// GN with cached coefficients: phase 0 lin_kernel, 1 jvpc_kernel, 2 gnb_kernel
cudaError_t launch_gnc(int phase, bool paired, const ProjArgs& A, int grid, int block, size_t smem, cudaStream_t s);
cudaError_t set_gnc_smem_limit(size_t smem);
cudaError_t launch_jvp_combine(const ProjArgs& A, const int32_t* tabs, int ntab, int B, cudaStream_t s);
cudaError_t launch_fwd_combine(bool paired, const ProjArgs& A, const int32_t* tabs, int ntab, int B, cudaStream_t s);
cudaError_t launch_gnw(bool paired, const ProjArgs& A, const int32_t* tabs, int ntab, int B, cudaStream_t s,
                       bool sino = false);
cudaError_t launch_jsq(bool paired, const ProjArgs& A, double* sq, int grid, int block, size_t smem, cudaStream_t s);
cudaError_t launch_jsq_member(const double* sq, int ntab, int B, int nblk, double* partial, cudaStream_t s);
__global__ void finite_scan_kernel(const float* __restrict__ x, size_t n, int32_t* flag);
int proj_warps(int mode);
int proj_ctas_per_sm(int mode);
}  // namespace pget
