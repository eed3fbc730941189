// kernels.cuh -- kernel argument blocks and declarations (library-private).
#pragma once
#include <cuda_runtime.h>

#include "internal.h"

namespace pget {

enum { MODE_FWD = 0, MODE_JVP = 1, MODE_VJP = 2, MODE_GN = 3 };
enum { SC_INIT = 0, SC_GAMMA = 1, SC_ZETA = 2, SC_PRED = 3, SC_TRIAL = 4 };

struct ProjArgs {
    const RayP* rays;       // [n_ab][R] oriented-frame fixed-point ray parameters
    const int32_t* groups;  // [n_groups][32] comb ray groups (-1 = idle lane)
    const int32_t* task_ab; // [n_ab] angle-bank order (class 0, then class 1)
    const float* w;         // [J] sub-ray weights (float)
    const float2* img2[2];  // [B][P][P] (lam, mu): normal / transposed, zero halo
    const float4* img4[2];  // [B][P][P] (lam, mu, dlam, dmu)
    float2* slots;          // [C][KS][N][Ns] per-CTA fp32 partial gradients (g_lam, g_mu)
    const float* win;       // [B][n_ab][n_det] VJP weights
    float* y;               // [B][n_ab][n_det]
    float* dy;              // [B][n_ab][n_det]
    int N, Ns, P, n_det, J, R, n_ab, n_class0, B, n_groups, KS;
    int n_tab;              // traced angle-banks per member
    int n_parts;            // ray parts per angle-bank: tasks per member = n_tab * n_parts
    int part_det[Geometry::kMaxParts + 1];   // detectors of part p: [part_det[p], part_det[p+1])
    int part_grp[Geometry::kMaxParts + 1];   // comb groups of part p
    int dup_half;           // n_angles / 2 when duplicate angle-banks are merged (geometry dup), else 0
    int RbA, RbB, nbA, nbB, passesA, passesB;   // sweep A: 32 adjacent rays per warp; sweep B: comb groups
    int stage_bytes, off_wacc, off_rout, off_gsh;   // dynamic shared memory layout (bytes)
    float delta;            // Delta
    float cf, ch;           // -Delta log2(e), -Delta log2(e) / 2
};

// Partial-gradient slots: the tasks (member, angle-bank) of one orientation class of one member are
// cut into chunks of kChunk consecutive tasks; a CTA accumulates each chunk it touches into its own
// fp32 slot (so a slot sums at most kChunk angle-banks) and reduce_slots_kernel adds the slots in fp64.
constexpr int kChunk = 16;

__host__ __device__ inline int64_t chunk_of(int64_t t, int n_tab, int n_class0)
{
    const int64_t m = t / n_tab;
    const int k = static_cast<int>(t - m * n_tab);
    const int nc0 = (n_class0 + kChunk - 1) / kChunk, nc1 = (n_tab - n_class0 + kChunk - 1) / kChunk;
    const int local = k < n_class0 ? k / kChunk : nc0 + (k - n_class0) / kChunk;
    return m * (nc0 + nc1) + local;
}

struct CGState {
    double zeta, a, bcg;
    int stop, pad_;
};


__global__ void pack2_kernel(const float* lam, const float* mu, const float* slam, const float* smu, float2* out,
                             float2* outT, float* ut_lam, float* ut_mu, int N, int P, int B);
__global__ void pack4_kernel(const float* lam, const float* mu, const float* dl, const float* dm, float4* out,
                             float4* outT, int N, int P, int B);
__global__ void reduce_slots_kernel(const float2* slots, double2* part, int N, int Ns, int n_tp, int n_class0, int B,
                                    int C, int KS, int G);
__global__ void finish_kernel(const double2* part, int G, const float* xl, const float* xm, float alpha, float beta,
                              float sign, float* outl, float* outm, const float* dotl, const float* dotm,
                              double* partial, float* copy1l, float* copy1m, float* copy2l, float* copy2m,
                              float* zerol, float* zerom, int N);
__global__ void residual_kernel(float* y, const float* ymeas, double* partial, int nper);
__global__ void sumsq_kernel(const float* x, double* partial, int nper);
__global__ void regsq_kernel(const float* xl, const float* xm, double* partial, int N);
__global__ void dot2_kernel(const float* al, const float* am, const float* bl, const float* bm, double* partial,
                            int n2);
__global__ void cg_update1_kernel(float* sl, float* sm, float* zl, float* zm, const float* pl, const float* pm,
                                  const float* ql, const float* qm, const CGState* st, double* partial, int n2);
__global__ void cg_update2_kernel(const float* zl, const float* zm, float* pl, float* pm, const CGState* st,
                                  int n2);
__global__ void scalar_kernel(int op, int k, const double* p0, const double* p1, const double* p2, int nblk,
                              CGState* st, pget_gn_stats* stats, int B, double alpha, double beta);

}  // namespace pget

namespace pget {
cudaError_t launch_proj(int mode, int maxg, bool paired, const ProjArgs& A, int grid, size_t smem, cudaStream_t s);
cudaError_t set_proj_smem_limit(int mode, size_t smem);
int proj_warps(int mode);
int proj_ctas_per_sm(int mode);
}  // namespace pget
