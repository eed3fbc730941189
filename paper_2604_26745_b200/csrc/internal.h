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
    std::vector<int32_t> task_ab_p;   // bank-0 traced angle-banks (class 0, then class 1); empty without dup
    int n_class0_p = 0;
    int64_t n_samples_traced_p = 0;
    int P;        // padded image side (rows = cols = P, even): N + 2 kHalo rounded up to even
    // orientation classes: class 0 = |dV| >= |dU| (image used as is), class 1 = transposed image
    std::vector<int8_t> orient;   // [n_ab]
    std::vector<int32_t> task_ab; // [n_tab] traced angle-banks in processing order: class 0, then class 1
    int n_class0 = 0;
    // ray parts: a task is (member, traced angle-bank, part); part p owns detectors
    // [part_det[p], part_det[p+1]) so that the static task ranges of the persistent CTAs balance
    static constexpr int kMaxParts = 8;
    int n_parts = 1;
    int part_det[kMaxParts + 1] = {0};
    int part_grp[kMaxParts + 1] = {0};   // comb groups of part p: [part_grp[p], part_grp[p+1])
    // comb groups: <= 32 rays of one part whose offsets differ pairwise by >= comb_S rays (>= 2 sqrt2 px)
    int comb_S = 1;
    int n_groups = 0;
    std::vector<int32_t> groups;  // [n_groups][32] ray index in the angle-bank, -1 = idle lane
    // device tables
    RayP* d_rays = nullptr;       // [n_ab][R] oriented frame
    int32_t* d_groups = nullptr;  // [n_groups][32]
    int32_t* d_task_ab = nullptr; // [n_tab + task_ab_p.size()]: task_ab then task_ab_p
    float* d_w = nullptr;         // [J] float weights
    std::vector<float> wf;        // host copy of the float weights
    int sm_count = 148;
    size_t smem_optin = 227 * 1024;
};

}  // namespace pget

struct pget_geometry_s {
    pget::Geometry g;
};

namespace pget {
// geometry.cpp
pget_status build_geometry(const pget_geometry_desc* d, Geometry* g, std::string* err);
void build_ray_params(const Geometry& g, std::vector<RayP>* rays);
void build_parts(Geometry* g, int np);
}  // namespace pget
