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
    // launch geometry
    int R;        // rays per angle-bank = n_det * J
    int R_pad;    // rounded up to a multiple of 32
    int n_ab;     // n_angles * n_banks
    int Hp, Wp;   // padded image rows / cols
    // device tables
    RayP* d_rays = nullptr;      // [n_ab][R]
    int8_t* d_abdir = nullptr;   // [n_ab] sign of dV
    float* d_w = nullptr;        // [J] float weights
    std::vector<float> wf;       // host copy of the float weights
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
void build_ray_params(const Geometry& g, std::vector<RayP>* rays, std::vector<int8_t>* abdir);
}  // namespace pget
