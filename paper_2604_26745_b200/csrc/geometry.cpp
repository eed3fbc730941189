// geometry.cpp -- host geometry builder of libpget (native C++, fp64).
//
// Builds the O1 tables of SURVEY.md §8(c.2) for the detector geometry of
// PAPER.md:33 (two opposing banks of detectors, full rotation) and the
// parallel-ray line parametrisation s*theta_perp + t*theta of PAPER.md:48-54
// (eq:fwd_model).  The fp64 operation order follows the O1 text exactly and the
// file is compiled with -ffp-contract=off, so the exported tables are bit-exact
// with any other implementation of the same text (tests/test_abi.py compares them
// with the oracle's; the two share no code).  It then derives the library's own
// 32.32 fixed-point sample parametrisation (RayP) used by the kernels.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <vector>

#include "internal.h"

namespace pget {

static const double kPi = 3.14159265358979323846;

pget_status build_geometry(const pget_geometry_desc* d, Geometry* g, std::string* err)
{
    if (!d) { *err = "desc is NULL"; return PGET_ERR_INVALID_ARGUMENT; }
    char buf[256];
    if (d->n_px < 2 || d->n_px > 8192 || d->n_angles < 1 || d->n_angles > 1000000 || d->n_banks < 1 ||
        d->n_banks > 2 || d->n_det < 2 || d->n_det > 100000 || d->n_subrays < 1 ||
        d->n_subrays > kMaxSubrays || d->batch < 1 || !(d->subray_sigma > 0.0) || !(d->step_px > 0.0) ||
        !std::isfinite(d->subray_sigma) || !std::isfinite(d->step_px) || !std::isfinite(d->bank1_shift) ||
        d->step_px > 4.0) {
        std::snprintf(buf, sizeof buf,
                      "invalid geometry desc (n_px=%d n_angles=%d n_banks=%d n_det=%d J=%d batch=%d "
                      "sigma=%g step=%g shift=%g)",
                      d->n_px, d->n_angles, d->n_banks, d->n_det, d->n_subrays, d->batch, d->subray_sigma,
                      d->step_px, d->bank1_shift);
        *err = buf;
        return PGET_ERR_INVALID_ARGUMENT;
    }
    if (!std::isfinite(d->det_radius) || !std::isfinite(d->c_slope) || !std::isfinite(d->r_slope) ||
        (d->det_radius > 0.0 && (d->c_slope < 0.0 || d->r_slope < 0.0))) {
        *err = "invalid model variant (det_radius, c_slope, r_slope must be finite; slopes >= 0)";
        return PGET_ERR_INVALID_ARGUMENT;
    }
    if (d->pixel_basis != 0 && d->pixel_basis != 1) {
        *err = "pixel_basis must be 0 or 1";
        return PGET_ERR_INVALID_ARGUMENT;
    }
    g->desc = *d;
    g->sid = d->pixel_basis == 1;
    const int N = d->n_px, nA = d->n_angles, nB = d->n_banks, nd = d->n_det, J = d->n_subrays;

    // t-lattice: h = 2/N, Delta = step_px h, T = Delta ceil((sqrt2 + h)/Delta), n_t = 2T/Delta
    g->h = 2.0 / N;
    g->delta = d->step_px * g->h;
    const double m = std::ceil((std::sqrt(2.0) + g->h) / g->delta);
    g->T = g->delta * m;
    g->n_t = 2 * static_cast<int>(m);

    // angles theta_a = 2 pi a / n_A; bank b: phi = theta_a + b pi
    g->angles.resize(nA);
    for (int a = 0; a < nA; ++a) g->angles[a] = 2.0 * kPi * static_cast<double>(a) / static_cast<double>(nA);
    g->dirs.resize(static_cast<size_t>(nA) * nB * 2);
    for (int a = 0; a < nA; ++a)
        for (int b = 0; b < nB; ++b) {
            const double phi = g->angles[a] + static_cast<double>(b) * kPi;
            g->dirs[(static_cast<size_t>(a) * nB + b) * 2 + 0] = std::cos(phi);
            g->dirs[(static_cast<size_t>(a) * nB + b) * 2 + 1] = std::sin(phi);
        }

    // offsets sigma_{b,d,j} = s_d (+ shift p on bank 1) + delta_j; p = 2/(n_det-1)
    const double p = 2.0 / static_cast<double>(nd - 1);
    g->offsets.resize(static_cast<size_t>(nB) * nd * J);
    for (int b = 0; b < nB; ++b)
        for (int dd = 0; dd < nd; ++dd) {
            double s = static_cast<double>(2 * dd - (nd - 1)) / static_cast<double>(nd - 1);
            if (b == 1) s = s + d->bank1_shift * p;
            for (int j = 0; j < J; ++j) {
                const double dj = static_cast<double>(2 * j + 1 - J) / static_cast<double>(2 * J) * p;
                g->offsets[(static_cast<size_t>(b) * nd + dd) * J + j] = s + dj;
            }
        }

    // weights w_j = exp(-delta_j^2 / (2 (sigma p)^2)) / sum
    g->weights.resize(J);
    {
        const double sp = d->subray_sigma * p;
        double sum = 0.0;
        for (int j = 0; j < J; ++j) {
            const double dj = static_cast<double>(2 * j + 1 - J) / static_cast<double>(2 * J) * p;
            g->weights[j] = std::exp(-(dj * dj) / (2.0 * sp * sp));
            sum += g->weights[j];
        }
        for (int j = 0; j < J; ++j) g->weights[j] = g->weights[j] / sum;
    }
    g->wf.resize(J);
    for (int j = 0; j < J; ++j) g->wf[j] = static_cast<float>(g->weights[j]);

    // model variant (N3, reading R-N3): d_i = det_radius - t_i, c_i = 1 + c_slope d_i, W_j(d_i) the
    // normalised Gaussian response of width sigma p (1 + r_slope d_i) (the O1-style fp64 text order)
    g->var = d->det_radius > 0.0;
    g->var_c.clear();
    g->var_w.clear();
    if (g->var) {
        if (d->det_radius < g->T) {
            std::snprintf(buf, sizeof buf, "det_radius %g < T %g: a sample would lie behind the detector",
                          d->det_radius, g->T);
            *err = buf;
            return PGET_ERR_INVALID_ARGUMENT;
        }
        g->var_c.resize(g->n_t);
        g->var_w.resize(static_cast<size_t>(J) * g->n_t);
        for (int i = 0; i < g->n_t; ++i) {
            const double t = -g->T + (i + 0.5) * g->delta;
            const double dd = d->det_radius - t;
            g->var_c[i] = 1.0 + d->c_slope * dd;
            const double sp = d->subray_sigma * p * (1.0 + d->r_slope * dd);
            double sum = 0.0;
            for (int j = 0; j < J; ++j) {
                const double dj = static_cast<double>(2 * j + 1 - J) / static_cast<double>(2 * J) * p;
                g->var_w[static_cast<size_t>(j) * g->n_t + i] = std::exp(-(dj * dj) / (2.0 * sp * sp));
                sum += g->var_w[static_cast<size_t>(j) * g->n_t + i];
            }
            for (int j = 0; j < J; ++j)
                g->var_w[static_cast<size_t>(j) * g->n_t + i] = g->var_w[static_cast<size_t>(j) * g->n_t + i] / sum;
        }
    }

    // clip: slab test of x(t) = sigma omega_perp + t omega against |x|,|y| <= 1 + h/2
    const double bb = 1.0 + g->h / 2.0;
    g->clip.resize(static_cast<size_t>(nA) * nB * nd * J * 2);
    int64_t nominal = 0;
    for (int a = 0; a < nA; ++a)
        for (int b = 0; b < nB; ++b) {
            const double c = g->dirs[(static_cast<size_t>(a) * nB + b) * 2 + 0];
            const double s = g->dirs[(static_cast<size_t>(a) * nB + b) * 2 + 1];
            const double om[2] = {c, s};
            const double op[2] = {-s, c};
            for (int dd = 0; dd < nd; ++dd)
                for (int j = 0; j < J; ++j) {
                    const double sigma = g->offsets[(static_cast<size_t>(b) * nd + dd) * J + j];
                    double tin = -INFINITY, tout = INFINITY;
                    for (int k = 0; k < 2; ++k) {
                        const double base = sigma * op[k];
                        if (om[k] == 0.0) {
                            if (std::fabs(base) > bb) { tin = INFINITY; tout = -INFINITY; }
                        } else {
                            const double t1 = (-bb - base) / om[k];
                            const double t2 = (bb - base) / om[k];
                            const double lo = t1 < t2 ? t1 : t2, hi = t1 < t2 ? t2 : t1;
                            if (lo > tin) tin = lo;
                            if (hi < tout) tout = hi;
                        }
                    }
                    int32_t ilo = 0, ihi = -1;
                    if (tin <= tout) {
                        double lo = std::ceil((tin + g->T) / g->delta - 0.5);
                        double hi = std::floor((tout + g->T) / g->delta - 0.5);
                        if (lo < 0.0) lo = 0.0;
                        if (hi > static_cast<double>(g->n_t - 1)) hi = static_cast<double>(g->n_t - 1);
                        if (lo <= hi) { ilo = static_cast<int32_t>(lo); ihi = static_cast<int32_t>(hi); }
                    }
                    const size_t r = ((static_cast<size_t>(a) * nB + b) * nd + dd) * J + j;
                    g->clip[2 * r] = ilo;
                    g->clip[2 * r + 1] = ihi;
                    nominal += ihi - ilo + 1;
                }
        }
    g->n_samples_nominal = nominal * d->batch;

    g->R = nd * J;
    g->n_ab = nA * nB;
    g->P = (N + 2 * kHalo + 1) & ~1;   // even: 16-B aligned rows of float2 for the bulk band copies

    // orientation classes: class 1 when the ray runs closer to the x axis,
    // so that in its oriented frame every ray crosses image rows at >= 1/sqrt2 rows per pixel.
    g->orient.resize(g->n_ab);
    g->task_ab.clear();
    for (int ab = 0; ab < g->n_ab; ++ab) {
        const double c = g->dirs[static_cast<size_t>(ab) * 2 + 0];
        const double s = g->dirs[static_cast<size_t>(ab) * 2 + 1];
        g->orient[ab] = std::fabs(c) > std::fabs(s) ? 1 : 0;
    }
    g->dup = (nA % 2 == 0) && nB == 2 && d->bank1_shift == 0.0 && !g->sid;   // pixel basis: every angle-bank
    g->pair = g->dup && !g->var;   // the variant's opposite-direction attenuation does not factor
    auto traced = [&](int ab) { return !g->dup || (ab / nB) < nA / 2; };
    for (int cls = 0; cls < 2; ++cls)
        for (int ab = 0; ab < g->n_ab; ++ab)
            if (traced(ab) && g->orient[ab] == cls) g->task_ab.push_back(ab);
    g->n_tab = static_cast<int>(g->task_ab.size());
    g->n_samples_traced = 0;
    for (int ab : g->task_ab)
        for (int r = 0; r < g->R; ++r) {
            const size_t k = static_cast<size_t>(ab) * g->R + r;
            const int32_t lo = g->clip[2 * k], hi = g->clip[2 * k + 1];
            if (hi >= lo) g->n_samples_traced += hi - lo + 1;
        }
    g->n_samples_traced *= d->batch;
    g->n_class0 = 0;
    for (int ab = 0; ab < g->n_ab; ++ab) g->n_class0 += traced(ab) && g->orient[ab] == 0;
    g->task_ab_p.clear();
    g->n_class0_p = 0;
    g->n_samples_traced_p = 0;
    if (g->dup) {
        for (int ab : g->task_ab)
            if (ab % nB == 0) {
                g->task_ab_p.push_back(ab);
                g->n_class0_p += g->orient[ab] == 0;
                for (int r = 0; r < g->R; ++r) {
                    const size_t k = static_cast<size_t>(ab) * g->R + r;
                    const int32_t lo = g->clip[2 * k], hi = g->clip[2 * k + 1];
                    if (hi >= lo) g->n_samples_traced_p += hi - lo + 1;
                }
            }
        g->n_samples_traced_p *= d->batch;
    }

    {
        const double a = (p / J) / g->h;   // ray spacing in pixels
        long S = static_cast<long>(std::ceil((2.0 * std::sqrt(2.0) + 1e-6) / a));
        if (S < 1) S = 1;
        if (S > g->R) S = g->R;
        g->comb_S = static_cast<int>(S);
        g->gnbC_stride = a < 0.5 ? 2 : 1;   // measured (LM iteration, stride 1/2/3/4): config 4 25.0/24.0/24.2/24.7 ms, config 2 4.83/4.77/4.80/4.85
        // samples whose 2x2 bilinear support contains a given pixel: rays within the support's
        // width (2 sqrt2 px) x samples of one ray inside it; consecutive samples in one cell
        const double st = d->step_px;
        const double n_near = (std::floor(2.0 * std::sqrt(2.0) / a) + 2.0) * (std::floor(2.0 * std::sqrt(2.0) / st) + 2.0);
        g->cellmax = static_cast<int>(std::floor(std::sqrt(2.0) / st)) + 1;
        g->gnb_int = n_near < 512.0 * g->cellmax;
    }
    if (g->sid) {
        // crossings per ray (interior pixel edges of both axes + 1: the pixel-basis "samples") and the
        // most rays through one pixel: per bank, the most offsets inside any window of the width of a
        // pixel's projection (<= sqrt2 h), summed over the angle-banks (the fixed-point scale, sid.cu)
        const double hN = 0.5 * N;
        int64_t cross = 0;
        for (int ab = 0; ab < g->n_ab; ++ab) {
            const int b = ab % nB;
            const double c = g->dirs[static_cast<size_t>(ab) * 2], s = g->dirs[static_cast<size_t>(ab) * 2 + 1];
            for (int r = 0; r < g->R; ++r) {
                const double sigma = g->offsets[static_cast<size_t>(b) * g->R + r];
                const double X0[2] = {(-sigma * s + 1.0) * hN, (sigma * c + 1.0) * hN}, w[2] = {c * hN, s * hN};
                double tin = -INFINITY, tout = INFINITY;
                bool ok = true;
                for (int k = 0; k < 2; ++k) {
                    if (w[k] == 0.0) { ok = ok && X0[k] > 0.0 && X0[k] < N; continue; }
                    const double t1 = -X0[k] / w[k], t2 = (N - X0[k]) / w[k];
                    tin = std::max(tin, std::min(t1, t2));
                    tout = std::min(tout, std::max(t1, t2));
                }
                if (!ok || !(tin < tout)) continue;
                int64_t n = 1;
                for (int k = 0; k < 2; ++k) {
                    const double a = X0[k] + tin * w[k], e = X0[k] + tout * w[k];
                    const double lo = std::min(a, e), hi = std::max(a, e);
                    n += std::max<int64_t>(0, static_cast<int64_t>(std::ceil(hi)) - static_cast<int64_t>(std::floor(lo)) - 1);
                }
                cross += n;
            }
        }
        g->n_samples_nominal = cross * d->batch;
        g->n_samples_traced = g->n_samples_nominal;
        const double win = std::sqrt(2.0) * g->h * (1.0 + 1e-9);
        double nh = 0.0;
        for (int b = 0; b < nB; ++b) {
            std::vector<double> o(g->offsets.begin() + static_cast<size_t>(b) * g->R,
                                  g->offsets.begin() + static_cast<size_t>(b + 1) * g->R);
            std::sort(o.begin(), o.end());
            int best = 0;
            for (size_t i = 0, k = 0; i < o.size(); ++i) {
                while (o[i] - o[k] > win) ++k;
                best = std::max(best, static_cast<int>(i - k + 1));
            }
            nh += best;
        }
        g->sid_nhits = nh * nA;
    }
    return PGET_OK;
}

// 32.32 fixed-point sample positions in padded pixel coordinates, in each angle-bank's oriented
// frame (class 1: u and v swapped, the ray samples the transposed image).
void build_ray_params(const Geometry& g, std::vector<RayP>* rays)
{
    const int nB = g.desc.n_banks, nd = g.desc.n_det, J = g.desc.n_subrays;
    rays->resize(static_cast<size_t>(g.n_ab) * g.R);
    const double scale = 4294967296.0;   // 2^32
    const int64_t bias = int64_t(1) << 8; // +2^-24 px: round the 23-bit fraction to nearest
    const double t0 = -g.T + 0.5 * g.delta;
    for (int ab = 0; ab < g.n_ab; ++ab) {
        const int b = ab % nB;
        const double c = g.dirs[static_cast<size_t>(ab) * 2 + 0];
        const double s = g.dirs[static_cast<size_t>(ab) * 2 + 1];
        const double du = g.delta * c / g.h, dv = g.delta * s / g.h;
        const int64_t dU = std::llround(du * scale), dV = std::llround(dv * scale);
        const bool tr = g.orient[ab] != 0;
        for (int dd = 0; dd < nd; ++dd)
            for (int j = 0; j < J; ++j) {
                const double sigma = g.offsets[(static_cast<size_t>(b) * nd + dd) * J + j];
                const double x0 = sigma * (-s) + t0 * c;
                const double y0 = sigma * c + t0 * s;
                const double u0 = (x0 + 1.0) / g.h - 0.5 + kHalo;
                const double v0 = (y0 + 1.0) / g.h - 0.5 + kHalo;
                RayP& rp = (*rays)[static_cast<size_t>(ab) * g.R + dd * J + j];
                const int64_t U0 = std::llround(u0 * scale) + bias, V0 = std::llround(v0 * scale) + bias;
                rp.U0 = tr ? V0 : U0;
                rp.V0 = tr ? U0 : V0;
                rp.dU = tr ? dV : dU;
                rp.dV = tr ? dU : dV;
                const size_t r = static_cast<size_t>(ab) * nd * J + dd * J + j;
                rp.ilo = g.clip[2 * r];
                rp.ihi = g.clip[2 * r + 1];
            }
    }
}

}  // namespace pget
