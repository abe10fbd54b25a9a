// ref_capi.cpp -- extern "C" entry points into the reference translation
// units compiled unmodified into oracle/_ref/libepls_ref.so (see
// oracle/Makefile).  TEST INFRASTRUCTURE ONLY: tests/ use it to pin the
// oracle restatement and to generate golden vectors (tests/golden/), and
// bench.py --impl reference times ref_blf_ls on the host cores.
//
// Status: 0 ok, 1 std::invalid_argument, 7 std::length_error, 9 other.
#include <chrono>
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <vector>

#include "../blfls_oracle.h"
#include "epls/bilateral.hpp"
#include "epls/image.hpp"
#include "epls/metrics.hpp"
#include "epls/pipelines.hpp"
#include "epls/serial.hpp"
#include "epls/solver.hpp"
#include "epls/testimage.hpp"

using namespace epls;

namespace {

PlanarImage wrap(const double* p, int c, int h, int w)
{
    PlanarImage img(w, h, c);
    std::memcpy(img.data().data(), p, sizeof(double) * img.size());
    return img;
}

void unwrap(const PlanarImage& img, double* out)
{
    std::memcpy(out, img.data().data(), sizeof(double) * img.size());
}

template <class F>
int guarded(F&& f)
{
    try {
        f();
        return 0;
    } catch (const std::invalid_argument&) {
        return 1;
    } catch (const std::length_error&) {
        return 7;
    } catch (...) {
        return 9;
    }
}

// pipelines.cpp:18-31 (anonymous-namespace helpers, restated)
PlanarImage to_unit_range(const PlanarImage& grad)
{
    PlanarImage out = grad;
    for (double& v : out.data()) v = (v + 1.0) * 0.5;
    return out;
}

PlanarImage plane_view(const PlanarImage& img, int c)
{
    PlanarImage out(img.width(), img.height(), 1);
    std::copy(img.plane(c), img.plane(c) + img.plane_size(), out.plane(0));
    return out;
}

// Brute-force joint BLF with an explicit radius.  When radius equals the
// reference's ceil(3*sigma_s) (bilateral.cpp:37) this is the unmodified
// reference blf_brute; otherwise the restatement orc_blf_brute_r, which
// follows bilateral.cpp:28-77 with only the radius changed.
PlanarImage blf_r(const PlanarImage& src, const PlanarImage& guide, const RangeSpatialParams& p,
                  int radius)
{
    if (radius < 0 || radius == static_cast<int>(std::ceil(3.0 * p.sigma_s)))
        return blf_brute(src, guide, p);
    PlanarImage out(src.width(), src.height(), src.channels());
    const int st = orc_blf_brute_r(src.data().data(), src.channels(), guide.data().data(),
                                   guide.channels(), src.height(), src.width(), radius, p.sigma_s,
                                   p.sigma_r, out.data().data());
    if (st != 0) throw std::invalid_argument("blf_brute_r: invalid input");
    return out;
}

// pipelines.cpp:57-94, BLF_LS branch, blf_r substituted for blf_grid at
// pipelines.cpp:47; every other step calls the reference function.
PlanarImage smooth_brute(const PlanarImage& g, const SmootherSpec& spec, int radius,
                         double* t_blf, double* t_solve)
{
    require_finite(g, "smooth");
    if (spec.guidance && (spec.guidance->width() != g.width() ||
                          spec.guidance->height() != g.height() ||
                          spec.guidance->channels() != g.channels()))
        throw std::invalid_argument("smooth: guidance image shape does not match input");
    const auto t0 = std::chrono::steady_clock::now();
    auto [gn, rec] = normalize_to_unit(g);
    const int pad = spec.solve.pad;
    const PlanarImage gp = reflect_pad(gn, pad);
    const GradientField grads = forward_gradients(gp);
    GradientField guide_grads;
    if (spec.guidance) {
        const PlanarImage guide_n = normalize_to_unit(*spec.guidance).first;
        guide_grads = forward_gradients(reflect_pad(guide_n, pad));
    }
    const GradientField& gg = spec.guidance ? guide_grads : grads;
    GradientField target{PlanarImage(gp.width(), gp.height(), gp.channels()),
                         PlanarImage(gp.width(), gp.height(), gp.channels())};
    for (int axis = 0; axis < 2; ++axis) {
        const PlanarImage& src = axis == 0 ? grads.gx : grads.gy;
        const PlanarImage& gd = axis == 0 ? gg.gx : gg.gy;
        PlanarImage& dst = axis == 0 ? target.gx : target.gy;
        for (int c = 0; c < gp.channels(); ++c) {
            const PlanarImage filtered =
                blf_r(to_unit_range(plane_view(src, c)), to_unit_range(plane_view(gd, c)), spec.blf,
                      radius);
            const double* s = filtered.plane(0);
            double* o = dst.plane(c);
            for (std::size_t i = 0; i < dst.plane_size(); ++i) o[i] = 2.0 * s[i] - 1.0;
        }
    }
    const auto t1 = std::chrono::steady_clock::now();
    const SolveParams inner{spec.solve.lambda, 0};
    PlanarImage u = crop_border(lsgrad_solve_fft(gp, target, inner), pad);
    PlanarImage out = denormalize(u, rec);
    const auto t2 = std::chrono::steady_clock::now();
    if (t_blf) *t_blf += std::chrono::duration<double>(t1 - t0).count();
    if (t_solve) *t_solve += std::chrono::duration<double>(t2 - t1).count();
    return out;
}

} // namespace

extern "C" {

int ref_blf_brute(const double* src, int cs, const double* guide, int cg, int h, int w,
                  double sigma_s, double sigma_r, double* out)
{
    return guarded([&] {
        unwrap(blf_brute(wrap(src, cs, h, w), wrap(guide, cg, h, w), {sigma_s, sigma_r}), out);
    });
}

int ref_serial_blf_brute(const double* src, int cs, const double* guide, int cg, int h, int w,
                         double sigma_s, double sigma_r, double* out)
{
    return guarded([&] {
        unwrap(serial::blf_brute(wrap(src, cs, h, w), wrap(guide, cg, h, w), {sigma_s, sigma_r}),
               out);
    });
}

int ref_blf_grid(const double* src, const double* guide, int h, int w, double sigma_s,
                 double sigma_r, double* out)
{
    return guarded([&] {
        unwrap(blf_grid(wrap(src, 1, h, w), wrap(guide, 1, h, w), {sigma_s, sigma_r}), out);
    });
}

int ref_forward_gradients(const double* img, int c, int h, int w, double* gx, double* gy)
{
    return guarded([&] {
        const GradientField g = forward_gradients(wrap(img, c, h, w));
        unwrap(g.gx, gx);
        unwrap(g.gy, gy);
    });
}

int ref_normalize_to_unit(const double* img, int c, int h, int w, double* out, double* lo,
                          double* hi)
{
    return guarded([&] {
        auto [n, rec] = normalize_to_unit(wrap(img, c, h, w));
        unwrap(n, out);
        *lo = rec.lo;
        *hi = rec.hi;
    });
}

int ref_lsgrad_solve_fft(const double* g, const double* tx, const double* ty, int c, int h, int w,
                         double lambda, int pad, double* u)
{
    return guarded([&] {
        const GradientField t{wrap(tx, c, h, w), wrap(ty, c, h, w)};
        unwrap(lsgrad_solve_fft(wrap(g, c, h, w), t, {lambda, pad}), u);
    });
}

int ref_ls_solve_fft(const double* g, int c, int h, int w, double lambda, int pad, double* u)
{
    return guarded([&] { unwrap(ls_solve_fft(wrap(g, c, h, w), {lambda, pad}), u); });
}

int ref_difference_otf(int h, int w, double* ox, double* oy)
{
    return guarded([&] {
        auto [a, b] = difference_otf(h, w);
        std::memcpy(ox, a.data(), sizeof(double) * 2 * a.size());
        std::memcpy(oy, b.data(), sizeof(double) * 2 * b.size());
    });
}

int ref_spectral_denominator(int h, int w, double lambda, double* out)
{
    return guarded([&] { unwrap(spectral_denominator(h, w, lambda), out); });
}

int ref_dense_solve(const double* g, const double* tx, const double* ty, int c, int h, int w,
                    double lambda, double* u)
{
    return guarded([&] {
        const PlanarImage gi = wrap(g, c, h, w);
        if (tx && ty)
            unwrap(ls_solve_dense_oracle(gi, GradientField{wrap(tx, c, h, w), wrap(ty, c, h, w)},
                                         lambda),
                   u);
        else
            unwrap(ls_solve_dense_oracle(gi, lambda), u);
    });
}

// The reference's own smooth() (BLF_LS runs the bilateral grid, pipelines.cpp:47).
int ref_smooth_grid(const double* g, int c, int h, int w, const double* guide, double sigma_s,
                    double sigma_r, double lambda, int pad, double* out)
{
    return guarded([&] {
        SmootherSpec s;
        s.kind = SmootherKind::BLF_LS;
        s.blf = {sigma_s, sigma_r};
        s.solve = {lambda, pad};
        PlanarImage gd;
        if (guide) {
            gd = wrap(guide, c, h, w);
            s.guidance = &gd;
        }
        unwrap(smooth(wrap(g, c, h, w), s), out);
    });
}

int ref_smooth_brute(const double* g, int c, int h, int w, const double* guide, int radius,
                     double sigma_s, double sigma_r, double lambda, int pad, double* out)
{
    return guarded([&] {
        SmootherSpec s;
        s.kind = SmootherKind::BLF_LS;
        s.blf = {sigma_s, sigma_r};
        s.solve = {lambda, pad};
        PlanarImage gd;
        if (guide) {
            gd = wrap(guide, c, h, w);
            s.guidance = &gd;
        }
        unwrap(smooth_brute(wrap(g, c, h, w), s, radius, nullptr, nullptr), out);
    });
}

// The north-star cascade over the reference pieces: f <- smooth_brute(f)
// `iters` times with the guide fixed; a 1-channel guide for a c-channel image
// is replicated (smooth() rejects the mismatch, pipelines.cpp:60-62).
int ref_blf_ls_pad(const double* g, int c, int h, int w, const double* guide, int guide_c,
                   int radius, double sigma_s, double sigma_r, double lambda, int iters, int pad,
                   double* out, double* t_blf, double* t_solve)
{
    return guarded([&] {
        if (iters < 1) throw std::invalid_argument("blf_ls: iters must be >= 1");
        SmootherSpec s;
        s.kind = SmootherKind::BLF_LS;
        s.blf = {sigma_s, sigma_r};
        s.solve = {lambda, pad};
        PlanarImage gd;
        if (guide) {
            if (guide_c != 1 && guide_c != c)
                throw std::invalid_argument("blf_ls: guide channels must be 1 or match");
            gd = PlanarImage(w, h, c);
            for (int ch = 0; ch < c; ++ch)
                std::memcpy(gd.plane(ch), guide + static_cast<std::size_t>(guide_c == 1 ? 0 : ch) * h * w,
                            sizeof(double) * h * w);
            s.guidance = &gd;
        }
        if (t_blf) *t_blf = 0.0;
        if (t_solve) *t_solve = 0.0;
        PlanarImage f = wrap(g, c, h, w);
        for (int k = 0; k < iters; ++k) f = smooth_brute(f, s, radius, t_blf, t_solve);
        unwrap(f, out);
    });
}

int ref_blf_ls(const double* g, int c, int h, int w, const double* guide, int guide_c, int radius,
               double sigma_s, double sigma_r, double lambda, int iters, double* out,
               double* t_blf, double* t_solve)
{
    return ref_blf_ls_pad(g, c, h, w, guide, guide_c, radius, sigma_s, sigma_r, lambda, iters, 0, out,
                          t_blf, t_solve);
}

int ref_nc_filter(const double* src, int cs, const double* guide, int cg, int h, int w,
                  double sigma_s, double sigma_r, int iters, double* out)
{
    return guarded([&] {
        unwrap(nc_filter(wrap(src, cs, h, w), wrap(guide, cg, h, w), {sigma_s, sigma_r, iters}), out);
    });
}

int ref_serial_nc_filter(const double* src, int cs, const double* guide, int cg, int h, int w,
                         double sigma_s, double sigma_r, int iters, double* out)
{
    return guarded([&] {
        unwrap(serial::nc_filter(wrap(src, cs, h, w), wrap(guide, cg, h, w), {sigma_s, sigma_r, iters}),
               out);
    });
}

double ref_nc_box_radius(double sigma_s, int iter, int total)
{
    return nc_box_radius(sigma_s, iter, total);
}

int ref_smooth_nc(const double* g, int c, int h, int w, const double* guide, double sigma_s,
                  double sigma_r, int dt_iters, double lambda, int pad, double* out)
{
    return guarded([&] {
        SmootherSpec s;
        s.kind = SmootherKind::NC_LS;
        s.dt = {sigma_s, sigma_r, dt_iters};
        s.solve = {lambda, pad};
        PlanarImage gd;
        if (guide) {
            gd = wrap(guide, c, h, w);
            s.guidance = &gd;
        }
        unwrap(smooth(wrap(g, c, h, w), s), out);
    });
}

int ref_rolling_nc_ls(const double* g, int c, int h, int w, double sigma_s, double sigma_r,
                      int dt_iters, double lambda, int pad, int n, double init_sigma, double* out)
{
    return guarded([&] {
        unwrap(rolling_nc_ls(wrap(g, c, h, w), {sigma_s, sigma_r, dt_iters}, {lambda, pad},
                             {n, init_sigma}),
               out);
    });
}

int ref_random_image(int w, int h, int c, unsigned long long seed, double lo, double hi, double* out)
{
    return guarded([&] { unwrap(testimage::random_image(w, h, c, seed, lo, hi), out); });
}

int ref_natural_scene(int w, int h, int c, unsigned long long seed, double* out)
{
    return guarded([&] { unwrap(testimage::natural_scene(w, h, c, seed), out); });
}

int ref_gaussian_blur(const double* img, int c, int h, int w, double sigma, double* out)
{
    return guarded([&] { unwrap(gaussian_blur(wrap(img, c, h, w), sigma), out); });
}

double ref_max_abs_gradient(const double* img, int c, int h, int w)
{
    return max_abs_gradient(wrap(img, c, h, w));
}

} // extern "C"
