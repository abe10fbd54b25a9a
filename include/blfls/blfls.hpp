// blfls.hpp -- C++ host API over the C ABI (blfls.h), mirroring the
// reference library's entry points and error behaviour:
//
//   blfls::Image                    ~ epls::PlanarImage (include/epls/image.hpp:9-41):
//                                     planar doubles, channels in {1, 3}
//   blfls::SmootherSpec             ~ epls::SmootherSpec (pipelines.hpp:16-23)
//   blfls::smooth(g, spec)          ~ epls::smooth (pipelines.cpp:57-94), BLF_LS / NC_LS
//   blfls::rolling_nc_ls(...)       ~ epls::rolling_nc_ls (pipelines.cpp:96-117)
//   blfls::gaussian_blur(img, s)    ~ epls::gaussian_blur (image.cpp:114-158)
//   blfls::blf_brute(src, guide, p) ~ epls::blf_brute (bilateral.cpp:28-77)
//   blfls::flash_no_flash(a, f, s)  ~ epls::flash_no_flash (applications.cpp:58-64)
//   blfls::blf_ls(...)              the north-star cascade (iters smooth() calls)
//   blfls::lsgrad_solve_fft(...)    ~ epls::lsgrad_solve_fft (solver.cpp:88-124)
//
// Errors throw like the reference: std::invalid_argument for shape,
// parameter and non-finite input; std::runtime_error for CUDA failures;
// std::domain_error for configurations outside the GPU envelope.  Header-only;
// link against paper_1812_07122_b200/_lib/libblfls.so.
#pragma once

#include <cmath>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "blfls/blfls.h"

namespace blfls {

class Image {
public:
    Image() = default;
    Image(int width, int height, int channels, double fill = 0.0)
        : width_(width), height_(height), channels_(channels)
    {
        // image.cpp:14-17
        if (width <= 0 || height <= 0)
            throw std::invalid_argument("PlanarImage: width and height must be positive");
        if (channels != 1 && channels != 3)
            throw std::invalid_argument("PlanarImage: channels must be 1 or 3");
        data_.assign(static_cast<std::size_t>(width) * height * channels, fill);
    }
    int width() const { return width_; }
    int height() const { return height_; }
    int channels() const { return channels_; }
    std::size_t plane_size() const { return static_cast<std::size_t>(width_) * height_; }
    std::size_t size() const { return data_.size(); }
    double& at(int c, int y, int x) { return data_[plane_size() * c + static_cast<std::size_t>(y) * width_ + x]; }
    double at(int c, int y, int x) const { return data_[plane_size() * c + static_cast<std::size_t>(y) * width_ + x]; }
    std::vector<double>& data() { return data_; }
    const std::vector<double>& data() const { return data_; }
    bool same_shape(const Image& o) const
    {
        return width_ == o.width_ && height_ == o.height_ && channels_ == o.channels_;
    }

private:
    int width_ = 0, height_ = 0, channels_ = 0;
    std::vector<double> data_;
};

struct RangeSpatialParams {
    double sigma_s = 8.0;
    double sigma_r = 0.1;
};

struct SolveParams {
    double lambda = 1024.0;
    int pad = 16;  // reflect padding (solver.hpp:12-15); 0 = periodic
};

struct DtParams {  // domain_transform.hpp:7-11
    double sigma_s = 8.0;
    double sigma_r = 0.1;
    int iterations = 3;
};

struct RollingParams {  // pipelines.hpp:25-28
    int n = 3;
    double init_sigma = 2.5;
};

enum class SmootherKind { BLF_LS, NC_LS };  // the gradient-filter kinds of pipelines.hpp:11

struct SmootherSpec {
    SmootherKind kind = SmootherKind::BLF_LS;
    RangeSpatialParams blf{12.0, 0.04};
    DtParams dt{12.0, 0.05, 3};
    SolveParams solve{};
    const Image* guidance = nullptr;
    int radius = -1;  // < 0: ceil(3 sigma_s) as bilateral.cpp:37
    int device = 0;
    int backend = BLFLS_BACKEND_BRUTE;  // or BLFLS_BACKEND_GRID (the reference's blf_grid)
};

namespace detail {

inline void check(blfls_status st)
{
    if (st == BLFLS_OK) return;
    const std::string msg = blfls_last_error();
    switch (st) {
        case BLFLS_EINVAL:
        case BLFLS_ENONFINITE: throw std::invalid_argument(msg);
        case BLFLS_EUNSUPPORTED: throw std::domain_error(msg);
        default: throw std::runtime_error(msg);
    }
}

struct PlanDeleter {
    void operator()(blfls_plan_s* p) const { blfls_plan_destroy(p); }
};
using PlanPtr = std::unique_ptr<blfls_plan_s, PlanDeleter>;

inline PlanPtr make_plan(int h, int w, int c, int gc, int radius, double ss, double sr, double lam,
                         int batch, int device, int pad = 0, int backend = BLFLS_BACKEND_BRUTE,
                         int dt_iterations = 0)
{
    blfls_params p{h, w, c, gc, radius, ss, sr, lam, batch, device, pad, backend, dt_iterations};
    blfls_plan_t raw = nullptr;
    check(blfls_plan_create(&p, &raw));
    return PlanPtr(raw);
}

inline std::vector<float> to_f32(const Image& img)
{
    std::vector<float> v(img.size());
    for (std::size_t i = 0; i < v.size(); ++i) v[i] = static_cast<float>(img.data()[i]);
    return v;
}

}  // namespace detail

/// `iters` cascaded smooth() calls with the brute-force (joint) BLF, guide
/// held fixed.  guide: nullptr, 1 channel, or img.channels() channels.
inline Image blf_ls(const Image& img, const Image* guide, double lambda, double sigma_s,
                    double sigma_r, int iters = 1, int radius = -1, int device = 0, int pad = 0,
                    int backend = BLFLS_BACKEND_BRUTE, int dt_iterations = 0)
{
    if (guide && (guide->width() != img.width() || guide->height() != img.height() ||
                  (guide->channels() != 1 && guide->channels() != img.channels())))
        throw std::invalid_argument("smooth: guidance image shape does not match input");
    auto plan = detail::make_plan(img.height(), img.width(), img.channels(),
                                  guide ? guide->channels() : 0, radius, sigma_s, sigma_r, lambda,
                                  1, device, pad, backend, dt_iterations);
    std::vector<float> in = detail::to_f32(img), out(img.size()), gd;
    if (guide) gd = detail::to_f32(*guide);
    detail::check(blfls_run(plan.get(), in.data(), guide ? gd.data() : nullptr, 1, iters,
                            out.data(), nullptr, BLFLS_HOST_PTRS | BLFLS_CHECK_FINITE | BLFLS_SYNC));
    Image res(img.width(), img.height(), img.channels());
    for (std::size_t i = 0; i < out.size(); ++i) res.data()[i] = out[i];
    return res;
}

/// `iters` cascaded smooth() calls of kind NC_LS (nc_filter, domain_transform.cpp:138-156).
inline Image nc_ls(const Image& img, const Image* guide, double lambda, const DtParams& dt,
                   int iters = 1, int device = 0, int pad = 0)
{
    if (dt.iterations < 1) throw std::invalid_argument("nc_filter: iterations must be >= 1");
    return blf_ls(img, guide, lambda, dt.sigma_s, dt.sigma_r, iters, 0, device, pad,
                  BLFLS_BACKEND_DT, dt.iterations);
}

/// epls::smooth for kinds BLF_LS (brute-force BLF, or the grid via spec.backend)
/// and NC_LS, including reflect padding.
inline Image smooth(const Image& g, const SmootherSpec& spec)
{
    if (spec.guidance && !spec.guidance->same_shape(g))
        throw std::invalid_argument("smooth: guidance image shape does not match input");
    if (spec.kind == SmootherKind::NC_LS)
        return nc_ls(g, spec.guidance, spec.solve.lambda, spec.dt, 1, spec.device, spec.solve.pad);
    return blf_ls(g, spec.guidance, spec.solve.lambda, spec.blf.sigma_s, spec.blf.sigma_r, 1,
                  spec.radius, spec.device, spec.solve.pad, spec.backend);
}

/// epls::gaussian_blur (image.cpp:114-158) on the GPU.
inline Image gaussian_blur(const Image& img, double sigma, int device = 0)
{
    std::vector<float> in = detail::to_f32(img), out(img.size());
    detail::check(blfls_gaussian_blur(in.data(), img.channels(), img.height(), img.width(), sigma,
                                      out.data(), device, nullptr, BLFLS_HOST_PTRS | BLFLS_SYNC));
    Image res(img.width(), img.height(), img.channels());
    for (std::size_t i = 0; i < out.size(); ++i) res.data()[i] = out[i];
    return res;
}

/// epls::blf_brute (bilateral.cpp:28-77): standalone (joint) bilateral filter;
/// radius < 0 is the reference's ceil(3 sigma_s).
inline Image blf_brute(const Image& src, const Image& guide, const RangeSpatialParams& p,
                       int radius = -1, int device = 0)
{
    if (src.width() != guide.width() || src.height() != guide.height())
        throw std::invalid_argument("bilateral: src and guide dimensions differ");
    std::vector<float> s = detail::to_f32(src), g = detail::to_f32(guide), out(src.size());
    detail::check(blfls_blf_brute(s.data(), src.channels(), g.data(), guide.channels(), src.height(),
                                  src.width(), 1, radius, p.sigma_s, p.sigma_r, out.data(), device,
                                  nullptr, BLFLS_HOST_PTRS | BLFLS_CHECK_FINITE | BLFLS_SYNC));
    Image res(src.width(), src.height(), src.channels());
    for (std::size_t i = 0; i < out.size(); ++i) res.data()[i] = out[i];
    return res;
}

/// epls::rolling_nc_ls (pipelines.cpp:96-117).
inline Image rolling_nc_ls(const Image& g, const DtParams& dt, const SolveParams& sp,
                           const RollingParams& rp, int device = 0)
{
    if (rp.n < 1) throw std::invalid_argument("rolling_nc_ls: n must be >= 1");
    if (!(rp.init_sigma > 0.0))
        throw std::invalid_argument("rolling_nc_ls: init_sigma must be positive");
    Image guide = gaussian_blur(g, rp.init_sigma, device);
    Image u;
    for (int k = 0; k < rp.n; ++k) {
        u = nc_ls(g, &guide, sp.lambda, dt, 1, device, sp.pad);
        guide = u;
    }
    return u;
}

/// epls::flash_no_flash: joint smoothing of `noflash` guided by `flash`.
inline Image flash_no_flash(const Image& noflash, const Image& flash, SmootherSpec spec)
{
    if (!noflash.same_shape(flash))
        throw std::invalid_argument("flash_no_flash: image shapes differ");
    spec.guidance = &flash;
    return smooth(noflash, spec);
}

/// epls::lsgrad_solve_fft (targets and image reflect-padded by `pad`).
inline Image lsgrad_solve_fft(const Image& g, const Image& tx, const Image& ty, double lambda,
                              int device = 0, int pad = 0)
{
    if (!g.same_shape(tx) || !g.same_shape(ty))
        throw std::invalid_argument("lsgrad_solve_fft: target shape does not match image");
    if (pad < 0) throw std::invalid_argument("solver: pad must be >= 0");
    auto plan = detail::make_plan(g.height(), g.width(), g.channels(), 0, 1, 1.0, 1.0, lambda, 1,
                                  device, pad);
    std::vector<float> a = detail::to_f32(g), b = detail::to_f32(tx), c = detail::to_f32(ty),
                       out(g.size());
    detail::check(blfls_solve(plan.get(), a.data(), b.data(), c.data(), 1, out.data(), nullptr,
                              BLFLS_HOST_PTRS | BLFLS_CHECK_FINITE | BLFLS_SYNC));
    Image res(g.width(), g.height(), g.channels());
    for (std::size_t i = 0; i < out.size(); ++i) res.data()[i] = out[i];
    return res;
}

}  // namespace blfls
