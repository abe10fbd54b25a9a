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
//   blfls::Plan                     a reusable plan (twiddles, spectral tables,
//                                   workspace, CUDA graphs, pinned staging):
//                                   the reference calls smooth() repeatedly with
//                                   one spec (pipelines.cpp:111-115); so do the
//                                   free functions here, through a per-thread
//                                   cache of Plans keyed on the spec
//   blfls::MultiPlan                several GPUs from one process (batch shards
//                                   or row bands, blfls_multi_*)
//
// Errors throw like the reference: std::invalid_argument for shape,
// parameter and non-finite input; std::runtime_error for CUDA failures;
// std::domain_error for configurations outside the GPU envelope.  Header-only;
// link against paper_1812_07122_b200/_lib/libblfls.so.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstring>
#include <list>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
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

inline blfls_params make_params(int h, int w, int c, int gc, int radius, double ss, double sr, double lam,
                                int batch, int device, int pad = 0, int backend = BLFLS_BACKEND_BRUTE,
                                int dt_iterations = 0)
{
    return blfls_params{h, w, c, gc, radius, ss, sr, lam, batch, device, pad, backend, dt_iterations};
}

inline PlanPtr make_plan(const blfls_params& p)
{
    blfls_plan_t raw = nullptr;
    check(blfls_plan_create(&p, &raw));
    return PlanPtr(raw);
}

// f(begin, end) over [0, n) on up to hardware_concurrency threads (chunks of
// >= 1 Mi elements; small ranges run inline): the double <-> float
// conversions of the Image interface
template <class F>
inline void parallel_for(std::size_t n, F&& f)
{
    constexpr std::size_t grain = std::size_t(1) << 20;
    std::size_t nt = std::max(1u, std::thread::hardware_concurrency());
    nt = std::min(nt, n / grain);
    if (nt <= 1) {
        f(std::size_t(0), n);
        return;
    }
    std::vector<std::thread> th;
    th.reserve(nt);
    const std::size_t per = (n + nt - 1) / nt;
    for (std::size_t t = 0; t < nt; ++t) {
        const std::size_t b = t * per, e = std::min(n, b + per);
        if (b < e) th.emplace_back([&f, b, e] { f(b, e); });
    }
    for (auto& t : th) t.join();
}

inline void to_float(const double* src, float* dst, std::size_t n)
{
    parallel_for(n, [&](std::size_t b, std::size_t e) {
        for (std::size_t i = b; i < e; ++i) dst[i] = static_cast<float>(src[i]);
    });
}

inline void to_double(const float* src, double* dst, std::size_t n)
{
    parallel_for(n, [&](std::size_t b, std::size_t e) {
        for (std::size_t i = b; i < e; ++i) dst[i] = src[i];
    });
}

inline std::vector<float> to_f32(const Image& img)
{
    std::vector<float> v(img.size());
    to_float(img.data().data(), v.data(), v.size());
    return v;
}

// page-locked float buffer (blfls_host_alloc), grown on demand
class PinnedFloats {
public:
    PinnedFloats() = default;
    PinnedFloats(const PinnedFloats&) = delete;
    PinnedFloats& operator=(const PinnedFloats&) = delete;
    ~PinnedFloats() { blfls_host_free(p_); }
    float* reserve(std::size_t n)
    {
        if (n > n_) {
            blfls_host_free(p_);
            p_ = nullptr;
            n_ = 0;
            void* q = nullptr;
            check(blfls_host_alloc(n * sizeof(float), &q));
            p_ = static_cast<float*>(q);
            n_ = n;
        }
        return p_;
    }

private:
    float* p_ = nullptr;
    std::size_t n_ = 0;
};

}  // namespace detail

/// A reusable BLF-LS plan: created once per (shape, parameters, device),
/// then run on any number of batches <= max_batch.  Not thread-safe (one per
/// host thread), like the C ABI's plans.
class Plan {
public:
    explicit Plan(const blfls_params& prm) : prm_(prm), plan_(detail::make_plan(prm)) {}
    Plan(int height, int width, int channels, int guide_channels, int radius, double sigma_s,
         double sigma_r, double lambda, int max_batch = 1, int device = 0, int pad = 0,
         int backend = BLFLS_BACKEND_BRUTE, int dt_iterations = 0)
        : Plan(detail::make_params(height, width, channels, guide_channels, radius, sigma_s, sigma_r,
                                   lambda, max_batch, device, pad, backend, dt_iterations))
    {
    }
    const blfls_params& params() const { return prm_; }
    blfls_plan_t handle() const { return plan_.get(); }
    std::size_t image_floats() const { return (std::size_t)prm_.height * prm_.width * prm_.channels; }
    std::size_t guide_floats() const { return (std::size_t)prm_.height * prm_.width * prm_.guide_channels; }

    /// float host buffers, batch x C x H x W (pinned memory is fastest);
    /// returns when `out` is written
    void run(const float* img, const float* guide, int batch, int iters, float* out,
             bool check_finite = true)
    {
        detail::check(blfls_run(plan_.get(), img, guide, batch, iters, out, nullptr,
                                BLFLS_HOST_PTRS | BLFLS_SYNC | (check_finite ? BLFLS_CHECK_FINITE : 0u)));
    }
    /// queued H2D / compute / D2H on the plan's streams; consecutive calls
    /// overlap.  Buffers must stay valid and `out` is readable after sync()
    /// (which throws std::invalid_argument for deferred non-finite input).
    void run_async(const float* img, const float* guide, int batch, int iters, float* out,
                   bool check_finite = true)
    {
        detail::check(blfls_run(plan_.get(), img, guide, batch, iters, out, nullptr,
                                BLFLS_HOST_PTRS | BLFLS_ASYNC | (check_finite ? BLFLS_CHECK_FINITE : 0u)));
    }
    void sync() { detail::check(blfls_sync(plan_.get())); }

    /// the Image interface: double <-> float through pinned staging reused
    /// across calls (multi-threaded conversion for large images)
    Image run(const Image& img, const Image* guide, int iters)
    {
        if (img.width() != prm_.width || img.height() != prm_.height || img.channels() != prm_.channels)
            throw std::invalid_argument("Plan::run: image shape does not match the plan");
        if ((guide != nullptr) != (prm_.guide_channels != 0) ||
            (guide && (guide->width() != img.width() || guide->height() != img.height() ||
                       guide->channels() != prm_.guide_channels)))
            throw std::invalid_argument("smooth: guidance image shape does not match input");
        float* in = in_.reserve(img.size());
        float* out = out_.reserve(img.size());
        detail::to_float(img.data().data(), in, img.size());
        float* gd = nullptr;
        if (guide) {
            gd = gd_.reserve(guide->size());
            detail::to_float(guide->data().data(), gd, guide->size());
        }
        run(in, gd, 1, iters, out);
        Image res(img.width(), img.height(), img.channels());
        detail::to_double(out, res.data().data(), img.size());
        return res;
    }

    /// lsgrad_solve_fft (solver.cpp:88-124) with this plan's lambda / pad
    Image solve(const Image& g, const Image& tx, const Image& ty)
    {
        if (!g.same_shape(tx) || !g.same_shape(ty))
            throw std::invalid_argument("lsgrad_solve_fft: target shape does not match image");
        const std::size_t n = g.size();
        float* a = in_.reserve(3 * n);
        float* out = out_.reserve(n);
        detail::to_float(g.data().data(), a, n);
        detail::to_float(tx.data().data(), a + n, n);
        detail::to_float(ty.data().data(), a + 2 * n, n);
        detail::check(blfls_solve(plan_.get(), a, a + n, a + 2 * n, 1, out, nullptr,
                                  BLFLS_HOST_PTRS | BLFLS_CHECK_FINITE | BLFLS_SYNC));
        Image res(g.width(), g.height(), g.channels());
        detail::to_double(out, res.data().data(), n);
        return res;
    }

private:
    blfls_params prm_;
    detail::PlanPtr plan_;
    detail::PinnedFloats in_, gd_, out_;
};

/// Several GPUs from one process (blfls_multi_*): BLFLS_MULTI_BATCH shards a
/// batch over the device list, BLFLS_MULTI_BAND splits one image into row
/// bands with NVLink peer stores of the targets.  A device may repeat.
class MultiPlan {
public:
    MultiPlan(const blfls_params& prm, const std::vector<int>& devices, int mode = BLFLS_MULTI_BATCH)
        : prm_(prm)
    {
        blfls_multi_t m = nullptr;
        detail::check(blfls_multi_create(&prm, devices.data(), (int)devices.size(), mode, &m));
        m_.reset(m);
    }
    const blfls_params& params() const { return prm_; }
    void run(const float* img, const float* guide, int batch, int iters, float* out, bool check_finite = true)
    {
        detail::check(blfls_multi_run(m_.get(), img, guide, batch, iters, out,
                                      BLFLS_HOST_PTRS | (check_finite ? BLFLS_CHECK_FINITE : 0u)));
    }

private:
    struct Deleter {
        void operator()(blfls_multi_s* m) const { blfls_multi_destroy(m); }
    };
    blfls_params prm_;
    std::unique_ptr<blfls_multi_s, Deleter> m_;
};

namespace detail {

// per-thread cache of Plans keyed on every plan parameter (LRU, 8 entries)
inline Plan& cached_plan(const blfls_params& p)
{
    thread_local std::list<Plan> cache;
    for (auto it = cache.begin(); it != cache.end(); ++it) {
        const blfls_params& q = it->params();
        if (q.height == p.height && q.width == p.width && q.channels == p.channels &&
            q.guide_channels == p.guide_channels && q.radius == p.radius && q.sigma_s == p.sigma_s &&
            q.sigma_r == p.sigma_r && q.lambda == p.lambda && q.max_batch == p.max_batch &&
            q.device == p.device && q.pad == p.pad && q.backend == p.backend &&
            q.dt_iterations == p.dt_iterations) {
            cache.splice(cache.begin(), cache, it);
            return cache.front();
        }
    }
    if (cache.size() >= 8) cache.pop_back();
    cache.emplace_front(p);
    return cache.front();
}

}  // namespace detail

/// `iters` cascaded smooth() calls with the brute-force (joint) BLF, guide
/// held fixed.  guide: nullptr, 1 channel, or img.channels() channels.
/// Repeated calls with the same shape and parameters reuse one cached Plan.
inline Image blf_ls(const Image& img, const Image* guide, double lambda, double sigma_s,
                    double sigma_r, int iters = 1, int radius = -1, int device = 0, int pad = 0,
                    int backend = BLFLS_BACKEND_BRUTE, int dt_iterations = 0)
{
    if (guide && (guide->width() != img.width() || guide->height() != img.height() ||
                  (guide->channels() != 1 && guide->channels() != img.channels())))
        throw std::invalid_argument("smooth: guidance image shape does not match input");
    Plan& plan = detail::cached_plan(detail::make_params(img.height(), img.width(), img.channels(),
                                                         guide ? guide->channels() : 0, radius, sigma_s,
                                                         sigma_r, lambda, 1, device, pad, backend,
                                                         dt_iterations));
    return plan.run(img, guide, iters);
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
    detail::to_double(out.data(), res.data().data(), out.size());
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
    detail::to_double(out.data(), res.data().data(), out.size());
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
    Plan& plan = detail::cached_plan(
        detail::make_params(g.height(), g.width(), g.channels(), 0, 1, 1.0, 1.0, lambda, 1, device, pad));
    return plan.solve(g, tx, ty);
}

}  // namespace blfls
