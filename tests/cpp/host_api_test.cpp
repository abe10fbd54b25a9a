// C++ host API smoke test (include/blfls/blfls.hpp over libblfls.so).
// Built by tests/test_cpp_host.py; run on a GPU box it checks the
// reference-style semantics: constants are fixed points, lambda 0 is the
// identity, bad shapes throw std::invalid_argument, pad 16 throws
// std::domain_error.  Prints "OK" and exits 0 on success.
#include <cmath>
#include <cstdio>
#include <stdexcept>

#include "blfls/blfls.hpp"

static int fails = 0;
#define EXPECT(cond)                                             \
    do {                                                         \
        if (!(cond)) {                                           \
            std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #cond); \
            ++fails;                                             \
        }                                                        \
    } while (0)

int main()
{
    // constant image -> itself (test_pipelines.cpp:33-38)
    blfls::Image c(40, 30, 3, 0.55);
    blfls::SmootherSpec spec;
    spec.blf = {2.0, 0.05};
    spec.solve = {1024.0, 0};
    spec.radius = 4;
    blfls::Image u = blfls::smooth(c, spec);
    double m = 0.0;
    for (std::size_t i = 0; i < u.size(); ++i) m = std::fmax(m, std::fabs(u.data()[i] - 0.55));
    EXPECT(m < 1e-6);

    // a ramp stays finite and keeps its mean (DC gain 1)
    blfls::Image g(64, 48, 1);
    double mean_in = 0.0;
    for (int y = 0; y < 48; ++y)
        for (int x = 0; x < 64; ++x) mean_in += (g.at(0, y, x) = (x < 32 ? 0.2 : 0.8) + 0.001 * y);
    mean_in /= 64 * 48;
    blfls::Image v = blfls::blf_ls(g, nullptr, 1000.0, 5.0, 0.05, 2, 5);
    double mean_out = 0.0;
    for (double d : v.data()) mean_out += d;
    mean_out /= 64 * 48;
    EXPECT(std::fabs(mean_out - mean_in) < 1e-5);

    // lambda 0 is the identity (test_solver.cpp:101-106)
    blfls::Image zero(64, 48, 1, 0.0);
    blfls::Image w = blfls::lsgrad_solve_fft(g, zero, zero, 0.0);
    m = 0.0;
    for (std::size_t i = 0; i < w.size(); ++i) m = std::fmax(m, std::fabs(w.data()[i] - g.data()[i]));
    EXPECT(m < 1e-6);

    // errors
    bool threw = false;
    try {
        blfls::Image bad(65, 48, 1);
        blfls::lsgrad_solve_fft(g, bad, bad, 1.0);
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    EXPECT(threw);
    {
        blfls::SmootherSpec s2;  // reference defaults: sigma 12 / 0.04, lambda 1024, pad 16
        s2.radius = 6;
        blfls::Image u2 = blfls::smooth(c, s2);
        double m2 = 0.0;
        for (std::size_t i = 0; i < u2.size(); ++i) m2 = std::fmax(m2, std::fabs(u2.data()[i] - 0.55));
        EXPECT(m2 < 1e-6);  // constants are fixed points with padding too
    }
    threw = false;
    try {
        blfls::Image nanimg(16, 16, 1, 0.5);
        nanimg.at(0, 3, 3) = std::nan("");
        blfls::blf_ls(nanimg, nullptr, 10.0, 1.0, 0.1, 1, 2);
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    EXPECT(threw);
    {
        // NC_LS keeps constants (test_pipelines.cpp:33-38) and rolling keeps them too
        // (test_pipelines.cpp:113-118); bad DtParams / RollingParams throw
        blfls::SmootherSpec s3;
        s3.kind = blfls::SmootherKind::NC_LS;
        s3.dt = {6.0, 0.05, 3};
        blfls::Image u3 = blfls::smooth(c, s3);
        double m3 = 0.0;
        for (std::size_t i = 0; i < u3.size(); ++i) m3 = std::fmax(m3, std::fabs(u3.data()[i] - 0.55));
        EXPECT(m3 < 1e-6);
        blfls::Image cst(24, 24, 1, 0.8);
        blfls::Image r3 = blfls::rolling_nc_ls(cst, {8.0, 0.02, 3}, {}, {2, 2.5});
        double m4 = 0.0;
        for (std::size_t i = 0; i < r3.size(); ++i) m4 = std::fmax(m4, std::fabs(r3.data()[i] - 0.8));
        EXPECT(m4 < 1e-6);
        bool t1 = false, t2 = false;
        try {
            blfls::rolling_nc_ls(cst, {8.0, 0.02, 3}, {}, {0, 2.5});
        } catch (const std::invalid_argument&) {
            t1 = true;
        }
        try {
            blfls::gaussian_blur(cst, -1.0);
        } catch (const std::invalid_argument&) {
            t2 = true;
        }
        EXPECT(t1);
        EXPECT(t2);
    }
    {
        // blf_brute: constants are fixed points; a guide of the wrong shape throws
        blfls::Image cst(20, 12, 3, 0.25), gd(20, 12, 1, 0.5), bad(21, 12, 1, 0.5);
        blfls::Image f = blfls::blf_brute(cst, gd, {2.0, 0.1});
        double m5 = 0.0;
        for (std::size_t i = 0; i < f.size(); ++i) m5 = std::fmax(m5, std::fabs(f.data()[i] - 0.25));
        EXPECT(m5 < 1e-6);
        bool t3 = false;
        try {
            blfls::blf_brute(cst, bad, {2.0, 0.1});
        } catch (const std::invalid_argument&) {
            t3 = true;
        }
        EXPECT(t3);
    }
    if (fails == 0) std::printf("OK\n");
    return fails == 0 ? 0 : 1;
}
