// C++ host API test (include/blfls/blfls.hpp over libblfls.so).
// Built by tests/test_cpp_host.py and linked against the CPU oracle
// (oracle/liboracle.so, test infrastructure only) as the checker.  On a GPU
// box it checks:
//  - blf_ls / smooth / flash_no_flash / lsgrad_solve_fft against the oracle
//    (the reference's algorithm in double) within the 1e-4 north-star gate;
//  - blfls::Plan reuse (Image and float interfaces, async calls) and the
//    per-thread plan cache give identical results on repeated calls;
//  - blfls::MultiPlan over the device list {0, 0}: batch shards and row
//    bands are bit-identical to one blfls_run on one device;
//  - the reference-style semantics: constants are fixed points, lambda 0 is
//    the identity, bad shapes / non-finite input throw std::invalid_argument.
// Prints "OK" and exits 0 on success.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <vector>

#include "blfls/blfls.hpp"

extern "C" {
int orc_blf_ls(const double* g, int c, int h, int w, const double* guide, int guide_c, int radius,
               double sigma_s, double sigma_r, double lambda, int iters, double* out);
int orc_lsgrad_solve_fft(const double* g, const double* tx, const double* ty, int c, int h, int w,
                         double lambda, int pad, double* u);
void orc_gen_plane(uint64_t seed, int h, int w, int n_sites, double noise_sigma, double p_sp, float* out);
}

static int fails = 0;
#define EXPECT(cond)                                             \
    do {                                                         \
        if (!(cond)) {                                           \
            std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #cond); \
            ++fails;                                             \
        }                                                        \
    } while (0)

static blfls::Image gen_image(int w, int h, int c, uint64_t seed)
{
    blfls::Image img(w, h, c);
    std::vector<float> plane((size_t)w * h);
    for (int k = 0; k < c; ++k) {
        orc_gen_plane(seed + k, h, w, 12, 0.03, 0.0, plane.data());
        for (size_t i = 0; i < plane.size(); ++i) img.data()[k * plane.size() + i] = plane[i];
    }
    return img;
}

static double max_abs(const std::vector<double>& a, const std::vector<double>& b)
{
    double m = 0.0;
    for (size_t i = 0; i < a.size(); ++i) m = std::fmax(m, std::fabs(a[i] - b[i]));
    return m;
}

static void oracle_checks()
{
    // self-guided RGB, joint gray guide, 3 iterations (a shrunken c2 / c5)
    const int w = 72, h = 40, r = 7;
    blfls::Image img = gen_image(w, h, 3, 4100), gd = gen_image(w, h, 1, 4200);
    std::vector<double> ref(img.size());
    orc_blf_ls(img.data().data(), 3, h, w, nullptr, 0, r, 7.0, 0.1, 1000.0, 3, ref.data());
    blfls::Image u = blfls::blf_ls(img, nullptr, 1000.0, 7.0, 0.1, 3, r);
    EXPECT(max_abs(u.data(), ref) <= 1e-4);
    orc_blf_ls(img.data().data(), 3, h, w, gd.data().data(), 1, r, 7.0, 0.1, 1000.0, 3, ref.data());
    blfls::Image uj = blfls::blf_ls(img, &gd, 1000.0, 7.0, 0.1, 3, r);
    EXPECT(max_abs(uj.data(), ref) <= 1e-4);
    // smooth() (one iteration, pad 0) and flash_no_flash with an RGB guide
    blfls::Image gd3 = gen_image(w, h, 3, 4300);
    blfls::SmootherSpec spec;
    spec.blf = {5.0, 0.05};
    spec.solve = {500.0, 0};
    spec.radius = 5;
    orc_blf_ls(img.data().data(), 3, h, w, gd3.data().data(), 3, 5, 5.0, 0.05, 500.0, 1, ref.data());
    blfls::Image f = blfls::flash_no_flash(img, gd3, spec);
    EXPECT(max_abs(f.data(), ref) <= 1e-4);
    // the solve stage
    blfls::Image tx = gen_image(w, h, 3, 4400), ty = gen_image(w, h, 3, 4500);
    for (double& v : tx.data()) v -= 0.5;
    for (double& v : ty.data()) v -= 0.5;
    orc_lsgrad_solve_fft(img.data().data(), tx.data().data(), ty.data().data(), 3, h, w, 100.0, 0, ref.data());
    blfls::Image s1 = blfls::lsgrad_solve_fft(img, tx, ty, 100.0);
    EXPECT(max_abs(s1.data(), ref) <= 1e-4);

    // Plan reuse: the Image interface twice, the cached free function, and
    // async float calls give the same bits
    blfls::Plan plan(h, w, 3, 1, r, 7.0, 0.1, 1000.0, 4, 0);
    blfls::Image p1 = plan.run(img, &gd, 3), p2 = plan.run(img, &gd, 3);
    EXPECT(max_abs(p1.data(), uj.data()) == 0.0);
    EXPECT(max_abs(p2.data(), uj.data()) == 0.0);
    const size_t ni = img.size(), ng = gd.size();
    std::vector<float> in(4 * ni), g(4 * ng), out(4 * ni), out2(4 * ni);
    for (int b = 0; b < 4; ++b) {
        blfls::Image ib = gen_image(w, h, 3, 5000 + 10 * b), gb = gen_image(w, h, 1, 5500 + b);
        for (size_t i = 0; i < ni; ++i) in[b * ni + i] = (float)ib.data()[i];
        for (size_t i = 0; i < ng; ++i) g[b * ng + i] = (float)gb.data()[i];
    }
    plan.run(in.data(), g.data(), 4, 3, out.data());
    plan.run_async(in.data(), g.data(), 4, 3, out2.data());
    plan.sync();
    bool same = true;
    for (size_t i = 0; i < out.size(); ++i) same = same && out[i] == out2[i];
    EXPECT(same);

    // MultiPlan over {0, 0}: batch shards == one blfls_run
    blfls_params prm = plan.params();
    {
        blfls::MultiPlan mp(prm, {0, 0}, BLFLS_MULTI_BATCH);
        std::vector<float> mo(4 * ni, -1.f);
        mp.run(in.data(), g.data(), 4, 3, mo.data());
        bool eq = true;
        for (size_t i = 0; i < mo.size(); ++i) eq = eq && mo[i] == out[i];
        EXPECT(eq);
        std::vector<float> m3(3 * ni, -1.f);  // an odd batch: shards of 2 and 1
        mp.run(in.data(), g.data(), 3, 3, m3.data());
        eq = true;
        for (size_t i = 0; i < m3.size(); ++i) eq = eq && m3[i] == out[i];
        EXPECT(eq);
    }
    // MultiPlan row bands ({0, 0}, {0, 0, 0}): one large-window gray image
    {
        const int bw = 128, bh = 96;
        blfls::Image big = gen_image(bw, bh, 1, 6100);
        blfls_params bp = blfls::detail::make_params(bh, bw, 1, 0, 15, 12.0, 0.08, 2000.0, 1, 0);
        blfls::Plan one(bp);
        std::vector<float> bi(big.size()), bo(big.size()), bm(big.size());
        for (size_t i = 0; i < bi.size(); ++i) bi[i] = (float)big.data()[i];
        one.run(bi.data(), nullptr, 1, 2, bo.data());
        for (int nb : {2, 3}) {
            std::vector<int> devs(nb, 0);
            blfls::MultiPlan band(bp, devs, BLFLS_MULTI_BAND);
            band.run(bi.data(), nullptr, 1, 2, bm.data());
            double m = 0.0;
            for (size_t i = 0; i < bm.size(); ++i) m = std::fmax(m, std::fabs((double)bm[i] - bo[i]));
            std::printf("band x%d vs one device: max-abs %.3g\n", nb, m);
            EXPECT(m == 0.0);
        }
        std::vector<double> bref(big.size());
        orc_blf_ls(big.data().data(), 1, bh, bw, nullptr, 0, 15, 12.0, 0.08, 2000.0, 2, bref.data());
        double m = 0.0;
        for (size_t i = 0; i < bm.size(); ++i) m = std::fmax(m, std::fabs(bm[i] - bref[i]));
        EXPECT(m <= 1e-4);
    }
}

int main()
{
    oracle_checks();
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
