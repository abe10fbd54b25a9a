/*
 * blfls_oracle.c -- CPU restatement of the reference BLF-LS hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see blfls_oracle.h).  Double precision, OpenMP
 * over rows, following the reference functions cited at each definition
 * (paths relative to /root/reference/proj).  The reference's FFT backend is
 * FFTW3 (CMakeLists.txt:14-15, unpinned, absent here); the restated FFT below
 * keeps FFTW's conventions (forward exp(-i), h x (w/2+1) half spectrum, c2r
 * scaled by 1/(h*w) as fft2d.cpp:49-51 does) and is pinned by the naive DFT
 * and the dense normal-equations solve exactly like test_solver.cpp:81-161.
 */
#include "blfls_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_PI 3.14159265358979323846264338327950288

int orc_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

static double now_s(void)
{
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* ------------------------------------------------------------------ FFT -- */

static int smallest_factor(int n)
{
    if (n % 4 == 0) return 4;
    if (n % 2 == 0) return 2;
    for (int p = 3; p * p <= n; p += 2)
        if (n % p == 0) return p;
    return n;
}

/* Recursive decimation-in-time mixed radix with a generic radix-p combine.
 * tw[j] = exp(sign*2*pi*i*j/N0) for the top-level length N0; a sub-transform
 * of length n uses twiddle stride N0/n. */
static void fft_rec2(int n, const double* in, int istride, double* out, const double* tw, int N0)
{
    if (n == 1) {
        out[0] = in[0];
        out[1] = in[1];
        return;
    }
    const int p = smallest_factor(n);
    const int m = n / p;
    double* sub = (double*)malloc(sizeof(double) * 2 * (size_t)n);
    for (int r = 0; r < p; ++r)
        fft_rec2(m, in + 2 * (size_t)r * istride, istride * p, sub + 2 * (size_t)r * m, tw, N0);
    const int tstep = N0 / n;
    for (int k = 0; k < m; ++k)
        for (int t = 0; t < p; ++t) {
            const int kk = k + t * m;
            double re = 0.0, im = 0.0;
            for (int r = 0; r < p; ++r) {
                const double* a = sub + 2 * ((size_t)r * m + k);
                const size_t ti = ((size_t)r * (size_t)kk % (size_t)n) * (size_t)tstep;
                const double wr = tw[2 * ti], wi = tw[2 * ti + 1];
                re += a[0] * wr - a[1] * wi;
                im += a[0] * wi + a[1] * wr;
            }
            out[2 * (size_t)kk] = re;
            out[2 * (size_t)kk + 1] = im;
        }
    free(sub);
}

static double* make_twiddles(int n, int sign)
{
    double* tw = (double*)malloc(sizeof(double) * 2 * (size_t)n);
    for (int j = 0; j < n; ++j) {
        const double a = sign * 2.0 * ORC_PI * (double)j / (double)n;
        tw[2 * j] = cos(a);
        tw[2 * j + 1] = sin(a);
    }
    return tw;
}

int orc_fft1d(int n, const double* in, double* out, int sign)
{
    if (n < 1) return ORC_EINVAL;
    double* tw = make_twiddles(n, sign < 0 ? -1 : 1);
    fft_rec2(n, in, 1, out, tw, n);
    free(tw);
    return ORC_OK;
}

/* strided batch helper: transform `count` sequences of length n */
static void fft_many(int n, int count, double* data, size_t seq_stride, size_t elem_stride,
                     const double* tw)
{
#pragma omp parallel
    {
        double* a = (double*)malloc(sizeof(double) * 2 * (size_t)n);
        double* b = (double*)malloc(sizeof(double) * 2 * (size_t)n);
#pragma omp for schedule(static)
        for (int s = 0; s < count; ++s) {
            double* base = data + 2 * (size_t)s * seq_stride;
            for (int j = 0; j < n; ++j) {
                a[2 * j] = base[2 * (size_t)j * elem_stride];
                a[2 * j + 1] = base[2 * (size_t)j * elem_stride + 1];
            }
            fft_rec2(n, a, 1, b, tw, n);
            for (int j = 0; j < n; ++j) {
                base[2 * (size_t)j * elem_stride] = b[2 * j];
                base[2 * (size_t)j * elem_stride + 1] = b[2 * j + 1];
            }
        }
        free(a);
        free(b);
    }
}

void orc_naive_dft2(const double* img, int h, int w, double* spec)
{
    /* test_solver.cpp:25-42 */
    for (int u = 0; u < h; ++u)
        for (int v = 0; v < w; ++v) {
            double re = 0.0, im = 0.0;
            for (int y = 0; y < h; ++y)
                for (int x = 0; x < w; ++x) {
                    const double ang = -2.0 * ORC_PI * ((double)u * y / h + (double)v * x / w);
                    re += img[(size_t)y * w + x] * cos(ang);
                    im += img[(size_t)y * w + x] * sin(ang);
                }
            spec[2 * ((size_t)u * w + v)] = re;
            spec[2 * ((size_t)u * w + v) + 1] = im;
        }
}

int orc_rfft2(const double* x, int h, int w, double* spec)
{
    /* fft2d.cpp:17-34: r2c 2-D, output h x (w/2+1), forward exp(-i) */
    if (h < 1 || w < 1) return ORC_EINVAL;
    const int wc = w / 2 + 1;
    double* rowbuf = (double*)malloc(sizeof(double) * 2 * (size_t)h * w);
    for (size_t i = 0; i < (size_t)h * w; ++i) {
        rowbuf[2 * i] = x[i];
        rowbuf[2 * i + 1] = 0.0;
    }
    double* twr = make_twiddles(w, -1);
    fft_many(w, h, rowbuf, (size_t)w, 1, twr);
    free(twr);
    for (int y = 0; y < h; ++y)
        for (int v = 0; v < wc; ++v) {
            spec[2 * ((size_t)y * wc + v)] = rowbuf[2 * ((size_t)y * w + v)];
            spec[2 * ((size_t)y * wc + v) + 1] = rowbuf[2 * ((size_t)y * w + v) + 1];
        }
    free(rowbuf);
    double* twc = make_twiddles(h, -1);
    fft_many(h, wc, spec, 1, (size_t)wc, twc);
    free(twc);
    return ORC_OK;
}

int orc_irfft2(double* spec, int h, int w, double* out)
{
    /* fft2d.cpp:36-52: c2r 2-D then scale by 1/(h*w) */
    if (h < 1 || w < 1) return ORC_EINVAL;
    const int wc = w / 2 + 1;
    double* twc = make_twiddles(h, +1);
    fft_many(h, wc, spec, 1, (size_t)wc, twc);
    free(twc);
    double* twr = make_twiddles(w, +1);
    const double scale = 1.0 / ((double)h * (double)w);
#pragma omp parallel
    {
        double* a = (double*)malloc(sizeof(double) * 2 * (size_t)w);
        double* b = (double*)malloc(sizeof(double) * 2 * (size_t)w);
#pragma omp for schedule(static)
        for (int y = 0; y < h; ++y) {
            const double* s = spec + 2 * (size_t)y * wc;
            /* Hermitian completion; the imaginary parts of DC and (even w)
             * Nyquist are ignored, as a c2r transform does. */
            for (int v = 0; v < w; ++v) {
                if (v < wc) {
                    a[2 * v] = s[2 * v];
                    a[2 * v + 1] = s[2 * v + 1];
                } else {
                    a[2 * v] = s[2 * (w - v)];
                    a[2 * v + 1] = -s[2 * (w - v) + 1];
                }
            }
            a[1] = 0.0;
            if (w % 2 == 0) a[2 * (w / 2) + 1] = 0.0;
            fft_rec2(w, a, 1, b, twr, w);
            for (int x = 0; x < w; ++x) out[(size_t)y * w + x] = b[2 * x] * scale;
        }
        free(a);
        free(b);
    }
    free(twr);
    return ORC_OK;
}

/* ---------------------------------------------------------- image.cpp -- */

int orc_normalize_to_unit(const double* img, size_t n, double* out, double* lo_out, double* hi_out)
{
    /* image.cpp:46-60 */
    for (size_t i = 0; i < n; ++i)
        if (!isfinite(img[i])) return ORC_ENONFINITE;
    double lo = img[0], hi = img[0];
    for (size_t i = 1; i < n; ++i) {
        if (img[i] < lo) lo = img[i];
        if (img[i] > hi) hi = img[i];
    }
    if (hi <= lo) {
        for (size_t i = 0; i < n; ++i) out[i] = 0.0;
        *lo_out = lo;
        *hi_out = lo + 1.0;
        return ORC_OK;
    }
    const double scale = 1.0 / (hi - lo);
    for (size_t i = 0; i < n; ++i) out[i] = (img[i] - lo) * scale;
    *lo_out = lo;
    *hi_out = hi;
    return ORC_OK;
}

int orc_denormalize(const double* img, size_t n, double lo, double hi, double* out)
{
    /* image.cpp:62-70 */
    if (!(hi > lo)) return ORC_EINVAL;
    const double range = hi - lo;
    for (size_t i = 0; i < n; ++i) out[i] = lo + img[i] * range;
    return ORC_OK;
}

void orc_forward_gradients(const double* img, int c, int h, int w, double* gx, double* gy)
{
    /* image.cpp:72-95 */
    for (int ch = 0; ch < c; ++ch) {
        const double* src = img + (size_t)ch * h * w;
        double* px = gx + (size_t)ch * h * w;
        double* py = gy + (size_t)ch * h * w;
#pragma omp parallel for schedule(static)
        for (int y = 0; y < h; ++y) {
            const int yn = (y + 1 == h) ? 0 : y + 1;
            for (int x = 0; x < w; ++x) {
                const int xn = (x + 1 == w) ? 0 : x + 1;
                px[(size_t)y * w + x] = src[(size_t)y * w + xn] - src[(size_t)y * w + x];
                py[(size_t)y * w + x] = src[(size_t)yn * w + x] - src[(size_t)y * w + x];
            }
        }
    }
}

int orc_reflect_index(int q, int n)
{
    /* image.cpp:185-191 */
    if (n == 1) return 0;
    const int period = 2 * (n - 1);
    q = abs(q) % period;
    return q < n ? q : period - q;
}

int orc_reflect_pad(const double* img, int c, int h, int w, int pad, double* out)
{
    /* image.cpp:193-212 */
    if (pad < 0) return ORC_EINVAL;
    const int hp = h + 2 * pad, wp = w + 2 * pad;
    for (int ch = 0; ch < c; ++ch) {
        const double* src = img + (size_t)ch * h * w;
        double* dst = out + (size_t)ch * hp * wp;
        for (int y = 0; y < hp; ++y) {
            const int sy = orc_reflect_index(y - pad, h);
            for (int x = 0; x < wp; ++x)
                dst[(size_t)y * wp + x] = src[(size_t)sy * w + orc_reflect_index(x - pad, w)];
        }
    }
    return ORC_OK;
}

int orc_crop_border(const double* img, int c, int h, int w, int pad, double* out)
{
    /* image.cpp:214-230; h, w are the padded dims */
    if (pad < 0 || w <= 2 * pad || h <= 2 * pad) return pad == 0 ? ORC_OK : ORC_EINVAL;
    const int ho = h - 2 * pad, wo = w - 2 * pad;
    for (int ch = 0; ch < c; ++ch)
        for (int y = 0; y < ho; ++y)
            memcpy(out + (size_t)ch * ho * wo + (size_t)y * wo,
                   img + (size_t)ch * h * w + (size_t)(y + pad) * w + pad, sizeof(double) * wo);
    return ORC_OK;
}

/* ------------------------------------------------------ bilateral.cpp -- */

int orc_blf_brute_r(const double* src, int cs, const double* guide, int cg, int h, int w,
                    int radius, double sigma_s, double sigma_r, double* out)
{
    /* bilateral.cpp:12-24 validation */
    if (!(sigma_s > 0.0) || !isfinite(sigma_s) || !(sigma_r > 0.0) || !isfinite(sigma_r))
        return ORC_EINVAL;
    if (cg != 1 && cg != cs) return ORC_EINVAL;
    const size_t plane = (size_t)h * w;
    for (size_t i = 0; i < plane * cs; ++i)
        if (!isfinite(src[i])) return ORC_ENONFINITE;
    for (size_t i = 0; i < plane * cg; ++i)
        if (!isfinite(guide[i])) return ORC_ENONFINITE;
    /* bilateral.cpp:37 fixes radius = ceil(3 sigma_s); explicit here */
    if (radius < 0) radius = (int)ceil(3.0 * sigma_s);
    const double inv2ss = 1.0 / (2.0 * sigma_s * sigma_s);
    const double inv2sr = 1.0 / (2.0 * sigma_r * sigma_r);
    const int kd = 2 * radius + 1;
    /* bilateral.cpp:41-47 spatial table */
    double* spatial = (double*)malloc(sizeof(double) * (size_t)kd * kd);
    for (int dy = -radius; dy <= radius; ++dy)
        for (int dx = -radius; dx <= radius; ++dx)
            spatial[(size_t)(dy + radius) * kd + (dx + radius)] =
                exp(-((double)dx * dx + (double)dy * dy) * inv2ss);
    /* bilateral.cpp:49-75 */
#pragma omp parallel for schedule(static)
    for (int y = 0; y < h; ++y) {
        double num[3];
        for (int x = 0; x < w; ++x) {
            for (int c = 0; c < cs; ++c) num[c] = 0.0;
            double z = 0.0;
            const int y0 = y - radius > 0 ? y - radius : 0;
            const int y1 = y + radius < h - 1 ? y + radius : h - 1;
            const int x0 = x - radius > 0 ? x - radius : 0;
            const int x1 = x + radius < w - 1 ? x + radius : w - 1;
            for (int ty = y0; ty <= y1; ++ty) {
                const double* srow = spatial + (size_t)(ty - y + radius) * kd + radius - x;
                for (int tx = x0; tx <= x1; ++tx) {
                    double d2 = 0.0;
                    for (int c = 0; c < cg; ++c) {
                        const double d = guide[c * plane + (size_t)y * w + x] -
                                         guide[c * plane + (size_t)ty * w + tx];
                        d2 += d * d;
                    }
                    const double wgt = srow[tx] * exp(-d2 * inv2sr);
                    z += wgt;
                    for (int c = 0; c < cs; ++c) num[c] += wgt * src[c * plane + (size_t)ty * w + tx];
                }
            }
            for (int c = 0; c < cs; ++c) out[c * plane + (size_t)y * w + x] = num[c] / z;
        }
    }
    free(spatial);
    return ORC_OK;
}

/* --------------------------------------------------------- solver.cpp -- */

double orc_diff_gain_sq(int k, int n)
{
    /* solver.cpp:24-28 */
    const double s = sin(ORC_PI * k / n);
    return 4.0 * s * s;
}

static int lsgrad_core(const double* g, const double* tx, const double* ty, int c, int h, int w,
                       double lambda, double* u)
{
    /* solver.cpp:100-122 at pad 0 */
    const int wc = w / 2 + 1;
    const size_t plane = (size_t)h * w;
    double* spec = (double*)malloc(sizeof(double) * 2 * (size_t)h * wc);
    double* sx = (double*)malloc(sizeof(double) * 2 * (size_t)h * wc);
    double* sy = (double*)malloc(sizeof(double) * 2 * (size_t)h * wc);
    if (!spec || !sx || !sy) {
        free(spec); free(sx); free(sy);
        return ORC_ENOMEM;
    }
    for (int ch = 0; ch < c; ++ch) {
        orc_rfft2(g + ch * plane, h, w, spec);
        if (tx) orc_rfft2(tx + ch * plane, h, w, sx);
        if (ty) orc_rfft2(ty + ch * plane, h, w, sy);
#pragma omp parallel for schedule(static)
        for (int uu = 0; uu < h; ++uu) {
            const double ay = -2.0 * ORC_PI * uu / h;
            const double oyr = cos(ay) - 1.0, oyi = sin(ay);
            const double gyv = orc_diff_gain_sq(uu, h);
            for (int v = 0; v < wc; ++v) {
                const double ax = -2.0 * ORC_PI * v / w;
                const double oxr = cos(ax) - 1.0, oxi = sin(ax);
                const size_t i = (size_t)uu * wc + v;
                const double den = 1.0 + lambda * (gyv + orc_diff_gain_sq(v, w));
                double nr = spec[2 * i], ni = spec[2 * i + 1];
                if (tx && ty) {
                    const double ar = oxr * sx[2 * i] - oxi * sx[2 * i + 1];
                    const double ai = oxr * sx[2 * i + 1] + oxi * sx[2 * i];
                    const double br = oyr * sy[2 * i] - oyi * sy[2 * i + 1];
                    const double bi = oyr * sy[2 * i + 1] + oyi * sy[2 * i];
                    nr += lambda * (ar + br);
                    ni += lambda * (ai + bi);
                }
                spec[2 * i] = nr / den;
                spec[2 * i + 1] = ni / den;
            }
        }
        orc_irfft2(spec, h, w, u + ch * plane);
    }
    free(spec); free(sx); free(sy);
    return ORC_OK;
}

static int all_finite(const double* a, size_t n)
{
    for (size_t i = 0; i < n; ++i)
        if (!isfinite(a[i])) return 0;
    return 1;
}

int orc_lsgrad_solve_fft(const double* g, const double* tx, const double* ty, int c, int h, int w,
                         double lambda, int pad, double* u)
{
    /* solver.cpp:15-21 validation, 88-124 */
    if (!(lambda >= 0.0) || !isfinite(lambda) || pad < 0) return ORC_EINVAL;
    const size_t n = (size_t)c * h * w;
    if (!all_finite(g, n)) return ORC_ENONFINITE;
    if (tx && !all_finite(tx, n)) return ORC_ENONFINITE;
    if (ty && !all_finite(ty, n)) return ORC_ENONFINITE;
    if (pad == 0) return lsgrad_core(g, tx, ty, c, h, w, lambda, u);
    const int hp = h + 2 * pad, wp = w + 2 * pad;
    const size_t np = (size_t)c * hp * wp;
    double* gp = (double*)malloc(sizeof(double) * np);
    double* txp = tx ? (double*)malloc(sizeof(double) * np) : NULL;
    double* typ = ty ? (double*)malloc(sizeof(double) * np) : NULL;
    double* up = (double*)malloc(sizeof(double) * np);
    orc_reflect_pad(g, c, h, w, pad, gp);
    if (tx) orc_reflect_pad(tx, c, h, w, pad, txp);
    if (ty) orc_reflect_pad(ty, c, h, w, pad, typ);
    int st = lsgrad_core(gp, txp, typ, c, hp, wp, lambda, up);
    if (st == ORC_OK) st = orc_crop_border(up, c, hp, wp, pad, u);
    free(gp); free(txp); free(typ); free(up);
    return st;
}

int orc_ls_solve_fft(const double* g, int c, int h, int w, double lambda, int pad, double* u)
{
    /* solver.cpp:67-86 == lsgrad with a zero target (test_solver.cpp:129-134) */
    return orc_lsgrad_solve_fft(g, NULL, NULL, c, h, w, lambda, pad, u);
}

int orc_dense_solve(const double* g, const double* tx, const double* ty, int c, int h, int w,
                    double lambda, double* u)
{
    /* wls.cpp:78-130: (I + lambda (Dx^T Dx + Dy^T Dy)) u = g + lambda (Dx^T tx + Dy^T ty),
     * circular differences (wls.cpp:78-99); Gaussian elimination with partial
     * pivoting replaces Eigen::PartialPivLU. */
    const int n = h * w;
    if (n > 4096) return ORC_EINVAL;
    if (!(lambda >= 0.0) || !isfinite(lambda)) return ORC_EINVAL;
    double* A = (double*)calloc((size_t)n * n, sizeof(double));
    double* b = (double*)malloc(sizeof(double) * n);
    if (!A || !b) {
        free(A); free(b);
        return ORC_ENOMEM;
    }
    /* D^T D for a forward difference D with rows e_i -> (-1 at i, +1 at j) */
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            const int i = y * w + x;
            const int je = y * w + (x + 1) % w;
            const int js = ((y + 1) % h) * w + x;
            const int jj[2] = {je, js};
            for (int a = 0; a < 2; ++a) {
                /* row of D: -e_i + e_j; D^T D += (e_j - e_i)(e_j - e_i)^T */
                const int j = jj[a];
                A[(size_t)i * n + i] += lambda;
                A[(size_t)j * n + j] += lambda;
                A[(size_t)i * n + j] -= lambda;
                A[(size_t)j * n + i] -= lambda;
            }
        }
    for (int i = 0; i < n; ++i) A[(size_t)i * n + i] += 1.0;
    /* LU with partial pivoting */
    int* piv = (int*)malloc(sizeof(int) * n);
    for (int k = 0; k < n; ++k) {
        int p = k;
        double best = fabs(A[(size_t)k * n + k]);
        for (int i = k + 1; i < n; ++i)
            if (fabs(A[(size_t)i * n + k]) > best) {
                best = fabs(A[(size_t)i * n + k]);
                p = i;
            }
        piv[k] = p;
        if (p != k)
            for (int j = 0; j < n; ++j) {
                const double t = A[(size_t)k * n + j];
                A[(size_t)k * n + j] = A[(size_t)p * n + j];
                A[(size_t)p * n + j] = t;
            }
        const double d = A[(size_t)k * n + k];
#pragma omp parallel for schedule(static)
        for (int i = k + 1; i < n; ++i) {
            const double f = A[(size_t)i * n + k] / d;
            A[(size_t)i * n + k] = f;
            if (f != 0.0)
                for (int j = k + 1; j < n; ++j) A[(size_t)i * n + j] -= f * A[(size_t)k * n + j];
        }
    }
    for (int ch = 0; ch < c; ++ch) {
        const double* gc = g + (size_t)ch * n;
        for (int i = 0; i < n; ++i) b[i] = gc[i];
        if (tx && ty) {
            const double* txc = tx + (size_t)ch * n;
            const double* tyc = ty + (size_t)ch * n;
            /* Dx^T t [i] = t[i - e] - t[i] (circular), same for y */
            for (int y = 0; y < h; ++y)
                for (int x = 0; x < w; ++x) {
                    const int i = y * w + x;
                    const int iw = y * w + (x - 1 + w) % w;
                    const int in = ((y - 1 + h) % h) * w + x;
                    b[i] += lambda * (txc[iw] - txc[i] + tyc[in] - tyc[i]);
                }
        }
        for (int k = 0; k < n; ++k)
            if (piv[k] != k) {
                const double t = b[k];
                b[k] = b[piv[k]];
                b[piv[k]] = t;
            }
        for (int i = 0; i < n; ++i) {
            double s = b[i];
            for (int j = 0; j < i; ++j) s -= A[(size_t)i * n + j] * b[j];
            b[i] = s;
        }
        for (int i = n - 1; i >= 0; --i) {
            double s = b[i];
            for (int j = i + 1; j < n; ++j) s -= A[(size_t)i * n + j] * b[j];
            b[i] = s / A[(size_t)i * n + i];
        }
        memcpy(u + (size_t)ch * n, b, sizeof(double) * n);
    }
    free(piv); free(A); free(b);
    return ORC_OK;
}

/* ------------------------------------------------------ pipelines.cpp -- */

/* gradient filter of smooth(): dt_iters == 0 -> brute-force BLF with `radius`
 * (north star, for blf_grid at pipelines.cpp:47); dt_iters > 0 -> nc_filter
 * with DtParams{sigma_s, sigma_r, dt_iters} (pipelines.cpp:48) */
static int smooth_core_k(const double* g, int c, int h, int w, const double* guide, int radius,
                         int dt_iters, double sigma_s, double sigma_r, double lambda, int pad,
                         double* out, double* t_blf, double* t_solve)
{
    const size_t n = (size_t)c * h * w;
    /* pipelines.cpp:59 */
    if (!all_finite(g, n)) return ORC_ENONFINITE;
    if (guide && !all_finite(guide, n)) return ORC_ENONFINITE;
    if (!(sigma_s > 0.0) || !isfinite(sigma_s) || !(sigma_r > 0.0) || !isfinite(sigma_r))
        return ORC_EINVAL;
    if (!(lambda >= 0.0) || !isfinite(lambda) || pad < 0) return ORC_EINVAL;
    const double t0 = now_s();
    /* pipelines.cpp:64 */
    double* gn = (double*)malloc(sizeof(double) * n);
    double lo, hi;
    orc_normalize_to_unit(g, n, gn, &lo, &hi);
    /* pipelines.cpp:76-78 */
    const int hp = h + 2 * pad, wp = w + 2 * pad;
    const size_t np = (size_t)c * hp * wp, pp = (size_t)hp * wp;
    double* gp = (double*)malloc(sizeof(double) * np);
    orc_reflect_pad(gn, c, h, w, pad, gp);
    double* gx = (double*)malloc(sizeof(double) * np);
    double* gy = (double*)malloc(sizeof(double) * np);
    orc_forward_gradients(gp, c, hp, wp, gx, gy);
    /* pipelines.cpp:81-87 */
    double* ggx = gx;
    double* ggy = gy;
    if (guide) {
        double* guide_n = (double*)malloc(sizeof(double) * n);
        double glo, ghi;
        orc_normalize_to_unit(guide, n, guide_n, &glo, &ghi);
        double* guide_p = (double*)malloc(sizeof(double) * np);
        orc_reflect_pad(guide_n, c, h, w, pad, guide_p);
        ggx = (double*)malloc(sizeof(double) * np);
        ggy = (double*)malloc(sizeof(double) * np);
        orc_forward_gradients(guide_p, c, hp, wp, ggx, ggy);
        free(guide_n);
        free(guide_p);
    }
    /* filter_gradients, pipelines.cpp:33-53 with blf_brute_r for blf_grid (47) */
    double* tx = (double*)malloc(sizeof(double) * np);
    double* ty = (double*)malloc(sizeof(double) * np);
    double* s01 = (double*)malloc(sizeof(double) * pp);
    double* g01 = (double*)malloc(sizeof(double) * pp);
    double* f01 = (double*)malloc(sizeof(double) * pp);
    for (int axis = 0; axis < 2; ++axis) {
        const double* src = axis == 0 ? gx : gy;
        const double* gd = axis == 0 ? ggx : ggy;
        double* dst = axis == 0 ? tx : ty;
        for (int ch = 0; ch < c; ++ch) {
            /* to_unit_range, pipelines.cpp:18-23 */
            for (size_t i = 0; i < pp; ++i) {
                s01[i] = (src[ch * pp + i] + 1.0) * 0.5;
                g01[i] = (gd[ch * pp + i] + 1.0) * 0.5;
            }
            if (dt_iters > 0)
                orc_nc_filter(s01, 1, g01, 1, hp, wp, sigma_s, sigma_r, dt_iters, f01);
            else
                orc_blf_brute_r(s01, 1, g01, 1, hp, wp, radius, sigma_s, sigma_r, f01);
            /* from_unit_range_into, pipelines.cpp:25-31 */
            for (size_t i = 0; i < pp; ++i) dst[ch * pp + i] = 2.0 * f01[i] - 1.0;
        }
    }
    const double t1 = now_s();
    /* pipelines.cpp:91-93 */
    double* up = (double*)malloc(sizeof(double) * np);
    int st = lsgrad_core(gp, tx, ty, c, hp, wp, lambda, up);
    double* uc = (double*)malloc(sizeof(double) * n);
    if (pad > 0)
        orc_crop_border(up, c, hp, wp, pad, uc);
    else
        memcpy(uc, up, sizeof(double) * n);
    orc_denormalize(uc, n, lo, hi, out);
    const double t2 = now_s();
    if (t_blf) *t_blf += t1 - t0;
    if (t_solve) *t_solve += t2 - t1;
    free(gn); free(gp); free(gx); free(gy);
    if (guide) {
        free(ggx);
        free(ggy);
    }
    free(tx); free(ty); free(s01); free(g01); free(f01); free(up); free(uc);
    return st;
}

static int smooth_core(const double* g, int c, int h, int w, const double* guide, int radius,
                       double sigma_s, double sigma_r, double lambda, int pad, double* out,
                       double* t_blf, double* t_solve)
{
    return smooth_core_k(g, c, h, w, guide, radius, 0, sigma_s, sigma_r, lambda, pad, out, t_blf,
                         t_solve);
}

int orc_smooth_brute(const double* g, int c, int h, int w, const double* guide, int radius,
                     double sigma_s, double sigma_r, double lambda, int pad, double* out)
{
    return smooth_core(g, c, h, w, guide, radius, sigma_s, sigma_r, lambda, pad, out, NULL, NULL);
}

static int cascade_core(const double* g, int c, int h, int w, const double* guide, int guide_c,
                        int radius, int dt_iters, double sigma_s, double sigma_r, double lambda,
                        int iters, int pad, double* out, double* t_blf, double* t_solve)
{
    if (c != 1 && c != 3) return ORC_EINVAL;
    if (h < 1 || w < 1 || iters < 1) return ORC_EINVAL;
    if (guide && guide_c != 1 && guide_c != c) return ORC_EINVAL;
    const size_t n = (size_t)c * h * w;
    double* guide_rep = NULL;
    if (guide) {
        guide_rep = (double*)malloc(sizeof(double) * n);
        for (int ch = 0; ch < c; ++ch)
            memcpy(guide_rep + (size_t)ch * h * w, guide + (size_t)(guide_c == 1 ? 0 : ch) * h * w,
                   sizeof(double) * (size_t)h * w);
    }
    double* f = (double*)malloc(sizeof(double) * n);
    memcpy(f, g, sizeof(double) * n);
    if (t_blf) *t_blf = 0.0;
    if (t_solve) *t_solve = 0.0;
    int st = ORC_OK;
    for (int k = 0; k < iters && st == ORC_OK; ++k) {
        st = smooth_core_k(f, c, h, w, guide_rep, radius, dt_iters, sigma_s, sigma_r, lambda, pad,
                           out, t_blf, t_solve);
        memcpy(f, out, sizeof(double) * n);
    }
    free(f);
    free(guide_rep);
    return st;
}

static int blf_ls_core(const double* g, int c, int h, int w, const double* guide, int guide_c,
                       int radius, double sigma_s, double sigma_r, double lambda, int iters, int pad,
                       double* out, double* t_blf, double* t_solve)
{
    return cascade_core(g, c, h, w, guide, guide_c, radius, 0, sigma_s, sigma_r, lambda, iters, pad,
                        out, t_blf, t_solve);
}

int orc_blf_ls_timed(const double* g, int c, int h, int w, const double* guide, int guide_c,
                     int radius, double sigma_s, double sigma_r, double lambda, int iters,
                     double* out, double* t_blf, double* t_solve)
{
    return blf_ls_core(g, c, h, w, guide, guide_c, radius, sigma_s, sigma_r, lambda, iters, 0, out,
                       t_blf, t_solve);
}

int orc_blf_ls(const double* g, int c, int h, int w, const double* guide, int guide_c, int radius,
               double sigma_s, double sigma_r, double lambda, int iters, double* out)
{
    return blf_ls_core(g, c, h, w, guide, guide_c, radius, sigma_s, sigma_r, lambda, iters, 0, out,
                       NULL, NULL);
}

int orc_blf_ls_pad(const double* g, int c, int h, int w, const double* guide, int guide_c,
                   int radius, double sigma_s, double sigma_r, double lambda, int iters, int pad,
                   double* out)
{
    if (pad < 0) return ORC_EINVAL;
    return blf_ls_core(g, c, h, w, guide, guide_c, radius, sigma_s, sigma_r, lambda, iters, pad, out,
                       NULL, NULL);
}

/* ------------------------------------------------- domain_transform.cpp -- */

double orc_nc_box_radius(double sigma_s, int iter, int total)
{
    /* domain_transform.cpp:9-17: per-pass Gaussian bandwidth, box of equal variance */
    const double sigma_i =
        sigma_s * sqrt(3.0) * pow(2.0, total - iter) / sqrt(pow(4.0, total) - 1.0);
    return sqrt(3.0) * sigma_i;
}

/* One scanline of n samples at stride `st`: normalized box over the warped
 * coordinates t (domain_transform.cpp:72-103 / 105-134).  The sliding bounds
 * and the prefix sums are evaluated in the reference's order. */
static void nc_box_line(double* v, size_t st, int n, const double* t, size_t tst, double radius,
                        double* prefix)
{
    prefix[0] = 0.0;
    for (int k = 0; k < n; ++k) prefix[k + 1] = prefix[k] + v[k * st];
    int lo = 0, hi = 0;
    for (int k = 0; k < n; ++k) {
        const double tk = t[k * tst];
        while (t[lo * tst] < tk - radius) ++lo;
        if (hi < k) hi = k;
        while (hi + 1 < n && t[(hi + 1) * tst] <= tk + radius) ++hi;
        const double inv = 1.0 / (hi - lo + 1);
        v[k * st] = (prefix[hi + 1] - prefix[lo]) * inv;
    }
}

int orc_nc_filter(const double* src, int cs, const double* guide, int cg, int h, int w,
                  double sigma_s, double sigma_r, int iters, double* out)
{
    /* domain_transform.cpp:21-29 (validate) */
    if (!(sigma_s > 0.0) || !(sigma_r > 0.0) || !isfinite(sigma_s) || !isfinite(sigma_r))
        return ORC_EINVAL;
    if (iters < 1 || h < 1 || w < 1 || cs < 1 || cg < 1) return ORC_EINVAL;
    const size_t pp = (size_t)h * w;
    if (!all_finite(src, cs * pp) || !all_finite(guide, cg * pp)) return ORC_ENONFINITE;
    const double ratio = sigma_s / sigma_r;
    /* transform_rows / transform_cols, domain_transform.cpp:31-68 */
    double* cth = (double*)malloc(sizeof(double) * pp);
    double* ctv = (double*)malloc(sizeof(double) * pp);
#pragma omp parallel for schedule(static)
    for (int y = 0; y < h; ++y) {
        double acc = 1.0;
        cth[(size_t)y * w] = acc;
        for (int x = 1; x < w; ++x) {
            double d = 0.0;
            for (int c = 0; c < cg; ++c)
                d += fabs(guide[c * pp + (size_t)y * w + x] - guide[c * pp + (size_t)y * w + x - 1]);
            acc += 1.0 + ratio * d;
            cth[(size_t)y * w + x] = acc;
        }
    }
#pragma omp parallel for schedule(static)
    for (int x = 0; x < w; ++x) {
        double acc = 1.0;
        ctv[x] = acc;
        for (int y = 1; y < h; ++y) {
            double d = 0.0;
            for (int c = 0; c < cg; ++c)
                d += fabs(guide[c * pp + (size_t)y * w + x] - guide[c * pp + (size_t)(y - 1) * w + x]);
            acc += 1.0 + ratio * d;
            ctv[(size_t)y * w + x] = acc;
        }
    }
    memcpy(out, src, sizeof(double) * cs * pp);
    /* nc_filter, domain_transform.cpp:138-156: rows then columns per pass */
    for (int it = 1; it <= iters; ++it) {
        const double radius = orc_nc_box_radius(sigma_s, it, iters);
#pragma omp parallel
        {
            double* prefix = (double*)malloc(sizeof(double) * ((h > w ? h : w) + 1));
#pragma omp for schedule(static)
            for (int y = 0; y < h; ++y)
                for (int c = 0; c < cs; ++c)
                    nc_box_line(out + c * pp + (size_t)y * w, 1, w, cth + (size_t)y * w, 1, radius,
                                prefix);
#pragma omp for schedule(static)
            for (int x = 0; x < w; ++x)
                for (int c = 0; c < cs; ++c)
                    nc_box_line(out + c * pp + x, (size_t)w, h, ctv + x, (size_t)w, radius, prefix);
            free(prefix);
        }
    }
    free(cth);
    free(ctv);
    return ORC_OK;
}

int orc_smooth_nc(const double* g, int c, int h, int w, const double* guide, double sigma_s,
                  double sigma_r, int dt_iters, double lambda, int pad, double* out)
{
    if (dt_iters < 1) return ORC_EINVAL;
    return smooth_core_k(g, c, h, w, guide, 0, dt_iters, sigma_s, sigma_r, lambda, pad, out, NULL,
                         NULL);
}

int orc_nc_ls(const double* g, int c, int h, int w, const double* guide, int guide_c,
              double sigma_s, double sigma_r, int dt_iters, double lambda, int iters, int pad,
              double* out)
{
    if (dt_iters < 1 || pad < 0) return ORC_EINVAL;
    return cascade_core(g, c, h, w, guide, guide_c, 0, dt_iters, sigma_s, sigma_r, lambda, iters,
                        pad, out, NULL, NULL);
}

/* image.cpp:99-158: separable Gaussian, radius ceil(3 sigma), clamped borders */
int orc_gaussian_blur(const double* img, int c, int h, int w, double sigma, double* out)
{
    if (!(sigma > 0.0) || !isfinite(sigma)) return ORC_EINVAL;
    const int r = (int)ceil(3.0 * sigma);
    double* k = (double*)malloc(sizeof(double) * (2 * r + 1));
    double sum = 0.0;
    for (int i = -r; i <= r; ++i) {
        k[i + r] = exp(-((double)i * i) / (2.0 * sigma * sigma));
        sum += k[i + r];
    }
    for (int i = 0; i <= 2 * r; ++i) k[i] /= sum;
    const size_t pp = (size_t)h * w;
    double* tmp = (double*)malloc(sizeof(double) * c * pp);
    for (int ch = 0; ch < c; ++ch) {
        const double* src = img + ch * pp;
        double* dst = tmp + ch * pp;
#pragma omp parallel for schedule(static)
        for (int y = 0; y < h; ++y)
            for (int x = 0; x < w; ++x) {
                double acc = 0.0;
                for (int i = -r; i <= r; ++i) {
                    int xi = x + i;
                    xi = xi < 0 ? 0 : (xi > w - 1 ? w - 1 : xi);
                    acc += k[i + r] * src[(size_t)y * w + xi];
                }
                dst[(size_t)y * w + x] = acc;
            }
    }
    for (int ch = 0; ch < c; ++ch) {
        const double* src = tmp + ch * pp;
        double* dst = out + ch * pp;
#pragma omp parallel for schedule(static)
        for (int y = 0; y < h; ++y)
            for (int x = 0; x < w; ++x) {
                double acc = 0.0;
                for (int i = -r; i <= r; ++i) {
                    int yi = y + i;
                    yi = yi < 0 ? 0 : (yi > h - 1 ? h - 1 : yi);
                    acc += k[i + r] * src[(size_t)yi * w + x];
                }
                dst[(size_t)y * w + x] = acc;
            }
    }
    free(tmp);
    free(k);
    return ORC_OK;
}

/* pipelines.cpp:96-117: guide <- blur(g); n times u <- smooth_nc(g, guide), guide <- u */
int orc_rolling_nc_ls(const double* g, int c, int h, int w, double sigma_s, double sigma_r,
                      int dt_iters, double lambda, int pad, int n, double init_sigma, double* out)
{
    if (n < 1 || !(init_sigma > 0.0)) return ORC_EINVAL;
    const size_t nn = (size_t)c * h * w;
    double* guide = (double*)malloc(sizeof(double) * nn);
    int st = orc_gaussian_blur(g, c, h, w, init_sigma, guide);
    for (int k = 0; k < n && st == ORC_OK; ++k) {
        st = orc_smooth_nc(g, c, h, w, guide, sigma_s, sigma_r, dt_iters, lambda, pad, out);
        memcpy(guide, out, sizeof(double) * nn);
    }
    free(guide);
    return st;
}

/* ------------------------------------------------------------ generator -- */

uint64_t orc_splitmix64_at(uint64_t seed, uint64_t j)
{
    /* testimage.cpp:14-20: state += gamma; mix.  Draw j sees state seed+(j+1)*gamma. */
    uint64_t z = seed + (j + 1) * 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

double orc_uniform_at(uint64_t seed, uint64_t j)
{
    /* testimage.cpp:21 */
    return (double)(orc_splitmix64_at(seed, j) >> 11) * 0x1.0p-53;
}

void orc_gen_plane(uint64_t seed, int h, int w, int n_sites, double noise_sigma, double p_sp,
                   float* out)
{
    double* sx = (double*)malloc(sizeof(double) * n_sites);
    double* sy = (double*)malloc(sizeof(double) * n_sites);
    double* lv = (double*)malloc(sizeof(double) * n_sites);
    for (int s = 0; s < n_sites; ++s) {
        sx[s] = orc_uniform_at(seed, 3 * (uint64_t)s) * w;
        sy[s] = orc_uniform_at(seed, 3 * (uint64_t)s + 1) * h;
        lv[s] = orc_uniform_at(seed, 3 * (uint64_t)s + 2);
    }
    const uint64_t base = 3 * (uint64_t)n_sites;
    const double rx = w > 1 ? 1.0 / (w - 1) : 0.0;
    const double ry = h > 1 ? 1.0 / (h - 1) : 0.0;
#pragma omp parallel for schedule(static)
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            int best = 0;
            double bd = 1e300;
            for (int s = 0; s < n_sites; ++s) {
                const double dx = x - sx[s], dy = y - sy[s];
                const double d = dx * dx + dy * dy;
                if (d < bd) {
                    bd = d;
                    best = s;
                }
            }
            const uint64_t i = (uint64_t)y * w + x;
            double v = lv[best] + 0.2 * ((x * rx + y * ry) * 0.5 - 0.5);
            const double u1 = orc_uniform_at(seed, base + 3 * i);
            const double u2 = orc_uniform_at(seed, base + 3 * i + 1);
            v += noise_sigma * sqrt(-2.0 * log(1.0 - u1)) * cos(2.0 * ORC_PI * u2);
            if (p_sp > 0.0) {
                const double u3 = orc_uniform_at(seed, base + 3 * i + 2);
                if (u3 < 0.5 * p_sp)
                    v = 0.0;
                else if (u3 < p_sp)
                    v = 1.0;
            }
            v = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
            out[i] = (float)v;
        }
    free(sx); free(sy); free(lv);
}
