/*
 * blfls_oracle.h -- CPU restatement of the reference BLF-LS hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_1812_07122_b200/,
 * include/, the CUDA library) links, loads or calls this code.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * use it, and only as the checker or the timed CPU baseline.
 *
 * Every function restates a function of the reference (paths relative to
 * /root/reference/proj) in plain C, double precision, OpenMP over rows like
 * the reference.  Layout is the reference's PlanarImage: C planes of H x W
 * doubles, row-major within each plane (include/epls/image.hpp:9-41).
 *
 * Parity pin: tests/test_oracle_pin.py checks this restatement against the
 * reference translation units compiled unmodified into oracle/_ref
 * (oracle/Makefile) and against the committed golden vectors in tests/golden/
 * that were produced from those units (tests/golden/make_golden.py).
 */
#ifndef BLFLS_ORACLE_H
#define BLFLS_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes mirror the C-ABI (include/blfls/blfls.h) */
#define ORC_OK 0
#define ORC_EINVAL 1
#define ORC_ENONFINITE 2
#define ORC_ENOMEM 4

/* complex numbers as interleaved (re, im) doubles */

/* Unnormalised 1-D DFT, out[k] = sum_j in[j] exp(sign*2*pi*i*j*k/n).  Any n >= 1
 * (mixed radix, generic odd radix for other primes). */
int orc_fft1d(int n, const double* in, double* out, int sign);

/* O(n^2) 2-D DFT of a real h x w plane, full spectrum h x w (test_solver.cpp:25-42). */
void orc_naive_dft2(const double* img, int h, int w, double* spec);

/* FFTW-convention half-spectrum r2c: h x (w/2+1) complex (src/fft2d.cpp:17-34). */
int orc_rfft2(const double* x, int h, int w, double* spec);
/* c2r with 1/(h*w) scaling; spec is clobbered (src/fft2d.cpp:36-52). */
int orc_irfft2(double* spec, int h, int w, double* out);

/* image.cpp:46-60; returns ORC_ENONFINITE on NaN/Inf. */
int orc_normalize_to_unit(const double* img, size_t n, double* out, double* lo, double* hi);
/* image.cpp:62-70 */
int orc_denormalize(const double* img, size_t n, double lo, double hi, double* out);
/* image.cpp:72-95, circular forward differences, per channel */
void orc_forward_gradients(const double* img, int c, int h, int w, double* gx, double* gy);
/* image.cpp:185-191 */
int orc_reflect_index(int q, int n);
/* image.cpp:193-212 / 214-230 */
int orc_reflect_pad(const double* img, int c, int h, int w, int pad, double* out);
int orc_crop_border(const double* img, int c, int h, int w, int pad, double* out);

/* bilateral.cpp:28-77 with an explicit window radius (the reference fixes
 * radius = ceil(3*sigma_s) at bilateral.cpp:37).  src has cs channels, guide
 * cg channels (1 or cs); range distance is the Euclidean norm over guide
 * channels.  radius < 0 means ceil(3*sigma_s). */
int orc_blf_brute_r(const double* src, int cs, const double* guide, int cg, int h, int w,
                    int radius, double sigma_s, double sigma_r, double* out);

/* solver.cpp:24-28 */
double orc_diff_gain_sq(int k, int n);
/* solver.cpp:88-124 (pad handled like the reference: reflect-pad g and targets, crop) */
int orc_lsgrad_solve_fft(const double* g, const double* tx, const double* ty, int c, int h, int w,
                         double lambda, int pad, double* u);
/* solver.cpp:67-86 */
int orc_ls_solve_fft(const double* g, int c, int h, int w, double lambda, int pad, double* u);
/* wls.cpp:78-130 restated with Gaussian elimination (Eigen is absent); tx/ty may be NULL.
 * Refuses planes beyond 4096 pixels like the reference (returns ORC_EINVAL). */
int orc_dense_solve(const double* g, const double* tx, const double* ty, int c, int h, int w,
                    double lambda, double* u);

/* pipelines.cpp:57-94 (BLF_LS branch) with blf_brute_r substituted for blf_grid
 * at pipelines.cpp:47.  guide is NULL (self-guided) or c channels like the
 * reference requires (pipelines.cpp:60-62). */
int orc_smooth_brute(const double* g, int c, int h, int w, const double* guide, int radius,
                     double sigma_s, double sigma_r, double lambda, int pad, double* out);

/* The north-star cascade: f <- smooth_brute(f) iters times, guide held fixed.
 * guide_c in {0 (none), 1, c}; a 1-channel guide for a c-channel image is
 * replicated into c channels (the reference rejects the mismatch). */
int orc_blf_ls(const double* g, int c, int h, int w, const double* guide, int guide_c, int radius,
               double sigma_s, double sigma_r, double lambda, int iters, double* out);
/* Same cascade with the reference's reflect padding (SolveParams::pad,
 * pipelines.cpp:76-92) in every smooth() call. */
int orc_blf_ls_pad(const double* g, int c, int h, int w, const double* guide, int guide_c,
                   int radius, double sigma_s, double sigma_r, double lambda, int iters, int pad,
                   double* out);

/* Per-stage split of one smooth_brute call (for the CPU baseline report):
 * returns seconds spent in the BLF stage and in the solve stage. */
int orc_blf_ls_timed(const double* g, int c, int h, int w, const double* guide, int guide_c,
                     int radius, double sigma_s, double sigma_r, double lambda, int iters,
                     double* out, double* t_blf, double* t_solve);

/* domain_transform.cpp:9-17 */
double orc_nc_box_radius(double sigma_s, int iter, int total);
/* domain_transform.cpp:21-156: normalized convolution over the domain
 * transform; guide has cg channels (L1 distance summed over them). */
int orc_nc_filter(const double* src, int cs, const double* guide, int cg, int h, int w,
                  double sigma_s, double sigma_r, int iters, double* out);
/* pipelines.cpp:57-94 with SmootherKind::NC_LS (nc_filter at pipelines.cpp:48);
 * guide NULL or c channels. */
int orc_smooth_nc(const double* g, int c, int h, int w, const double* guide, double sigma_s,
                  double sigma_r, int dt_iters, double lambda, int pad, double* out);
/* NC-LS cascade (iters smooth_nc calls, guide fixed, 1-channel guide replicated). */
int orc_nc_ls(const double* g, int c, int h, int w, const double* guide, int guide_c,
              double sigma_s, double sigma_r, int dt_iters, double lambda, int iters, int pad,
              double* out);
/* image.cpp:99-158 */
int orc_gaussian_blur(const double* img, int c, int h, int w, double sigma, double* out);
/* pipelines.cpp:96-117 */
int orc_rolling_nc_ls(const double* g, int c, int h, int w, double sigma_s, double sigma_r,
                      int dt_iters, double lambda, int pad, int n, double init_sigma, double* out);

/* SplitMix64 draw j (0-based) of the stream seeded with `seed`
 * (testimage.cpp:11-21: state += gamma, then mix). */
uint64_t orc_splitmix64_at(uint64_t seed, uint64_t j);
double orc_uniform_at(uint64_t seed, uint64_t j);

/* BASELINE.json synthetic generator (not in the reference).
 * One plane h x w from one seed: K Voronoi sites (levels U[0,1]) + ramp of
 * amplitude 0.2 + N(0, noise_sigma^2) + optional salt-and-pepper (p_sp total),
 * clipped to [0,1], rounded to float. */
void orc_gen_plane(uint64_t seed, int h, int w, int n_sites, double noise_sigma, double p_sp,
                   float* out);

int orc_num_threads(void);

#ifdef __cplusplus
}
#endif
#endif
