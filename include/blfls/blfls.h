/*
 * blfls.h -- C ABI of the B200-native BLF-LS hot path (sm_100a CUDA).
 *
 * This is the drop-in boundary.  The reference (/root/reference/proj) is a C++
 * library with no FFI; its seams for this path are
 *
 *   PlanarImage epls::smooth(const PlanarImage&, const SmootherSpec&)
 *       include/epls/pipelines.hpp:36, src/pipelines.cpp:57-94  (BLF_LS branch)
 *   PlanarImage epls::flash_no_flash(noflash, flash, spec)   (joint variant)
 *       include/epls/applications.hpp:29, src/applications.cpp:58-64
 *   filter_gradients (pipelines.cpp:33-53) + blf_brute (bilateral.hpp:26)
 *   PlanarImage epls::lsgrad_solve_fft(g, target, SolveParams)
 *       include/epls/solver.hpp:43, src/solver.cpp:88-124
 *   epls::detail::rfft2 / irfft2   src/fft2d.hpp:11,14
 *
 * and each entry point below names the one it replaces.  Conventions:
 *  - images are planar fp32, [batch][channel][row][col] (the reference's
 *    PlanarImage layout, image.hpp:9-41, one image after another);
 *  - buffers are caller-owned; BLFLS_HOST_PTRS says they are host memory
 *    (copied in/out on `stream` inside the call), otherwise device memory;
 *  - no exception crosses the ABI: std::invalid_argument of the reference maps
 *    to BLFLS_EINVAL, non-finite input (image.cpp:21-27) to BLFLS_ENONFINITE;
 *    blfls_last_error() returns a thread-local message for the last failure;
 *  - a plan is not thread-safe (one per host thread / stream); plans on
 *    different devices run concurrently;
 *  - there is no CPU fallback: without a usable sm_100 device every entry
 *    point that computes returns BLFLS_ECUDA.
 */
#ifndef BLFLS_H
#define BLFLS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BLFLS_ABI_VERSION 3

typedef enum blfls_status {
    BLFLS_OK = 0,
    BLFLS_EINVAL = 1,        /* std::invalid_argument in the reference */
    BLFLS_ENONFINITE = 2,    /* require_finite, image.cpp:21-27 */
    BLFLS_ECUDA = 3,         /* CUDA runtime error / no device */
    BLFLS_ENOMEM = 4,        /* device allocation failed */
    BLFLS_EUNSUPPORTED = 5   /* size/radius outside the supported envelope */
} blfls_status;

/* flags */
#define BLFLS_DEVICE_PTRS 0u
#define BLFLS_HOST_PTRS 1u     /* img/guide/out are host pointers (pinned is fastest) */
#define BLFLS_CHECK_FINITE 2u  /* reject NaN/Inf input like require_finite (one sync) */
#define BLFLS_SYNC 4u          /* synchronize `stream` before returning */
#define BLFLS_NO_GRAPH 8u      /* launch kernels directly instead of a cached CUDA graph */
#define BLFLS_TIME_STAGES 16u  /* bracket every stage with CUDA events (implies NO_GRAPH);
                                  read the sums with blfls_stage_times */
#define BLFLS_ASYNC 32u        /* with HOST_PTRS: return without waiting; the copies run on
                                  their own streams through two staging slots, so
                                  consecutive calls overlap H2D / compute / D2H.  Inputs
                                  must stay valid and outputs are readable only after
                                  blfls_sync (which also reports deferred non-finite
                                  input when CHECK_FINITE is set).  With device pointers
                                  the call stays ordered on `stream`; only the
                                  CHECK_FINITE verdict is deferred to blfls_sync (the
                                  input is still scanned on the device in every call,
                                  without a host round trip). */

typedef struct blfls_plan_s* blfls_plan_t;

/* Everything a plan is specialised on.  Mirrors SmootherSpec
 * (pipelines.hpp:16-23) for kind == BLF_LS (backends BRUTE, GRID) and
 * kind == NC_LS (backend DT). */
typedef struct blfls_params {
    int height, width;    /* image size, >= 2 each */
    int channels;         /* 1 or 3 (image.cpp:16-17) */
    int guide_channels;   /* 0 = self-guided; 1 = one grayscale guide shared by all
                             channels; == channels = per-channel guide (smooth()
                             with SmootherSpec::guidance, pipelines.cpp:81-84) */
    int radius;           /* BLF window radius r; < 0 means ceil(3*sigma_s) as
                             bilateral.cpp:37 */
    double sigma_s;       /* RangeSpatialParams (bilateral.hpp:10-13), or DtParams
                             (domain_transform.hpp:7-11) for BLFLS_BACKEND_DT */
    double sigma_r;
    double lambda;        /* SolveParams::lambda (solver.hpp:12-15); pad is 0 */
    int max_batch;        /* images per call the plan's workspace is sized for */
    int device;           /* CUDA device ordinal */
    int pad;              /* SolveParams::pad: reflect padding before the gradients and
                             the FFT solve, cropped at the end (pipelines.cpp:76-92,
                             image.cpp:185-230); 0 = periodic boundary.  Besides
                             blfls_run, blfls_solve honours it; the other stage
                             entry points require pad == 0. */
    int backend;          /* gradient filter: BLFLS_BACKEND_BRUTE (0, the north star:
                             brute-force BLF over the (2r+1)^2 window) or
                             BLFLS_BACKEND_GRID (1, the bilateral grid blf_grid that
                             the reference's smooth() runs, bilateral.cpp:112-207,
                             grid sampling = (sigma_s, sigma_r); radius unused) or
                             BLFLS_BACKEND_DT (2, nc_filter: normalized convolution
                             over the domain transform, domain_transform.cpp:138-156,
                             i.e. SmootherKind::NC_LS, pipelines.cpp:48; radius unused) */
    int dt_iterations;    /* DtParams::iterations for BLFLS_BACKEND_DT: >= 1, 0 means
                             the reference default 3 (pipelines.hpp:19); ignored by
                             the other backends */
} blfls_params;

#define BLFLS_BACKEND_BRUTE 0
#define BLFLS_BACKEND_GRID 1
#define BLFLS_BACKEND_DT 2

/* Validates like validate_params / validate_solve_params (bilateral.cpp:12-24,
 * solver.cpp:15-21) and caches twiddles, spectral denominators and workspaces. */
blfls_status blfls_plan_create(const blfls_params* params, blfls_plan_t* plan);
blfls_status blfls_plan_destroy(blfls_plan_t plan);

/* Full BLF-LS: `iters` cascaded smooth() calls (each one normalise -> circular
 * gradients -> brute-force (joint) BLF of each gradient field over the
 * (2r+1)^2 clipped window -> periodic FFT least-squares solve -> denormalise),
 * guide held fixed.  Replaces epls::smooth(g, spec) for kind == BLF_LS
 * (pipelines.cpp:57-94) with blf_brute in place of blf_grid, and
 * flash_no_flash (applications.cpp:58-64) when guide != NULL.
 * img/out: batch x C x H x W; guide: batch x guide_channels x H x W or NULL. */
blfls_status blfls_run(blfls_plan_t plan, const float* img, const float* guide, int batch,
                       int iters, float* out, void* stream, unsigned flags);

/* Wait for every call issued on the plan; returns BLFLS_ENONFINITE if an
 * ASYNC | CHECK_FINITE call since the previous sync saw NaN/Inf input. */
blfls_status blfls_sync(blfls_plan_t plan);

/* One iteration's gradient targets, as filter_gradients returns them
 * (pipelines.cpp:33-53): gradients of the [0,1]-normalised image, filtered by
 * the brute-force BLF.  tx/ty: batch x C x H x W. */
blfls_status blfls_filter_gradients(blfls_plan_t plan, const float* img, const float* guide,
                                    int batch, float* tx, float* ty, void* stream, unsigned flags);

/* Row-band form of blfls_filter_gradients for the multi-GPU band driver:
 * rows [y0, y1) of the targets of ONE image (batch index 0), written to
 * tx/ty as (y1-y0) x W planes per channel, in RAW image units (not
 * normalised; the solve consumes them directly).  The full image is read
 * (the window clips at the global top/bottom, gy wraps at y = H-1). */
blfls_status blfls_filter_gradients_rows(blfls_plan_t plan, const float* img, const float* guide,
                                         int y0, int y1, float* tx, float* ty, void* stream,
                                         unsigned flags);
/* Fused band exchange for multi-GPU row bands: as blfls_filter_gradients_rows,
 * but every target of rows [y0, y1) is stored at its global position in the
 * full-height (channels x H x W) tx / ty buffers of all `npeers` ranks (1..8,
 * NVLink peer-mapped device pointers, e.g. symmetric-memory buffers) by the
 * filter kernel itself, so no separate all-gather follows; the caller makes
 * the stores visible with a device barrier before the solve.  Brute-force
 * backend, pad 0, device pointers. */
blfls_status blfls_filter_gradients_rows_peers(blfls_plan_t plan, const float* img,
                                               const float* guide, int y0, int y1,
                                               float* const* tx_peers, float* const* ty_peers,
                                               int npeers, void* stream, unsigned flags);

/* lsgrad_solve_fft(g, {tx, ty}, {lambda, pad}) (solver.cpp:88-124) with the
 * plan's pad (image and targets reflect-padded as plain rasters, result
 * cropped); all arguments batch x C x H x W.  tx/ty may both be NULL
 * (ls_solve_fft, solver.cpp:67-86). */
blfls_status blfls_solve(blfls_plan_t plan, const float* g, const float* tx, const float* ty,
                         int batch, float* u, void* stream, unsigned flags);

/* detail::rfft2 (fft2d.cpp:17-34): x is batch*C planes of H x W; spec is
 * batch*C planes of H x (W/2+1) interleaved complex (re, im) fp32. */
blfls_status blfls_rfft2(blfls_plan_t plan, const float* x, int batch, float* spec, void* stream,
                         unsigned flags);
/* detail::irfft2 (fft2d.cpp:36-52) including the 1/(H*W) scaling. */
blfls_status blfls_irfft2(blfls_plan_t plan, const float* spec, int batch, float* out, void* stream,
                          unsigned flags);

/* Seeded synthetic planes of BASELINE.json (Voronoi levels + ramp + Gaussian
 * noise + optional salt-and-pepper, clipped to [0,1]); one seed per plane.
 * out: n_planes x H x W device memory. */
blfls_status blfls_generate(int height, int width, int n_planes, const uint64_t* seeds,
                            int n_sites, double noise_sigma, double p_salt_pepper, float* out,
                            void* stream, int device);

/* forward_gradients (image.cpp:72-95): circular forward differences of
 * `planes` planes, gx = f[y][(x+1) mod W] - f[y][x], gy = f[(y+1) mod H][x] -
 * f[y][x]; fp32, flags DEVICE_PTRS / HOST_PTRS and SYNC as for blfls_run. */
blfls_status blfls_forward_gradients(const float* img, int planes, int height, int width, float* gx,
                                     float* gy, int device, void* stream, unsigned flags);

/* blf_brute (bilateral.cpp:28-77): the standalone brute-force (joint)
 * bilateral filter of `batch` images of cs planes (1 or 3), guided by cg
 * planes (1 or cs; guide == NULL: guided by src itself, cg ignored).  Weights
 * exp(-|dxy|^2 / (2 sigma_s^2)) * exp(-|g(s) - g(t)|^2 / (2 sigma_r^2)) with the
 * Euclidean norm over the guide channels, window |dx|, |dy| <= radius clipped at
 * the border; radius < 0 means ceil(3 sigma_s) as the reference (bilateral.cpp:37).
 * fp32 in and out; flags DEVICE_PTRS / HOST_PTRS, CHECK_FINITE, SYNC as for
 * blfls_run.  BLFLS_EUNSUPPORTED when the tile (radius) exceeds shared memory. */
blfls_status blfls_blf_brute(const float* src, int cs, const float* guide, int cg, int height,
                             int width, int batch, int radius, double sigma_s, double sigma_r,
                             float* out, int device, void* stream, unsigned flags);

/* gaussian_blur (image.cpp:99-158): separable Gaussian of radius ceil(3 sigma),
 * weights exp(-i^2 / (2 sigma^2)) normalised to sum 1, clamped borders,
 * accumulated in double in the reference's tap order; `in` and `out` are
 * channels x height x width float planes (distinct buffers).  DEVICE_PTRS /
 * HOST_PTRS and SYNC as for blfls_run; stream NULL = legacy default stream.
 * The initial guidance of rolling_nc_ls (pipelines.cpp:109). */
blfls_status blfls_gaussian_blur(const float* in, int channels, int height, int width,
                                 double sigma, float* out, int device, void* stream,
                                 unsigned flags);

/* ------------------------------------------------------------ multi-GPU --
 * One process driving several devices (the C++ host's multi-GPU path; the
 * Python host uses one process per GPU over torch.distributed instead,
 * paper_1812_07122_b200/multigpu.py).  Two decompositions of epls::smooth
 * cascades:
 *
 *  BLFLS_MULTI_BATCH  the batch is split into contiguous shards, one per
 *                     device entry; each entry has its own plan, stream and
 *                     host thread and runs blfls_run(HOST_PTRS | ASYNC) on its
 *                     shard (no data-path exchange: images are independent,
 *                     pipelines.cpp:57-94 per image).
 *  BLFLS_MULTI_BAND   ONE image (max_batch 1) in row bands: per iteration every
 *                     entry filters its band and stores the band's targets
 *                     into the full-height target buffers of every entry
 *                     (NVLink peer stores from the filter kernel,
 *                     blfls_filter_gradients_rows_peers), then every entry
 *                     runs the full FFT solve redundantly, so each holds the
 *                     whole next iterate; ordering by cross-device events.
 *
 * A device may appear more than once (several entries on one GPU share it).
 * Distinct devices need peer access in band mode (BLFLS_EUNSUPPORTED
 * otherwise; there is no silent fallback).  Results are bit-identical to
 * blfls_run on one device.  img / guide / out are HOST pointers (flags may add
 * BLFLS_CHECK_FINITE); the call returns when `out` is complete. */
#define BLFLS_MULTI_BATCH 0
#define BLFLS_MULTI_BAND 1

typedef struct blfls_multi_s* blfls_multi_t;

/* params->max_batch = the largest batch per call (1 in band mode);
 * params->device is ignored: `devices` (n entries, 1..8) lists the GPUs. */
blfls_status blfls_multi_create(const blfls_params* params, const int* devices, int ndevices,
                                int mode, blfls_multi_t* multi);
blfls_status blfls_multi_run(blfls_multi_t multi, const float* img, const float* guide, int batch,
                             int iters, float* out, unsigned flags);
blfls_status blfls_multi_destroy(blfls_multi_t multi);

/* Page-locked host buffers (cudaHostAlloc) for HOST_PTRS calls, so host code
 * needs no CUDA runtime of its own (the C++ host's blfls::Plan staging). */
blfls_status blfls_host_alloc(size_t bytes, void** ptr);
blfls_status blfls_host_free(void* ptr);

/* Counters of the last blfls_run on this plan (for the bench's roofline). */
typedef struct blfls_stats {
    int radius;
    long long blf_launches;      /* grad+BLF kernel launches */
    long long kernel_launches;   /* all kernels issued by the last call */
    double exps;                 /* range-kernel exponentials the algorithm needs */
} blfls_stats;
blfls_status blfls_last_stats(blfls_plan_t plan, blfls_stats* stats);

/* Sums of the CUDA-event durations (ms) of every stage launched under
 * BLFLS_TIME_STAGES since the last call, and launch counts, indexed
 * 0 min/max, 1 grad+BLF, 2 row r2c, 3 column solve, 4 row c2r.  Synchronizes
 * the recorded events. */
blfls_status blfls_stage_times(blfls_plan_t plan, double* ms_sum5, long long* launches5);

/* Per-image (lo, hi) normalisation ranges the plan holds: out[0 .. 4*max_batch)
 * = two ping-pong slots of (lo, hi) per image (slot k%2 feeds iteration k).
 * Synchronizes the plan stream.  For tests of the fused min/max epilogue. */
blfls_status blfls_debug_ranges(blfls_plan_t plan, float* out);

/* Measured MUFU.EX2 throughput of `device` (ex2 per second), from a
 * dependency-free ex2 loop over all SMs: the SFU roofline denominator. */
blfls_status blfls_mufu_peak(int device, double* ex2_per_second, double* sm_clock_hz);

const char* blfls_last_error(void);
const char* blfls_version(void);
int blfls_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* BLFLS_H */
