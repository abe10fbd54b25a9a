// blfls_internal.cuh -- shared definitions of the sm_100a BLF-LS library.
#pragma once

#include <string>
#include <vector>

#include <cuda_runtime.h>
#include <stdint.h>

#include "blfls/blfls.h"

namespace blfls {

// ----------------------------------------------------------------- knobs --
// Kernel-selection overrides for A/B experiments.  The production library
// (default build) ignores the environment entirely: knob() returns the
// measured default.  Building with -DBLFLS_EXPERIMENTS (python -m
// paper_1812_07122_b200.build --experiments) reads BLFLS_* variables.
#ifdef BLFLS_EXPERIMENTS
int knob(const char* name, int def);
#else
constexpr int knob(const char*, int def) { return def; }
#endif

// sets the calling thread's blfls_last_error() message and returns st
blfls_status report(blfls_status st, const std::string& msg);

constexpr int kMaxRadius = 48;     // smem tile envelope (radius <= 48)
constexpr int kMaxPeers = 8;       // fused band exchange: ranks of one NVLink domain
constexpr int kMaxFftRadices = 32;
constexpr int kMaxGenericRadix = 31;

// log2(e)
constexpr float kLog2e = 1.4426950408889634f;

// ---------------------------------------------------------------- min/max --
// Order-preserving float <-> uint32 map so atomicMin/atomicMax on unsigned
// implement float min/max (the per-image global range of image.cpp:46-60).
__host__ __device__ inline uint32_t float_to_ordered(float f)
{
    uint32_t b;
#ifdef __CUDA_ARCH__
    b = __float_as_uint(f);
#else
    __builtin_memcpy(&b, &f, 4);
#endif
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

__host__ __device__ inline float ordered_to_float(uint32_t k)
{
    const uint32_t b = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
#ifdef __CUDA_ARCH__
    return __uint_as_float(b);
#else
    float f;
    __builtin_memcpy(&f, &b, 4);
    return f;
#endif
}

// --------------------------------------------------------------------- FFT --
// Stockham autosort, decimation in frequency, radix stages in `radix[]`.
// Stage with radix p, stride s (product of earlier radices), m = n/(s*p):
//   butterfly b in [0, n/p): k = b % s, q = b / s
//   a_r = x[b + r*n/p]                                  r in [0, p)
//   y[k + s*(p*q + t)] = tw[q*t*s] * sum_r a_r * w_p^{r*t}   t in [0, p)
// with tw[j] = exp(-2*pi*i*j/n).  The inverse conjugates every twiddle.
struct FftDesc {
    int n;
    int nstages;
    int radix[kMaxFftRadices];
    const float2* tw;  // n entries, device
};

// Bluestein transform of a length whose prime factors include one above the
// direct-stage threshold: chirp c_j = exp(-pi i j^2 / n) (n entries), the
// 5-smooth convolution length M >= 2n - 1 and its FFT (m), and the spectra of
// the chirp kernel for the forward / inverse direction with 1/M folded in.
struct BlueDesc {
    FftDesc m;
    const float2* chirp;
    const float2* hf;
    const float2* hi;
};

// launch geometry of one FFT pass: V vectors per CTA, threads = V * TV
struct FftGeom {
    FftDesc desc;
    bool bluestein = false;  // run the length-n transform as a length-M convolution
    BlueDesc blue{};
    int V, log2V, threads;
    int E;         // complex values per thread across a stage barrier (8 or 16)
    bool generic;  // a radix other than 2/3/4/5 occurs
    bool direct;   // a prime factor above 13 (direct DFT stage, 2x shared memory)
    int pmax;      // largest prime factor (root table of the direct stage)
    bool ct;       // a compile-time specialised engine exists for (n, V, threads)
};

// ---------------------------------------------------------------- BLF args --
struct BlfParams {
    const float* f;        // current image, batch x C x H x W
    const float* guide;    // batch x GC x H x W or nullptr (self-guided)
    float* tx;             // targets, batch x C x rows x W
    float* ty;
    const uint32_t* lohi;  // per image ordered (lo, hi) of f
    const uint32_t* glohi; // per image ordered (lo, hi) of the guide
    int H, W, C, GC;
    int y0, y1;            // output rows [y0, y1)
    int out_rows;          // rows per plane of tx/ty (H, or y1 - y0 for bands)
    int normalized_out;    // 1: write targets of the [0,1]-normalised image
    int radius;
    int poly_period;       // SFU offload period of k_grad_blf (< 0: per-mode default)
    int legacy_joint3;     // 1: shared-guide mode uses the unpacked kernel (experiments)
    int joint3_rows;       // output rows per thread of the packed shared-guide kernel
    int x2_poly;           // packed self-guided kernel: FMA-pipe exp2 period (< 0: off)
    int tile_rows;         // k_grad_blf tile height override (0: auto, 8 or 16)
    int cols_per_thread;   // experiment: outputs per thread of k_grad_blf (4 default, 8)
    float range_coef;      // sqrt(log2(e) / (8 sigma_r^2)): exponent scale for raw
                           // gradients of a unit-range image
    float cs[kMaxRadius + 1];  // log2 spatial weight -d^2/(2 sigma_s^2) * log2(e)
    float wrow[kMaxRadius + 1]; // exp2(cs[d]) : row factor
    // column-spatial pairs of two adjacent outputs (q, q + 1) at one source
    // column: cep[i] = (cs[|i - r|], cs[|i - r - 1|]), i in [0, 2r + 1]
    // (entries outside the window hold cs[r]; k_blf_p2.cu pair exponents)
    float2 cep[2 * kMaxRadius + 2];
    // row-factor fold of k_blf_j3r.cu: rfold[d + r] = wy(d - 1) / wy(d) for the
    // window rows d in (-r, r], rfold[0] = 1
    float rfold[2 * kMaxRadius + 2];
    // fused band exchange (multi-GPU row bands): npeers > 0 writes every target
    // into the full-height tx / ty of each peer (NVLink peer-mapped pointers,
    // rank order) instead of tx / ty -- the all-gather done by the epilogue
    int npeers;
    float* peer_tx[kMaxPeers];
    float* peer_ty[kMaxPeers];
};

// bilateral-grid backend (k_grid.cu)
struct GridParams {
    const float* f;        // (padded) image, planes x H x W
    const float* guide;    // (padded) guide or nullptr
    float* tx;             // targets, raw units
    float* ty;
    const uint32_t* lohi;  // per image ordered (lo, hi) of f (fp32)
    const uint32_t* glohi; // per image of the guide
    double* wgrid;         // [slots][cells] splat targets
    double* vgrid;
    double* blurred;       // [slots][cells] interleaved (w, v): the blurred grids
                           // (also scratch of the per-axis fallback blur)
    unsigned long long* erange;  // [slots][2] ordered (emin, emax) of guide01
    int H, W, C, GC;
    int plane0;            // first global plane of this launch
    int slots;             // plane-axes in this launch
    double ss, sr;         // grid sampling (sigma_s, sigma_r)
    int gw, gh, gdmax;     // grid dims (gd per slot <= gdmax)
    size_t cells;          // gw * gh * gdmax
    int normalized;        // 1: targets of the [0,1]-normalised image (stage entry)
};

// domain-transform backend (k_dt.cu): nc_filter per slot
struct DtParams {
    const float* f;        // (padded) image, planes x H x W
    const float* guide;    // (padded) guide or nullptr
    float* tx;             // targets, raw units
    float* ty;
    const uint32_t* lohi;  // per image ordered (lo, hi) of f
    const uint32_t* glohi; // per image of the guide
    double* cth;           // [slots][H][W] warped row coordinates
    double* ctv;           // [slots][H][W] warped column coordinates
    double* pc;            // [slots][pcplane] prefix sums of the current pass
    double* x;             // [slots][H][W] signal between passes
    double* g01;           // [slots][H][W] guide01 (the DT guide) of each slot
    size_t plane;          // H * W
    size_t pcplane;        // (H + 1) * (W + 1)
    int H, W, C, GC;
    int plane0;            // first global plane of this launch
    int slots;             // plane-axes in this launch
    int normalized;        // targets in normalised units (else raw)
    double ratio;          // sigma_s / sigma_r (domain_transform.cpp:142)
};

double nc_box_radius(double sigma_s, int iter, int total);
// returns the number of kernels launched, or -1 on a launch error
bool dt_configure(int iterations, double sigma_s);
size_t blf_plain_smem(int cg, int cs, int R);
cudaError_t launch_forward_gradients(const float* img, float* gx, float* gy, int planes, int H, int W,
                                     int nsm, cudaStream_t st);
cudaError_t launch_blf_plain(const float* src, int cs, const float* guide, int cg, float* out, int batch,
                             int H, int W, int R, double sigma_s, double sigma_r, const float* tables,
                             cudaStream_t st);
int launch_dt_filter(const DtParams& p, int iterations, double sigma_s, int nsm, cudaStream_t st);
std::vector<double> gaussian_weights(double sigma);
cudaError_t launch_gaussian_blur(const float* in, float* out, double* tmp, const double* k, int r,
                                 int C, int H, int W, int nsm, cudaStream_t st);

struct SolveParams {
    const float* f;      // image (batch x C x H x W)
    const float* tx;     // targets or nullptr
    const float* ty;
    float2* spec;        // planes x H x spitch
    float* out;          // output image (oH x oW per plane: the padded grid cropped by opad)
    int oH, oW, opad;
    uint32_t* lohi_out;  // per image ordered (lo, hi) of out, or nullptr
    const float* gain_x; // 4 sin^2(pi v / W), v in [0, W/2]
    const float* gain_y; // 4 sin^2(pi u / H)
    const float2* post;  // exp(-2 pi i v / W), v in [0, W/2]  (real-FFT split)
    int H, W, C;
    int plane0;          // global index of the first plane (per-image min/max slot)
    int spitch;          // complex elements per spectrum row
    int wc;              // W/2 + 1
    float lambda;
    float inv_hw;        // 1 / (H W)
    int mode;            // column pass: 1 fwd, 2 inv, 3 fwd+scale+inv
    // mode 3 as a cyclic tridiagonal solve per spectrum column (k_col_tri.cu):
    // two float4 per column (tri_tables); nullptr: the column FFT pair runs
    const float4* tri;
    int tri_rpt;         // rows per thread the tables were built for
    // the tridiagonal column pass also resets the per-image (lo, hi) slots the
    // row c2r epilogue reduces into (one launch fewer per iteration)
    uint32_t* lohi_reset;
    int lohi_reset_n;
};

// tridiagonal column pass (k_col_tri.cu)
int tri_rows_per_thread(int H, int wc, int planes, int nsm);
bool tri_supported(int H, int rpt);
void tri_tables(int H, int W, int wc, double lambda, int rpt, std::vector<float4>& tri);
cudaError_t launch_col_tri(const SolveParams& p, int planes, int nsm, cudaStream_t st);


// high-radix solve passes (k_solve2.cu): false when no geometry exists for n
bool launch_v2_pass(int which, const SolveParams& p, int n, const float2* tw, int planes, int nsm,
                    cudaStream_t st);


// shared-gray-guide filter with packed accumulation (k_blf_j3.cu); false: not covered
bool launch_grad_blf_j3(const BlfParams& p, int batch, cudaStream_t st, cudaError_t* err);
// two output rows per thread, row factor folded into the sums (k_blf_j3r.cu); false: not covered
bool launch_grad_blf_j3r(const BlfParams& p, int batch, cudaStream_t st, cudaError_t* err);
// eight outputs per thread, factorised exponents (k_blf_j8.cu); false: not covered
bool launch_grad_blf_j8(const BlfParams& p, int batch, cudaStream_t st, cudaError_t* err);

// self-guided filter, two output rows per thread (k_blf_p2r.cu); false: not covered
bool launch_grad_blf_p2r(const BlfParams& p, int nplanes, int nsm, cudaStream_t st, cudaError_t* err);
// self / per-channel-joint filter with packed accumulation (k_blf_p2.cu); false: not covered
bool launch_grad_blf_p2(const BlfParams& p, int mode, int batch, cudaStream_t st, cudaError_t* err);

}  // namespace blfls
