// k_grid.cu -- bilateral-grid backend of the gradient filter: the filter the
// reference's smooth() actually runs for BLF_LS (pipelines.cpp:46-48 ->
// blf_grid, bilateral.cpp:112-207), offered beside the brute-force north-star
// kernel for exact parity with the shipped pipeline.
//
// Per gradient plane (image b, channel c, axis a) -- one CTA column per
// plane-axis "slot" in every launch (blockIdx.z = slot):
//   1. src01 / guide01 = ((gn[x+1] - gn[x]) + 1) * 0.5 with gn = (f - lo) * scale,
//      evaluated in double exactly as image.cpp:57-58, :89-90 and
//      pipelines.cpp:21 do, so nearest-cell indices (std::lround) are
//      bit-identical to the reference's; emin / emax of guide01 per slot.
//   2. splat (bilateral.cpp:146-164): cell += {1, src01} (double atomics).
//   3. separable 5-tap blur, sigma 1 cell, along y, x, range
//      (bilateral.cpp:82-108, 166-173), out of place.
//   4. trilinear slice (bilateral.cpp:175-205); T = 2 * out - 1
//      (pipelines.cpp:25-31) scaled to raw image units (* (hi - lo)) for the
//      FFT solve, which runs on the raw image (normalisation fold).
// Grid geometry per slot: gw = floor((W-1)/ss)+5, gh = floor((H-1)/ss)+5,
// gd = floor((emax-emin)/sr)+5 <= floor(1/sr)+5 (guide01 lies in [0, 1]); the
// workspace is sized for the bound and each slot reads its own gd.
#include "blfls_internal.cuh"

namespace blfls {



__device__ __forceinline__ unsigned long long dbl_to_ordered(double d)
{
    unsigned long long b = __double_as_longlong(d);
    return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double ordered_to_dbl(unsigned long long k)
{
    const unsigned long long b = (k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k;
    return __longlong_as_double(b);
}

// slot -> (image b, channel c, axis a); slot = (plane0 + local plane) * 2 + axis
struct Slot {
    int b, c, axis;
};
__device__ __forceinline__ Slot slot_of(const GridParams& p, int z)
{
    const int gp = p.plane0 * 2 + z;
    Slot s;
    s.axis = gp & 1;
    const int plane = gp >> 1;
    s.b = plane / p.C;
    s.c = plane - s.b * p.C;
    return s;
}

// normalisation (lo, scale) of an image in double, image.cpp:46-60
__device__ __forceinline__ void norm_of(const uint32_t* lohi, int b, double& lo, double& scale)
{
    const double l = (double)ordered_to_float(lohi[2 * b]);
    const double h = (double)ordered_to_float(lohi[2 * b + 1]);
    lo = l;
    scale = h > l ? 1.0 / (h - l) : 0.0;  // constant image -> zeros
}

// ((gn[next] - gn[here]) + 1) * 0.5, every operation rounded as the reference's
__device__ __forceinline__ double grad01(const float* img, int H, int W, int y, int x, int axis,
                                         double lo, double scale)
{
    const int xn = axis == 0 ? (x + 1 == W ? 0 : x + 1) : x;
    const int yn = axis == 0 ? y : (y + 1 == H ? 0 : y + 1);
    const double a = __dmul_rn(__dsub_rn((double)__ldg(img + (size_t)yn * W + xn), lo), scale);
    const double b = __dmul_rn(__dsub_rn((double)__ldg(img + (size_t)y * W + x), lo), scale);
    return __dmul_rn(__dadd_rn(__dsub_rn(a, b), 1.0), 0.5);
}

__device__ __forceinline__ void slot_images(const GridParams& p, const Slot& s, const float*& src,
                                            const float*& gde, double& slo, double& ssc, double& glo,
                                            double& gsc)
{
    const size_t plane = (size_t)p.H * p.W;
    src = p.f + ((size_t)s.b * p.C + s.c) * plane;
    norm_of(p.lohi, s.b, slo, ssc);
    if (p.guide) {
        gde = p.guide + ((size_t)s.b * p.GC + (p.GC == 1 ? 0 : s.c)) * plane;
        norm_of(p.glohi, s.b, glo, gsc);
    } else {
        gde = src;
        glo = slo;
        gsc = ssc;
    }
}

__global__ void k_grid_clear(GridParams p)
{
    const size_t total = p.cells * p.slots;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (size_t)gridDim.x * blockDim.x) {
        p.wgrid[i] = 0.0;
        p.vgrid[i] = 0.0;
    }
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < (size_t)p.slots) {
        p.erange[2 * i] = ~0ull;
        p.erange[2 * i + 1] = 0ull;
    }
}

// emin / emax of guide01 per slot; grid (blocks, slots)
__global__ void k_grid_erange(GridParams p)
{
    const Slot s = slot_of(p, blockIdx.y);
    const float *src, *gde;
    double slo, ssc, glo, gsc;
    slot_images(p, s, src, gde, slo, ssc, glo, gsc);
    double lo = 1e300, hi = -1e300;
    const size_t n = (size_t)p.H * p.W;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) {
        const int y = (int)(i / p.W), x = (int)(i - (size_t)y * p.W);
        const double e = grad01(gde, p.H, p.W, y, x, s.axis, glo, gsc);
        lo = fmin(lo, e);
        hi = fmax(hi, e);
    }
    for (int o = 16; o > 0; o >>= 1) {
        lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(&p.erange[2 * blockIdx.y], dbl_to_ordered(lo));
        atomicMax(&p.erange[2 * blockIdx.y + 1], dbl_to_ordered(hi));
    }
}

__device__ __forceinline__ int slot_gd(const GridParams& p, int z, double& emin)
{
    emin = ordered_to_dbl(p.erange[2 * z]);
    const double emax = ordered_to_dbl(p.erange[2 * z + 1]);
    int gd = (int)floor((emax - emin) / p.sr) + 1 + 4;
    return gd > p.gdmax ? p.gdmax : gd;
}

// bilateral.cpp:146-164 (sy = gw*gd, sx = gd, sz = 1)
__global__ void k_grid_splat(GridParams p)
{
    const int z = blockIdx.y;
    const Slot s = slot_of(p, z);
    const float *src, *gde;
    double slo, ssc, glo, gsc;
    slot_images(p, s, src, gde, slo, ssc, glo, gsc);
    double emin;
    const int gd = slot_gd(p, z, emin);
    double* wg = p.wgrid + (size_t)z * p.cells;
    double* vg = p.vgrid + (size_t)z * p.cells;
    const size_t n = (size_t)p.H * p.W;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) {
        const int y = (int)(i / p.W), x = (int)(i - (size_t)y * p.W);
        const int gy = (int)llround(y / p.ss) + 2;
        const int gx = (int)llround(x / p.ss) + 2;
        const double e = grad01(gde, p.H, p.W, y, x, s.axis, glo, gsc);
        const int gz = (int)llround(__ddiv_rn(__dsub_rn(e, emin), p.sr)) + 2;
        const size_t cell = ((size_t)gy * p.gw + gx) * gd + gz;
        atomicAdd(wg + cell, 1.0);
        atomicAdd(vg + cell, grad01(src, p.H, p.W, y, x, s.axis, slo, ssc));
    }
}

// grid_blur_axis (bilateral.cpp:82-108) along axis `ax` (0 y, 1 x, 2 range),
// out of place from `in` to `out`; the taps are summed in the reference's
// order.  grid (blocks, slots).
__global__ void k_grid_blur(GridParams p, const double* in, double* out, int ax)
{
    const int z = blockIdx.y;
    double emin;
    const int gd = slot_gd(p, z, emin);
    const size_t n = (size_t)p.gh * p.gw * gd;
    const double* g = in + (size_t)z * p.cells;
    double* o = out + (size_t)z * p.cells;
    const double r0 = exp(-2.0), r1 = exp(-0.5);
    const double ksum = r0 + r1 + 1.0 + r1 + r0;
    const double k[5] = {r0 / ksum, r1 / ksum, 1.0 / ksum, r1 / ksum, r0 / ksum};
    const int nlen = ax == 0 ? p.gh : (ax == 1 ? p.gw : gd);
    const size_t stride = ax == 0 ? (size_t)p.gw * gd : (ax == 1 ? (size_t)gd : 1);
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) {
        const int iz = (int)(i % gd);
        const size_t r = i / gd;
        const int ix = (int)(r % p.gw), iy = (int)(r / p.gw);
        const int pos = ax == 0 ? iy : (ax == 1 ? ix : iz);
        double acc = 0.0;
#pragma unroll
        for (int t = -2; t <= 2; ++t) {
            const int j = pos + t;
            if (j >= 0 && j < nlen) acc += k[t + 2] * g[i + (long long)t * (long long)stride];
        }
        o[i] = acc;
    }
}

// bilateral.cpp:175-205 + from_unit_range (pipelines.cpp:25-31) + raw scaling
__global__ void k_grid_slice(GridParams p)
{
    const int z = blockIdx.y;
    const Slot s = slot_of(p, z);
    const float *src, *gde;
    double slo, ssc, glo, gsc;
    slot_images(p, s, src, gde, slo, ssc, glo, gsc);
    double emin;
    const int gd = slot_gd(p, z, emin);
    const double* wg = p.wtmp + (size_t)z * p.cells;  // blurred (see launch_grid_blf)
    const double* vg = p.vtmp + (size_t)z * p.cells;
    const size_t sy = (size_t)p.gw * gd, sx = gd;
    const size_t n = (size_t)p.H * p.W;
    const double range = ssc > 0.0 ? 1.0 / ssc : 1.0;
    float* dst = (s.axis == 0 ? p.tx : p.ty) + ((size_t)s.b * p.C + s.c) * n;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) {
        const int y = (int)(i / p.W), x = (int)(i - (size_t)y * p.W);
        const double fy = y / p.ss + 2;
        const double fx = x / p.ss + 2;
        const double e = grad01(gde, p.H, p.W, y, x, s.axis, glo, gsc);
        const double fz = (e - emin) / p.sr + 2;
        const int iy = min((int)fy, p.gh - 2);
        const int ix = min((int)fx, p.gw - 2);
        const int iz = min((int)fz, gd - 2);
        const double ay = fy - iy, ax = fx - ix, az = fz - iz;
        double wsum = 0.0, vsum = 0.0;
#pragma unroll
        for (int dy = 0; dy < 2; ++dy)
#pragma unroll
            for (int dx = 0; dx < 2; ++dx)
#pragma unroll
                for (int dz = 0; dz < 2; ++dz) {
                    const double cw = (dy ? ay : 1.0 - ay) * (dx ? ax : 1.0 - ax) * (dz ? az : 1.0 - az);
                    const size_t ci = sy * (iy + dy) + sx * (ix + dx) + (iz + dz);
                    wsum += cw * wg[ci];
                    vsum += cw * vg[ci];
                }
        const double v = grad01(src, p.H, p.W, y, x, s.axis, slo, ssc);
        const double out = wsum > 1e-12 ? vsum / wsum : v;
        dst[i] = (float)((2.0 * out - 1.0) * (p.normalized ? 1.0 : range));
    }
}

cudaError_t launch_grid_blf(const GridParams& p, int nsm, cudaStream_t st)
{
    const unsigned blocks = (unsigned)(nsm * 4);
    k_grid_clear<<<blocks * p.slots, 256, 0, st>>>(p);
    dim3 g2(blocks, p.slots);
    k_grid_erange<<<g2, 256, 0, st>>>(p);
    k_grid_splat<<<g2, 256, 0, st>>>(p);
    // y, x, range (bilateral.cpp:166-173): grid -> tmp -> grid -> tmp
    for (int w = 0; w < 2; ++w) {
        double* g = w ? p.vgrid : p.wgrid;
        double* t = w ? p.vtmp : p.wtmp;
        k_grid_blur<<<g2, 256, 0, st>>>(p, g, t, 0);
        k_grid_blur<<<g2, 256, 0, st>>>(p, t, g, 1);
        k_grid_blur<<<g2, 256, 0, st>>>(p, g, t, 2);
    }
    k_grid_slice<<<g2, 256, 0, st>>>(p);
    return cudaGetLastError();
}

}  // namespace blfls
