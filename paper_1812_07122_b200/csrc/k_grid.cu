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
//   2. splat (bilateral.cpp:146-164): cell += {1, src01}, integer (fixed
//      point) accumulation so the result is independent of atomic order.
//   3. separable 5-tap blur, sigma 1 cell, along y, x, range
//      (bilateral.cpp:82-108, 166-173), out of place.
//   4. trilinear slice (bilateral.cpp:175-205); T = 2 * out - 1
//      (pipelines.cpp:25-31) scaled to raw image units (* (hi - lo)) for the
//      FFT solve, which runs on the raw image (normalisation fold).
// Grid geometry per slot: gw = floor((W-1)/ss)+5, gh = floor((H-1)/ss)+5,
// gd = floor((emax-emin)/sr)+5 <= floor(1/sr)+5 (guide01 lies in [0, 1]); the
// workspace is sized for the bound and each slot reads its own gd.
#include <cmath>
#include <cstdlib>

#include "blfls_internal.cuh"
#include "slot_common.cuh"

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

// Splat accumulators are integers so that the sums, and hence the output,
// do not depend on atomic ordering (run-to-run byte-identical, the property
// the reference gets from its serial splat, bilateral.cpp:142-145): counts
// exactly, values src01 in [0, 1] in fixed point with 2^-39 resolution
// (quantisation <= 1e-12, far below the float output's round-off).
constexpr double kFixedScale = 549755813888.0;  // 2^39
__device__ __forceinline__ unsigned long long to_fixed(double v)
{
    return (unsigned long long)__double2ll_rn(v * kFixedScale);
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

// emin / emax of guide01 per slot; grid (blocks, slots), rows grid-strided
__global__ void k_grid_erange(GridParams p)
{
    const Slot s = slot_of(p, blockIdx.y);
    const float *src, *gde;
    double slo, ssc, glo, gsc;
    slot_images(p, s, src, gde, slo, ssc, glo, gsc);
    double lo = 1e300, hi = -1e300;
    for (int y = blockIdx.x; y < p.H; y += gridDim.x)
        for (int x = threadIdx.x; x < p.W; x += blockDim.x) {
            const double e = grad01(gde, p.H, p.W, y, x, s.axis, glo, gsc);
            lo = fmin(lo, e);
            hi = fmax(hi, e);
        }
    for (int o = 16; o > 0; o >>= 1) {
        lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if ((threadIdx.x & 31) == 0 && lo <= hi) {
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

// bilateral.cpp:146-164 (sy = gw*gd, sx = gd, sz = 1); global-atomic variant
// for grids whose tile block does not fit in shared memory
__global__ void k_grid_splat(GridParams p)
{
    const int z = blockIdx.y;
    const Slot s = slot_of(p, z);
    const float *src, *gde;
    double slo, ssc, glo, gsc;
    slot_images(p, s, src, gde, slo, ssc, glo, gsc);
    double emin;
    const int gd = slot_gd(p, z, emin);
    unsigned long long* wg = reinterpret_cast<unsigned long long*>(p.wgrid) + (size_t)z * p.cells;
    unsigned long long* vg = reinterpret_cast<unsigned long long*>(p.vgrid) + (size_t)z * p.cells;
    for (int y = blockIdx.x; y < p.H; y += gridDim.x) {
        const int gy = (int)llround(y / p.ss) + 2;
        for (int x = threadIdx.x; x < p.W; x += blockDim.x) {
            const int gx = (int)llround(x / p.ss) + 2;
            const double e = grad01(gde, p.H, p.W, y, x, s.axis, glo, gsc);
            const int gz = (int)llround(__ddiv_rn(__dsub_rn(e, emin), p.sr)) + 2;
            const size_t cell = ((size_t)gy * p.gw + gx) * gd + gz;
            atomicAdd(wg + cell, 1ull);
            atomicAdd(vg + cell, to_fixed(grad01(src, p.H, p.W, y, x, s.axis, slo, ssc)));
        }
    }
}

// Tile-privatised splat: a CTA owns a TP x TP pixel tile (TP <= 64), whose
// nearest cells span at most (TP/ss + 2)^2 x gd cells; it accumulates them in
// shared memory with native 32-bit atomics (count, and the fixed-point value
// split into 20-bit low and high words: a 4096-pixel tile cannot overflow
// either) and flushes each non-empty cell with one 64-bit global atomic.
// grid (tiles, slots); dynamic smem = 3 * ncx * ncy * gd words.
__global__ void k_grid_splat_tiled(GridParams p, int lgTP, int ncx, int ncy)
{
    extern __shared__ unsigned sacc[];  // [3][ncy][ncx][gd]: count, value lo, value hi
    __shared__ int tgx[64], tgy[64];    // tile-local nearest cells of each column / row
    const int TP = 1 << lgTP;
    const int z = blockIdx.y;
    const Slot s = slot_of(p, z);
    const float *src, *gde;
    double slo, ssc, glo, gsc;
    slot_images(p, s, src, gde, slo, ssc, glo, gsc);
    double emin;
    const int gd = slot_gd(p, z, emin);
    const int tiles_x = (p.W + TP - 1) >> lgTP;
    const int tx0 = (blockIdx.x % tiles_x) << lgTP, ty0 = (blockIdx.x / tiles_x) << lgTP;
    const int cx0 = (int)llround(tx0 / p.ss) + 2, cy0 = (int)llround(ty0 / p.ss) + 2;
    const int n = ncx * ncy * gd;
    unsigned* scount = sacc;
    unsigned* slo20 = sacc + n;
    unsigned* shi = sacc + 2 * n;
    for (int i = threadIdx.x; i < 3 * n; i += blockDim.x) sacc[i] = 0u;
    if (threadIdx.x < TP) {
        tgx[threadIdx.x] = (int)llround((tx0 + (int)threadIdx.x) / p.ss) + 2 - cx0;
        tgy[threadIdx.x] = (int)llround((ty0 + (int)threadIdx.x) / p.ss) + 2 - cy0;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < TP * TP; i += blockDim.x) {
        const int ly = i >> lgTP, lx = i & (TP - 1);
        const int y = ty0 + ly, x = tx0 + lx;
        if (y >= p.H || x >= p.W) continue;
        const double e = grad01(gde, p.H, p.W, y, x, s.axis, glo, gsc);
        const int gz = (int)llround(__ddiv_rn(__dsub_rn(e, emin), p.sr)) + 2;
        const int c = (tgy[ly] * ncx + tgx[lx]) * gd + gz;
        const unsigned long long q = to_fixed(grad01(src, p.H, p.W, y, x, s.axis, slo, ssc));
        atomicAdd(&scount[c], 1u);
        atomicAdd(&slo20[c], (unsigned)(q & 0xfffffu));
        atomicAdd(&shi[c], (unsigned)(q >> 20));
    }
    __syncthreads();
    unsigned long long* wg = reinterpret_cast<unsigned long long*>(p.wgrid) + (size_t)z * p.cells;
    unsigned long long* vg = reinterpret_cast<unsigned long long*>(p.vgrid) + (size_t)z * p.cells;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const unsigned w = scount[i];
        if (w == 0u) continue;
        const int gz = i % gd, r = i / gd;
        const int gx = r % ncx + cx0, gy = r / ncx + cy0;
        if (gx >= p.gw || gy >= p.gh) continue;
        const size_t cell = ((size_t)gy * p.gw + gx) * gd + gz;
        atomicAdd(wg + cell, (unsigned long long)w);
        atomicAdd(vg + cell, ((unsigned long long)shi[i] << 20) + slo20[i]);
    }
}

// grid_blur_axis (bilateral.cpp:82-108) along axis `ax` (0 y, 1 x, 2 range),
// out of place from `in` to `out`; the taps are summed in the reference's
// order.  grid (blocks, slots).
__global__ void k_grid_blur(GridParams p, const double* in, double* out, int ax, double in_scale,
                            int ostride, int ooff)
{
    const int z = blockIdx.y;
    double emin;
    const int gd = slot_gd(p, z, emin);
    const double* g = in + (size_t)z * p.cells;
    double* o = out + (size_t)z * p.cells * ostride + ooff;
    const double r0 = exp(-2.0), r1 = exp(-0.5);
    const double ksum = r0 + r1 + 1.0 + r1 + r0;
    const double k[5] = {r0 / ksum, r1 / ksum, 1.0 / ksum, r1 / ksum, r0 / ksum};
    const int nlen = ax == 0 ? p.gh : (ax == 1 ? p.gw : gd);
    const int stride = ax == 0 ? p.gw * gd : (ax == 1 ? gd : 1);
    const int row = p.gw * gd;  // one grid row (iy fixed) is contiguous
    for (int iy = blockIdx.x; iy < p.gh; iy += gridDim.x) {
        const double* gr = g + (size_t)iy * row;
        double* orow = o + (size_t)iy * row * ostride;
        for (int j = threadIdx.x; j < row; j += blockDim.x) {
            const int pos = ax == 0 ? iy : (ax == 1 ? j / gd : j % gd);
            double acc = 0.0;
#pragma unroll
            for (int t = -2; t <= 2; ++t) {
                const int q = pos + t;
                if (q >= 0 && q < nlen) {
                    double v = gr[j + t * stride];
                    if (in_scale != 0.0)  // first pass: integer splat accumulators
                        v = (double)__double_as_longlong(v) * in_scale;
                    acc += k[t + 2] * v;
                }
            }
            orow[(size_t)j * ostride] = acc;
        }
    }
}

// The three blur passes fused (bilateral.cpp:166-173: y, then x, then range,
// each grid_blur_axis): a CTA owns a B x B block of (y, x) cells with every
// range cell, loads it with a 2-cell halo (converting the integer splat
// accumulators), blurs y into T1 (B x (B+4) x gd), x into T2 (B x B x gd,
// reusing the load buffer) and range on the way out to `out`.  Taps outside
// the grid are dropped exactly as the reference's blur drops them.  Runs for
// the count grid (w = 0) and then the value grid (w = 1).  grid (tiles, slots).
__global__ void k_grid_blur3(GridParams p, int B)
{
    extern __shared__ double sm[];
    const int z = blockIdx.y;
    double emin;
    const int gd = slot_gd(p, z, emin);
    const double r0 = exp(-2.0), r1 = exp(-0.5);
    const double ksum = r0 + r1 + 1.0 + r1 + r0;
    const double k[5] = {r0 / ksum, r1 / ksum, 1.0 / ksum, r1 / ksum, r0 / ksum};
    const int BH = B + 4;
    const int tiles_x = (p.gw + B - 1) / B;
    const int x0 = (blockIdx.x % tiles_x) * B, y0 = (blockIdx.x / tiles_x) * B;
    const int rowL = BH * gd;  // one halo row of the load buffer
    double* L = sm;                      // [BH][BH][gd], later T2 [B][B][gd]
    double* T1 = sm + (size_t)BH * rowL;  // [B][BH][gd]
    // Each phase walks a row offset j (x * gd + z within a tile row) per
    // thread and loops over the tile rows, so the index divisions happen once
    // per j rather than once per cell.
    const int rowB = B * gd;
    for (int w = 0; w < 2; ++w) {
        const unsigned long long* in =
            reinterpret_cast<const unsigned long long*>(w ? p.vgrid : p.wgrid) + (size_t)z * p.cells;
        double* out = p.blurred + (size_t)z * p.cells * 2 + w;
        const double scale = w ? 1.0 / kFixedScale : 1.0;
        for (int j = threadIdx.x; j < rowL; j += blockDim.x) {  // load with halo
            const int gx = x0 - 2 + j / gd;
            const bool xin = gx >= 0 && gx < p.gw;
            const long long off = (long long)(x0 - 2) * gd + j;
            for (int ly = 0; ly < BH; ++ly) {
                const int gy = y0 - 2 + ly;
                double v = 0.0;
                if (xin && gy >= 0 && gy < p.gh) v = (double)in[(size_t)gy * p.gw * gd + off] * scale;
                L[ly * rowL + j] = v;
            }
        }
        __syncthreads();
        for (int j = threadIdx.x; j < rowL; j += blockDim.x)  // y
            for (int ly = 0; ly < B; ++ly) {
                const int gy = y0 + ly;
                double acc = 0.0;
#pragma unroll
                for (int t = -2; t <= 2; ++t)
                    if (gy + t >= 0 && gy + t < p.gh) acc += k[t + 2] * L[(ly + 2 + t) * rowL + j];
                T1[ly * rowL + j] = acc;
            }
        __syncthreads();
        for (int j = threadIdx.x; j < rowB; j += blockDim.x) {  // x
            const int gx = x0 + j / gd;
            unsigned ok = 0;
#pragma unroll
            for (int t = -2; t <= 2; ++t) ok |= (gx + t >= 0 && gx + t < p.gw) ? 1u << (t + 2) : 0u;
            for (int ly = 0; ly < B; ++ly) {
                const double* r = T1 + ly * rowL + j + 2 * gd;
                double acc = 0.0;
#pragma unroll
                for (int t = -2; t <= 2; ++t)
                    if (ok >> (t + 2) & 1u) acc += k[t + 2] * r[t * gd];
                L[ly * rowB + j] = acc;
            }
        }
        __syncthreads();
        for (int j = threadIdx.x; j < rowB; j += blockDim.x) {  // range, store
            const int lx = j / gd, iz = j - lx * gd;
            const int gx = x0 + lx;
            if (gx >= p.gw) continue;
            for (int ly = 0; ly < B && y0 + ly < p.gh; ++ly) {
                const double* r = L + ly * rowB + j;
                double acc = 0.0;
#pragma unroll
                for (int t = -2; t <= 2; ++t)
                    if (iz + t >= 0 && iz + t < gd) acc += k[t + 2] * r[t];
                out[(((size_t)(y0 + ly) * p.gw + gx) * gd + iz) * 2] = acc;
            }
        }
        __syncthreads();
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
    const double2* bg = reinterpret_cast<const double2*>(p.blurred) + (size_t)z * p.cells;
    const int sy = p.gw * gd, sx = gd;
    const size_t n = (size_t)p.H * p.W;
    const double range = ssc > 0.0 ? 1.0 / ssc : 1.0;
    const double scale = 2.0 * (p.normalized ? 1.0 : range), shift = p.normalized ? 1.0 : range;
    // The trilinear weights are continuous in (fy, fx, fz), so the cell
    // coordinates are formed with reciprocals instead of the reference's
    // divisions (bilateral.cpp:182-184): a 1-ulp coordinate change moves the
    // output by ~1e-16, far inside the float output's tolerance.
    const double inv_ss = 1.0 / p.ss, inv_sr = 1.0 / p.sr;
    float* dst = (s.axis == 0 ? p.tx : p.ty) + ((size_t)s.b * p.C + s.c) * n;
    for (int y = blockIdx.x; y < p.H; y += gridDim.x) {
        const double fy = y * inv_ss + 2;
        const int iy = min((int)fy, p.gh - 2);
        const double ay = fy - iy;
        for (int x = threadIdx.x; x < p.W; x += blockDim.x) {
            const double fx = x * inv_ss + 2;
            const double e = grad01(gde, p.H, p.W, y, x, s.axis, glo, gsc);
            const double fz = (e - emin) * inv_sr + 2;
            const int ix = min((int)fx, p.gw - 2);
            const int iz = min((int)fz, gd - 2);
            const double ax = fx - ix, az = fz - iz;
            const double2* c0 = bg + sy * iy + sx * ix + iz;
            double wsum = 0.0, vsum = 0.0;
#pragma unroll
            for (int dy = 0; dy < 2; ++dy)
#pragma unroll
                for (int dx = 0; dx < 2; ++dx) {
                    const double wyx = (dy ? ay : 1.0 - ay) * (dx ? ax : 1.0 - ax);
                    const int o = sy * dy + sx * dx;
                    const double w0 = wyx * (1.0 - az), w1 = wyx * az;
                    const double2 a = c0[o], b = c0[o + 1];
                    wsum += w0 * a.x + w1 * b.x;
                    vsum += w0 * a.y + w1 * b.y;
                }
            double out;
            if (wsum > 1e-12)
                out = vsum / wsum;
            else
                out = grad01(src, p.H, p.W, y, x, s.axis, slo, ssc);
            dst[(size_t)y * p.W + x] = (float)(out * scale - shift);
        }
    }
}

cudaError_t launch_grid_blf(const GridParams& p, int nsm, cudaStream_t st, int* launches)
{
    *launches = 4;  // clear, erange, splat, slice (+ blur below)
    const unsigned blocks = (unsigned)(nsm * 4);
    k_grid_clear<<<blocks * p.slots, 256, 0, st>>>(p);
    dim3 g2(blocks, p.slots);
    k_grid_erange<<<g2, 256, 0, st>>>(p);
    // privatised splat when a pixel tile's cell block fits in 64 KB of smem
    int TP = 0, lgTP = 0, ncx = 0;
    for (int lg = 6; lg >= 3; --lg) {
        const int nc = (int)std::ceil((1 << lg) / p.ss) + 2;
        if ((size_t)nc * nc * p.gdmax * 3 * sizeof(unsigned) <= 64 * 1024) {
            TP = 1 << lg;
            lgTP = lg;
            ncx = nc;
            break;
        }
    }
    if (TP) {
        const size_t smem = (size_t)ncx * ncx * p.gdmax * 3 * sizeof(unsigned);
        if (smem > 48 * 1024)
            cudaFuncSetAttribute(k_grid_splat_tiled, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        dim3 gt((unsigned)(((p.W + TP - 1) / TP) * ((p.H + TP - 1) / TP)), p.slots);
        k_grid_splat_tiled<<<gt, 256, smem, st>>>(p, lgTP, ncx, ncx);
    } else {
        k_grid_splat<<<g2, 256, 0, st>>>(p);
    }
    // y, x, range (bilateral.cpp:166-173): grid -> tmp -> grid -> tmp
    // fused 3-axis blur when a B x B cell block (+ halo, all range cells) fits
    int B = 0;
    size_t bsmem = 0;
    static const int forced_b = knob("BLFLS_GRID_BLUR_B", 0);
    for (int b : {8, 16, 4}) {  // 8: best measured (c5: 3.83 vs 4.03 ms at 16)
        if (forced_b && b != forced_b) continue;
        const size_t need = (size_t)((b + 4) * (b + 4) + b * (b + 4)) * p.gdmax * sizeof(double);
        if (need <= 112 * 1024) {
            B = b;
            bsmem = need;
            break;
        }
    }
    if (B) {
        if (bsmem > 48 * 1024)
            cudaFuncSetAttribute(k_grid_blur3, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsmem);
        dim3 gb((unsigned)(((p.gw + B - 1) / B) * ((p.gh + B - 1) / B)), p.slots);
        k_grid_blur3<<<gb, 256, bsmem, st>>>(p, B);
        *launches += 1;
    } else {
        // y, x, range per grid; scratch: the (not yet written) blurred buffer
        // for the counts, the dead count grid for the values
        const double fs = 1.0 / kFixedScale;
        k_grid_blur<<<g2, 256, 0, st>>>(p, p.wgrid, p.blurred, 0, 1.0, 1, 0);
        k_grid_blur<<<g2, 256, 0, st>>>(p, p.blurred, p.wgrid, 1, 0.0, 1, 0);
        k_grid_blur<<<g2, 256, 0, st>>>(p, p.wgrid, p.blurred, 2, 0.0, 2, 0);
        k_grid_blur<<<g2, 256, 0, st>>>(p, p.vgrid, p.wgrid, 0, fs, 1, 0);
        k_grid_blur<<<g2, 256, 0, st>>>(p, p.wgrid, p.vgrid, 1, 0.0, 1, 0);
        k_grid_blur<<<g2, 256, 0, st>>>(p, p.vgrid, p.blurred, 2, 0.0, 2, 1);
        *launches += 6;
    }
    k_grid_slice<<<g2, 256, 0, st>>>(p);
    return cudaGetLastError();
}

}  // namespace blfls
