// k_dt.cu -- domain-transform backend of the gradient filter: nc_filter
// (domain_transform.cpp:138-156), the filter the reference's smooth() runs
// for SmootherKind::NC_LS (pipelines.cpp:48), plus gaussian_blur
// (image.cpp:99-158), the initial guidance of rolling_nc_ls.
//
// The reference filters every scanline sequentially: warped coordinates
// ct(k) = ct(k-1) + (1 + ratio * |g(k) - g(k-1)|) (ct(0) = 1), prefix sums of
// the signal, and a window [lo, hi] = {j : |ct(j) - ct(k)| <= radius} found by
// two monotone pointers.  The B200 version keeps the two sequential
// recurrences sequential -- one lane per scanline, additions in the
// reference's order, so ct and the prefix sums are bit-identical -- and makes
// the window step fully parallel: since ct is strictly increasing (steps >= 1)
// the two-pointer bounds equal lower_bound(ct(k) - radius) and
// upper_bound(ct(k) + radius) - 1, which one thread per sample finds by a
// local scan of <= radius steps each way.  The output (pc[hi+1] - pc[lo]) /
// (hi - lo + 1) is therefore the reference's value exactly, in double.
//
// Per slot (image b, channel c, axis a) the signal is src01 and the guide is
// guide01 of that axis and channel (pipelines.cpp:39-47), evaluated from the
// fp32 planes in double with the reference's rounding (slot_common.cuh).
//
// Kernels per smooth() call and slot group, T = DtParams::iterations:
//   k_dt_rows_scan<CT>, k_dt_cols_scan<CT>      warped coordinates ct_h, ct_v
//   T x { k_dt_rows_scan<PREFIX>, k_dt_window<ROWS>,
//         k_dt_cols_scan<PREFIX>, k_dt_window<COLS> }  (the last writes T = 2v-1)
// The scans are sequential per line with only H or W lines per slot, so they
// are latency-bound: each keeps one batch of raw loads in flight while it
// consumes the previous one.
// Row scans stage 32 x 32 tiles through shared memory so that the lane-per-row
// recurrences read and write coalesced; column scans are coalesced directly.
#include <cmath>
#include <vector>

#include "blfls_internal.cuh"
#include "slot_common.cuh"

namespace blfls {

namespace {

constexpr int kScanWarps = 4;  // rows-scan CTA: 4 warps x 32 rows
constexpr int kColU = 16;      // column scan: rows per prefetched batch

// A sample as loaded, before the double arithmetic: SRC 0 = a gradient of an
// fp32 image (the two samples of the forward difference, converted with
// grad01's rounding at use), SRC 1 = a double plane value.  Keeping the raw
// loads lets a scan issue the next batch's loads before it consumes the
// current one (software pipelining of the latency-bound recurrences).
template <int SRC>
struct Raw;
template <>
struct Raw<0> {
    float a, b;
};
template <>
struct Raw<1> {
    double v;
};

struct SlotSrc {
    const float* img;  // SRC 0
    double lo, scale;
    const double* plane;  // SRC 1
    int axis;
};

template <int SRC>
__device__ __forceinline__ Raw<SRC> load_raw(const SlotSrc& q, int H, int W, int y, int x);
template <>
__device__ __forceinline__ Raw<0> load_raw<0>(const SlotSrc& q, int H, int W, int y, int x)
{
    const int xn = q.axis == 0 ? (x + 1 == W ? 0 : x + 1) : x;
    const int yn = q.axis == 0 ? y : (y + 1 == H ? 0 : y + 1);
    return {__ldg(q.img + (size_t)yn * W + xn), __ldg(q.img + (size_t)y * W + x)};
}
template <>
__device__ __forceinline__ Raw<1> load_raw<1>(const SlotSrc& q, int H, int W, int y, int x)
{
    return {q.plane[(size_t)y * W + x]};
}

// grad01 of slot_common.cuh from the two loaded samples
__device__ __forceinline__ double to_val(const Raw<0>& r, const SlotSrc& q)
{
    const double a = __dmul_rn(__dsub_rn((double)r.a, q.lo), q.scale);
    const double b = __dmul_rn(__dsub_rn((double)r.b, q.lo), q.scale);
    return __dmul_rn(__dadd_rn(__dsub_rn(a, b), 1.0), 0.5);
}
__device__ __forceinline__ double to_val(const Raw<1>& r, const SlotSrc&) { return r.v; }

// OP 0 (ct): the guide; OP 1 (prefix): the signal (src01 on the first pass,
// SRC 0, else the plane x of the previous pass, SRC 1)
template <int OP>
__device__ __forceinline__ SlotSrc slot_src(const DtParams& p, int z)
{
    const Slot s = slot_of(p, z);
    const float *src, *gde;
    double slo, ssc, glo, gsc;
    slot_images(p, s, src, gde, slo, ssc, glo, gsc);
    SlotSrc q;
    q.axis = s.axis;
    q.img = OP == 0 ? gde : src;
    q.lo = OP == 0 ? glo : slo;
    q.scale = OP == 0 ? gsc : ssc;
    q.plane = p.x + (size_t)z * p.plane;
    return q;
}

// one step of the reference's scanline recurrences: ct (transform_rows/cols,
// domain_transform.cpp:31-68: d = 0 + |g(k) - g(k-1)|, acc += 1 + ratio*d,
// no contraction) or the prefix sum (box_pass_*: pc[k+1] = pc[k] + v[k])
template <int OP>
__device__ __forceinline__ double scan_step(double acc, double v, double& prev, bool first,
                                            double ratio)
{
    if (OP == 0) {
        if (!first) acc = __dadd_rn(acc, __dadd_rn(1.0, __dmul_rn(ratio, fabs(__dsub_rn(v, prev)))));
        prev = v;
        return acc;
    }
    return __dadd_rn(acc, v);
}

// Row scans: OP 0 -> ct_h (transform_rows, domain_transform.cpp:31-49);
// OP 1 -> pc[y][0..W] (box_pass_rows :81-88).  One warp per 32 rows: the
// warp loads a 32 x 32 tile coalesced (rows of the tile), each lane then
// scans its own row through shared memory; the next tile's loads are in
// flight during the scan.  grid (ceil(H / 128), slots), block 128.
template <int OP, int SRC>
__global__ void __launch_bounds__(32 * kScanWarps) k_dt_rows_scan(DtParams p)
{
    __shared__ double tile[kScanWarps][32][33];
    const int z = blockIdx.y;
    const SlotSrc q = slot_src<OP>(p, z);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int y0 = (blockIdx.x * kScanWarps + warp) * 32;
    if (y0 >= p.H) return;
    double (*t)[33] = tile[warp];
    const int my = y0 + lane;  // the row this lane scans
    const int nr = min(32, p.H - y0);
    double acc = OP == 0 ? 1.0 : 0.0, prev = 0.0;
    double* pcz = p.pc + (size_t)z * p.pcplane;
    double* ctz = p.cth + (size_t)z * p.plane;
    if (OP == 1 && my < p.H) pcz[(size_t)my * (p.W + 1)] = 0.0;
    Raw<SRC> cur[32], nxt[32];
#pragma unroll
    for (int r = 0; r < 32; ++r)
        if (r < nr && lane < p.W) cur[r] = load_raw<SRC>(q, p.H, p.W, y0 + r, lane);
    for (int x0 = 0; x0 < p.W; x0 += 32) {
        const int xl = x0 + lane;
        const int xn = xl + 32;
        if (x0 + 32 < p.W) {
#pragma unroll
            for (int r = 0; r < 32; ++r)
                if (r < nr && xn < p.W) nxt[r] = load_raw<SRC>(q, p.H, p.W, y0 + r, xn);
        }
#pragma unroll
        for (int r = 0; r < 32; ++r)
            if (r < nr && xl < p.W) t[r][lane] = to_val(cur[r], q);
        __syncwarp();
        const int nc = min(32, p.W - x0);
        if (my < p.H) {
            for (int c = 0; c < nc; ++c) {
                acc = scan_step<OP>(acc, t[lane][c], prev, x0 + c == 0, p.ratio);
                t[lane][c] = acc;
            }
        }
        __syncwarp();
#pragma unroll 4
        for (int r = 0; r < 32; ++r) {
            if (r < nr && xl < p.W) {
                if (OP == 0)
                    ctz[(size_t)(y0 + r) * p.W + xl] = t[r][lane];
                else
                    pcz[(size_t)(y0 + r) * (p.W + 1) + xl + 1] = t[r][lane];
            }
        }
        __syncwarp();
#pragma unroll
        for (int r = 0; r < 32; ++r) cur[r] = nxt[r];
    }
}

// Column scans: OP 0 -> ct_v (transform_cols, domain_transform.cpp:51-68);
// OP 1 -> pc[0..H][x] (box_pass_cols :110-116).  One thread per column
// (coalesced across the warp), batches of kColU rows prefetched one batch
// ahead.  grid (ceil(W / 128), slots), block 128.
template <int OP, int SRC>
__global__ void __launch_bounds__(128) k_dt_cols_scan(DtParams p)
{
    const int z = blockIdx.y;
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= p.W) return;
    const SlotSrc q = slot_src<OP>(p, z);
    double* out = OP == 0 ? p.ctv + (size_t)z * p.plane : p.pc + (size_t)z * p.pcplane;
    double acc = OP == 0 ? 1.0 : 0.0, prev = 0.0;
    if (OP == 1) out[x] = 0.0;
    Raw<SRC> cur[kColU], nxt[kColU];
#pragma unroll
    for (int u = 0; u < kColU; ++u)
        if (u < p.H) cur[u] = load_raw<SRC>(q, p.H, p.W, u, x);
    for (int y0 = 0; y0 < p.H; y0 += kColU) {
        if (y0 + kColU < p.H) {
#pragma unroll
            for (int u = 0; u < kColU; ++u)
                if (y0 + kColU + u < p.H) nxt[u] = load_raw<SRC>(q, p.H, p.W, y0 + kColU + u, x);
        }
#pragma unroll
        for (int u = 0; u < kColU; ++u) {
            const int y = y0 + u;
            if (y < p.H) {
                acc = scan_step<OP>(acc, to_val(cur[u], q), prev, y == 0, p.ratio);
                out[(size_t)(OP == 0 ? y : y + 1) * p.W + x] = acc;
            }
        }
#pragma unroll
        for (int u = 0; u < kColU; ++u) cur[u] = nxt[u];
    }
}

// Window + normalized box (box_pass_rows :89-101 / box_pass_cols :117-131):
// one thread per sample.  DIR 0 rows, DIR 1 columns.  FINAL writes the target
// 2v - 1 (from_unit_range_into, pipelines.cpp:25-31) scaled to raw units as
// fp32 into tx / ty; otherwise the double plane x.  grid (ceil(H*W/256), slots).
template <int DIR, bool FINAL>
__global__ void __launch_bounds__(256) k_dt_window(DtParams p, double radius)
{
    const int z = blockIdx.y;
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= p.plane) return;
    const int y = (int)(i / (unsigned)p.W), x = (int)(i - (size_t)y * p.W);
    const double* t;
    const double* pc;
    size_t st, pst;
    int n, k;
    if (DIR == 0) {
        t = p.cth + (size_t)z * p.plane + (size_t)y * p.W;
        pc = p.pc + (size_t)z * p.pcplane + (size_t)y * (p.W + 1);
        st = 1;
        pst = 1;
        n = p.W;
        k = x;
    } else {
        t = p.ctv + (size_t)z * p.plane + x;
        pc = p.pc + (size_t)z * p.pcplane + x;
        st = p.W;
        pst = p.W;
        n = p.H;
        k = y;
    }
    const double tk = t[(size_t)k * st];
    const double tlo = __dsub_rn(tk, radius), thi = __dadd_rn(tk, radius);
    int lo = k, hi = k;
    while (lo > 0 && !(t[(size_t)(lo - 1) * st] < tlo)) --lo;
    while (hi + 1 < n && t[(size_t)(hi + 1) * st] <= thi) ++hi;
    const double inv = __ddiv_rn(1.0, (double)(hi - lo + 1));
    const double v = __dmul_rn(__dsub_rn(pc[(size_t)(hi + 1) * pst], pc[(size_t)lo * pst]), inv);
    if (FINAL) {
        const Slot s = slot_of(p, z);
        double lo_, scale;
        norm_of(p.lohi, s.b, lo_, scale);
        const double range = scale > 0.0 ? __ddiv_rn(1.0, scale) : 1.0;
        const double tgt = __dsub_rn(__dmul_rn(2.0, v), 1.0);
        float* dst = (s.axis == 0 ? p.tx : p.ty) + ((size_t)s.b * p.C + s.c) * p.plane;
        dst[i] = (float)(p.normalized ? tgt : tgt * range);
    } else {
        p.x[(size_t)z * p.plane + i] = v;
    }
}

// gaussian_blur passes (image.cpp:122-157): acc += k[i] * v[clamp] in tap order
__global__ void k_gauss_rows(const float* in, double* tmp, int H, int W, const double* k, int r)
{
    const size_t plane = (size_t)H * W;
    const int c = blockIdx.y;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < plane;
         i += (size_t)gridDim.x * blockDim.x) {
        const int y = (int)(i / (unsigned)W), x = (int)(i - (size_t)y * W);
        const float* row = in + c * plane + (size_t)y * W;
        double acc = 0.0;
        for (int j = -r; j <= r; ++j) {
            const int xi = min(max(x + j, 0), W - 1);
            acc = __dadd_rn(acc, __dmul_rn(k[j + r], (double)row[xi]));
        }
        tmp[c * plane + i] = acc;
    }
}

__global__ void k_gauss_cols(const double* tmp, float* out, int H, int W, const double* k, int r)
{
    const size_t plane = (size_t)H * W;
    const int c = blockIdx.y;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < plane;
         i += (size_t)gridDim.x * blockDim.x) {
        const int y = (int)(i / (unsigned)W), x = (int)(i - (size_t)y * W);
        const double* col = tmp + c * plane + x;
        double acc = 0.0;
        for (int j = -r; j <= r; ++j) {
            const int yi = min(max(y + j, 0), H - 1);
            acc = __dadd_rn(acc, __dmul_rn(k[j + r], col[(size_t)yi * W]));
        }
        out[c * plane + i] = (float)acc;
    }
}

}  // namespace

// domain_transform.cpp:9-17, evaluated on the host exactly as the reference
double nc_box_radius(double sigma_s, int iter, int total)
{
    const double sigma_i =
        sigma_s * std::sqrt(3.0) * std::pow(2.0, total - iter) / std::sqrt(std::pow(4.0, total) - 1.0);
    return std::sqrt(3.0) * sigma_i;
}

int launch_dt_filter(const DtParams& p, int iterations, double sigma_s, cudaStream_t st)
{
    const dim3 grows((unsigned)((p.H + 32 * kScanWarps - 1) / (32 * kScanWarps)), p.slots);
    const dim3 gcols((unsigned)((p.W + 127) / 128), p.slots);
    const dim3 gwin((unsigned)((p.plane + 255) / 256), p.slots);
    int launches = 0;
    k_dt_rows_scan<0, 0><<<grows, 32 * kScanWarps, 0, st>>>(p);
    k_dt_cols_scan<0, 0><<<gcols, 128, 0, st>>>(p);
    launches += 2;
    for (int it = 1; it <= iterations; ++it) {
        const double radius = nc_box_radius(sigma_s, it, iterations);
        if (it == 1)
            k_dt_rows_scan<1, 0><<<grows, 32 * kScanWarps, 0, st>>>(p);
        else
            k_dt_rows_scan<1, 1><<<grows, 32 * kScanWarps, 0, st>>>(p);
        k_dt_window<0, false><<<gwin, 256, 0, st>>>(p, radius);
        k_dt_cols_scan<1, 1><<<gcols, 128, 0, st>>>(p);
        if (it == iterations)
            k_dt_window<1, true><<<gwin, 256, 0, st>>>(p, radius);
        else
            k_dt_window<1, false><<<gwin, 256, 0, st>>>(p, radius);
        launches += 4;
    }
    return cudaGetLastError() == cudaSuccess ? launches : -1;
}

// weights of gaussian_kernel (image.cpp:99-111), host, reference order
std::vector<double> gaussian_weights(double sigma)
{
    const int r = (int)std::ceil(3.0 * sigma);
    std::vector<double> k(2 * r + 1);
    double sum = 0.0;
    for (int i = -r; i <= r; ++i) {
        k[i + r] = std::exp(-(static_cast<double>(i) * i) / (2.0 * sigma * sigma));
        sum += k[i + r];
    }
    for (double& v : k) v /= sum;
    return k;
}

cudaError_t launch_gaussian_blur(const float* in, float* out, double* tmp, const double* k, int r,
                                 int C, int H, int W, int nsm, cudaStream_t st)
{
    const dim3 g((unsigned)(nsm * 4), C);
    k_gauss_rows<<<g, 256, 0, st>>>(in, tmp, H, W, k, r);
    k_gauss_cols<<<g, 256, 0, st>>>(tmp, out, H, W, k, r);
    return cudaGetLastError();
}

}  // namespace blfls
