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
//   k_dt_prep                                   src01 -> x, guide01 -> g01 (double)
//   k_dt_rows_scan<CT>, k_dt_cols_scan<CT>      warped coordinates ct_h, ct_v
//   T x { k_dt_rows_scan<PREFIX>, k_dt_window<ROWS>,
//         k_dt_cols_scan<PREFIX>, k_dt_window<COLS> }  (the last writes T = 2v-1)
// The scans are sequential per line with only H or W lines per slot, so they
// would be latency-bound on loads: each warp streams its 32 lines through a
// kStages-deep cp.async ring of 32 x 32 double tiles, so only the dependent
// double additions of the recurrence remain on the critical path.
#include <cmath>
#include <vector>

#include "blfls_internal.cuh"
#include "slot_common.cuh"

namespace blfls {

namespace {

constexpr int kStages = 6;  // cp.async ring depth of the scans

// src01 / guide01 planes of every slot in double (the prep step of each smooth
// call): x <- src01 (the first pass's signal), g01 <- guide01.  Fully
// parallel; the scans that follow then stream double planes only.
// grid (blocks, slots), block 256.
__global__ void __launch_bounds__(256) k_dt_prep(DtParams p)
{
    const int z = blockIdx.y;
    const Slot s = slot_of(p, z);
    const float *src, *gde;
    double slo, ssc, glo, gsc;
    slot_images(p, s, src, gde, slo, ssc, glo, gsc);
    double* xz = p.x + (size_t)z * p.plane;
    double* gz = p.g01 + (size_t)z * p.plane;
    for (int y = blockIdx.x; y < p.H; y += gridDim.x)
        for (int x = threadIdx.x; x < p.W; x += blockDim.x) {
            const size_t i = (size_t)y * p.W + x;
            xz[i] = grad01(src, p.H, p.W, y, x, s.axis, slo, ssc);
            gz[i] = grad01(gde, p.H, p.W, y, x, s.axis, glo, gsc);
        }
}

__device__ __forceinline__ void cp_async8(void* dst, const void* src)
{
    const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

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

constexpr int kLPW = 8;    // scan lines per warp (more warps in flight; the chain is per lane)
constexpr int kScanCta = 4;  // warps per scan CTA

// Row scans: OP 0 -> ct_h from g01 (transform_rows, domain_transform.cpp:31-49);
// OP 1 -> pc[y][0..W] from x (box_pass_rows :81-88).  One warp per kLPW rows;
// kLPW x 32 chunks stream through a kStages-deep cp.async ring stored
// transposed ([column][row]), so each scanning lane reads its own row
// conflict-free; results overwrite the chunk in place and leave as coalesced
// row stores.  grid (ceil(H / (kLPW * kScanCta)), slots), block 32 * kScanCta.
template <int OP>
__global__ void __launch_bounds__(32 * kScanCta) k_dt_rows_scan(DtParams p)
{
    constexpr int S = kStages - 1;  // 4 warps x 5 stages: under the 48 KB static limit
    __shared__ double ring[kScanCta][S][32][kLPW + 1];
    const int z = blockIdx.y, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int y0 = (blockIdx.x * kScanCta + warp) * kLPW;
    if (y0 >= p.H) return;
    const int nr = min(kLPW, p.H - y0), W = p.W;
    const double* in = (OP == 0 ? p.g01 : p.x) + (size_t)z * p.plane;
    double* ctz = p.cth + (size_t)z * p.plane;
    double* pcz = p.pc + (size_t)z * p.pcplane;
    double (*rg)[32][kLPW + 1] = ring[warp];
    const int nch = (W + 31) / 32;
    auto issue = [&](int ch) {
        if (ch < nch) {
            const int x = ch * 32 + lane;
            if (x < W)
#pragma unroll
                for (int r = 0; r < kLPW; ++r)
                    if (r < nr) cp_async8(&rg[ch % S][lane][r], in + (size_t)(y0 + r) * W + x);
        }
        cp_async_commit();
    };
#pragma unroll
    for (int s = 0; s < S - 1; ++s) issue(s);
    double acc = OP == 0 ? 1.0 : 0.0, prev = 0.0;
    if (OP == 1 && lane < nr) pcz[(size_t)(y0 + lane) * (W + 1)] = 0.0;
    for (int ch = 0; ch < nch; ++ch) {
        issue(ch + S - 1);
        cp_async_wait<S - 1>();
        __syncwarp();
        const int x0 = ch * 32, nc = min(32, W - x0);
        double (*t)[kLPW + 1] = rg[ch % S];
        if (lane < nr) {
            if (nc == 32) {
#pragma unroll 8
                for (int c = 0; c < 32; ++c) {
                    acc = scan_step<OP>(acc, t[c][lane], prev, x0 + c == 0, p.ratio);
                    t[c][lane] = acc;
                }
            } else {
                for (int c = 0; c < nc; ++c) {
                    acc = scan_step<OP>(acc, t[c][lane], prev, x0 + c == 0, p.ratio);
                    t[c][lane] = acc;
                }
            }
        }
        __syncwarp();
        if (lane < nc) {
#pragma unroll
            for (int r = 0; r < kLPW; ++r) {
                if (r < nr) {
                    if (OP == 0)
                        ctz[(size_t)(y0 + r) * W + x0 + lane] = t[lane][r];
                    else
                        pcz[(size_t)(y0 + r) * (W + 1) + x0 + lane + 1] = t[lane][r];
                }
            }
        }
        __syncwarp();
    }
}

// Column scans: OP 0 -> ct_v from g01 (transform_cols, domain_transform.cpp:51-68);
// OP 1 -> pc[0..H][x] from x (box_pass_cols :110-116).  One warp per kLPW
// columns: 32-row chunks stream through the cp.async ring ([row][column],
// each row segment one 64 B copy group); lane c < kLPW scans column c.
// grid (ceil(W / (kLPW * kScanCta)), slots), block 32 * kScanCta.
template <int OP>
__global__ void __launch_bounds__(32 * kScanCta) k_dt_cols_scan(DtParams p)
{
    __shared__ double ring[kScanCta][kStages][32][kLPW];
    const int z = blockIdx.y, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int x0 = (blockIdx.x * kScanCta + warp) * kLPW;
    if (x0 >= p.W) return;
    const int H = p.W > 0 ? p.H : 0, W = p.W;
    const int ncol = min(kLPW, W - x0);
    const double* in = (OP == 0 ? p.g01 : p.x) + (size_t)z * p.plane;
    double* out = OP == 0 ? p.ctv + (size_t)z * p.plane : p.pc + (size_t)z * p.pcplane;
    double (*rg)[32][kLPW] = ring[warp];
    const int nch = (H + 31) / 32;
    // lane -> (row u0 + 4 j, column cc) of a chunk: 4 rows x 8 columns per pass
    const int cc = lane % kLPW, u0 = lane / kLPW;
    auto issue = [&](int ch) {
        if (ch < nch && cc < ncol) {
            const int ny = min(32, H - ch * 32);
#pragma unroll
            for (int j = 0; j < 32 / (32 / kLPW); ++j) {
                const int u = u0 + j * (32 / kLPW);
                if (u < ny) cp_async8(&rg[ch % kStages][u][cc], in + (size_t)(ch * 32 + u) * W + x0 + cc);
            }
        }
        cp_async_commit();
    };
#pragma unroll
    for (int s = 0; s < kStages - 1; ++s) issue(s);
    double acc = OP == 0 ? 1.0 : 0.0, prev = 0.0;
    const bool scans = lane < ncol;
    if (OP == 1 && scans) out[x0 + lane] = 0.0;
    for (int ch = 0; ch < nch; ++ch) {
        issue(ch + kStages - 1);
        cp_async_wait<kStages - 1>();
        __syncwarp();
        const int ny = min(32, H - ch * 32);
        double (*t)[kLPW] = rg[ch % kStages];
        if (scans) {
            for (int u = 0; u < ny; ++u) {
                acc = scan_step<OP>(acc, t[u][lane], prev, ch * 32 + u == 0, p.ratio);
                t[u][lane] = acc;
            }
        }
        __syncwarp();
        if (cc < ncol) {
#pragma unroll
            for (int j = 0; j < 32 / (32 / kLPW); ++j) {
                const int u = u0 + j * (32 / kLPW);
                if (u < ny) {
                    const int y = ch * 32 + u;
                    out[(size_t)(OP == 0 ? y : y + 1) * W + x0 + cc] = t[u][cc];
                }
            }
        }
        __syncwarp();
    }
}

// Window + normalized box (box_pass_rows :89-101 / box_pass_cols :117-131).
// The reference's two pointers end at lo = lower_bound(ct, ct[k] - r) and
// hi = upper_bound(ct, ct[k] + r) - 1; with ct steps >= 1 both lie within
// fl = floor(r) + 1 of k.  A CTA stages the ct and prefix-sum segments of its
// tile plus an fl halo along the scan direction in shared memory (one
// coalesced round trip).  Each thread then produces kKPT consecutive samples
// of one line: a bounded binary search seeds (lo, hi) at its first sample and
// the reference's own monotone two-pointer advance does the rest (about one
// probe per sample); 1 / (hi - lo + 1) comes from a shared table of exact
// reciprocals.  DIR 0 rows (CTA = 4 rows x 256 samples, a warp per row),
// DIR 1 columns (CTA = 32 columns x 32 rows).  FINAL writes the target
// 2v - 1 (from_unit_range_into, pipelines.cpp:25-31) scaled to raw units as
// fp32 into tx / ty; otherwise the double plane x.
constexpr int kKPT = 8;        // samples per thread
constexpr int kWinRow = 256;   // DIR 0: samples per row segment (32 lanes x kKPT)
constexpr int kWinRowsPerCta = 4;
constexpr int kWinCols = 32;   // DIR 1: columns per CTA
constexpr int kWinRows = 32;   // DIR 1: rows per CTA (8 groups x 4 samples)
constexpr int kKPTc = 4;

// staged index of sample a of line l: rows pad one double every 8 (lanes
// read samples 8 apart: at most 2-way bank conflicts), columns interleave lines
template <int DIR>
__device__ __forceinline__ int sidx(int a, int lines, int l)
{
    return DIR == 0 ? a + (a >> 3) : a * lines + l;
}

template <int DIR>
__device__ __forceinline__ void window_run(const double* st, const double* sp, const double* inv,
                                           int lines, int l, int a0, int k, int cnt, int n, int fl,
                                           double radius, double* vout)
{
    // seed at k: bounded binary searches (the window lies within fl of k)
    const int kk = k - a0;
    double tk = st[sidx<DIR>(kk, lines, l)];
    double tlo = __dsub_rn(tk, radius), thi = __dadd_rn(tk, radius);
    int first = max(0, k - fl) - a0, count = kk - first;
    while (count > 0) {
        const int step = count >> 1, it = first + step;
        if (st[sidx<DIR>(it, lines, l)] < tlo) {
            first = it + 1;
            count -= step + 1;
        } else {
            count = step;
        }
    }
    int lo = first;
    first = kk + 1;
    count = min(n - 1, k + fl) - a0 - kk;
    while (count > 0) {
        const int step = count >> 1, it = first + step;
        if (st[sidx<DIR>(it, lines, l)] <= thi) {
            first = it + 1;
            count -= step + 1;
        } else {
            count = step;
        }
    }
    int hi = first - 1;
    const int nmax = n - 1 - a0;
    for (int j = 0; j < cnt; ++j) {
        const int kj = kk + j;
        if (j > 0) {  // box_pass_*: advance the two pointers
            tk = st[sidx<DIR>(kj, lines, l)];
            tlo = __dsub_rn(tk, radius);
            thi = __dadd_rn(tk, radius);
            while (st[sidx<DIR>(lo, lines, l)] < tlo) ++lo;
            if (hi < kj) hi = kj;
            while (hi < nmax && st[sidx<DIR>((hi + 1), lines, l)] <= thi) ++hi;
        }
        vout[j] = __dmul_rn(__dsub_rn(sp[sidx<DIR>((hi + 1), lines, l)], sp[sidx<DIR>(lo, lines, l)]), inv[hi - lo + 1]);
    }
}

template <int DIR, bool FINAL>
__global__ void __launch_bounds__(DIR == 0 ? 32 * kWinRowsPerCta : 256) k_dt_window(DtParams p, double radius, int fl)
{
    extern __shared__ double wsm[];
    const int z = blockIdx.z;
    const int n = DIR == 0 ? p.W : p.H;
    constexpr int lines = DIR == 0 ? 1 : kWinCols;
    constexpr int nkt = DIR == 0 ? kWinRow : kWinRows;
    const int k0 = blockIdx.x * nkt;
    const int nk = min(nkt, n - k0);
    const int a0 = max(0, k0 - fl), a1 = min(n, k0 + nk + fl + 1);  // staged [a0, a1)
    const int na = a1 - a0;
    // per-line staging capacity (>= na + 1; rows add the 1-in-8 padding)
    const int span = DIR == 0 ? (nkt + 2 * fl + 2) * 9 / 8 + 2 : nkt + 2 * fl + 2;
    double* inv = wsm;                  // [2 fl + 3]
    double* base = wsm + 2 * fl + 3;
    const int tid = threadIdx.x;
    for (int c = tid; c < 2 * fl + 3; c += blockDim.x) inv[c] = c ? __ddiv_rn(1.0, (double)c) : 0.0;
    if (DIR == 0) {
        // warp w: row line0 + w; staging per warp [ct span][pc span]
        const int w = tid >> 5, lane = tid & 31;
        const int y = blockIdx.y * kWinRowsPerCta + w;
        double* st = base + (size_t)w * 2 * span;
        double* sp = st + span;
        const bool row_ok = y < p.H;
        if (row_ok) {
            const double* ct = p.cth + (size_t)z * p.plane + (size_t)y * p.W;
            const double* pc = p.pc + (size_t)z * p.pcplane + (size_t)y * (p.W + 1);
            for (int a = lane; a <= na; a += 32) {
                if (a < na) st[sidx<0>(a, 1, 0)] = ct[a0 + a];
                sp[sidx<0>(a, 1, 0)] = pc[a0 + a];
            }
        }
        __syncthreads();
        if (!row_ok) return;
        double v[kKPT];
        const int kb = k0 + lane * kKPT;
        const int cnt = min(kKPT, k0 + nk - kb);
        if (cnt > 0) window_run<0>(st, sp, inv, 1, 0, a0, kb, cnt, n, fl, radius, v);
        __syncwarp();
        // stage the outputs through the (consumed) ct segment for coalesced stores
        double* so = st;
        __syncwarp();
        for (int j = 0; j < cnt; ++j) so[sidx<0>(lane * kKPT + j, 1, 0)] = v[j];
        __syncwarp();
        const size_t row = (size_t)y * p.W;
        if (FINAL) {
            const Slot s = slot_of(p, z);
            double lo_, scale;
            norm_of(p.lohi, s.b, lo_, scale);
            const double mult = p.normalized ? 1.0 : (scale > 0.0 ? __ddiv_rn(1.0, scale) : 1.0);
            float* dst = (s.axis == 0 ? p.tx : p.ty) + ((size_t)s.b * p.C + s.c) * p.plane;
            for (int i = lane; i < nk; i += 32)
                dst[row + k0 + i] =
                    (float)__dmul_rn(__dsub_rn(__dmul_rn(2.0, so[sidx<0>(i, 1, 0)]), 1.0), mult);
        } else {
            double* xz = p.x + (size_t)z * p.plane;
            for (int i = lane; i < nk; i += 32) xz[row + k0 + i] = so[sidx<0>(i, 1, 0)];
        }
    } else {
        const int line0 = blockIdx.y * kWinCols;
        const int nl = min(kWinCols, p.W - line0);
        double* st = base;                    // [na][lines]
        double* sp = base + (size_t)span * lines;  // [na + 1][lines]
        const double* ct = p.ctv + (size_t)z * p.plane + line0;
        const double* pc = p.pc + (size_t)z * p.pcplane + line0;
        for (int i = tid; i < (na + 1) * lines; i += blockDim.x) {
            const int a = i / lines, l = i - a * lines;
            if (l < nl) {
                if (a < na) st[i] = ct[(size_t)(a0 + a) * p.W + l];
                sp[i] = pc[(size_t)(a0 + a) * p.W + l];
            }
        }
        __syncthreads();
        const int l = tid % kWinCols, g = tid / kWinCols;
        if (l >= nl) return;
        const int kb = k0 + g * kKPTc;
        const int cnt = min(kKPTc, k0 + nk - kb);
        if (cnt <= 0) return;
        double v[kKPTc];
        window_run<1>(st, sp, inv, lines, l, a0, kb, cnt, n, fl, radius, v);
        const int x = line0 + l;
        if (FINAL) {
            const Slot s = slot_of(p, z);
            double lo_, scale;
            norm_of(p.lohi, s.b, lo_, scale);
            const double mult = p.normalized ? 1.0 : (scale > 0.0 ? __ddiv_rn(1.0, scale) : 1.0);
            float* dst = (s.axis == 0 ? p.tx : p.ty) + ((size_t)s.b * p.C + s.c) * p.plane;
            for (int j = 0; j < cnt; ++j)
                dst[(size_t)(kb + j) * p.W + x] = (float)__dmul_rn(__dsub_rn(__dmul_rn(2.0, v[j]), 1.0), mult);
        } else {
            double* xz = p.x + (size_t)z * p.plane;
            for (int j = 0; j < cnt; ++j) xz[(size_t)(kb + j) * p.W + x] = v[j];
        }
    }
}

size_t dt_window_smem(int dir, int fl)
{
    const int span = dir == 0 ? (kWinRow + 2 * fl + 2) * 9 / 8 + 2 : kWinRows + 2 * fl + 2;
    const size_t per = dir == 0 ? (size_t)kWinRowsPerCta * 2 * span : (size_t)2 * span * kWinCols;
    return sizeof(double) * (per + 2 * fl + 3);
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

// Opt the window kernels into the shared memory of the widest (first) DT
// iteration; called once per plan, outside any stream capture.  Returns false
// when the window tile does not fit in shared memory.
bool dt_configure(int iterations, double sigma_s)
{
    const int fl = (int)std::floor(nc_box_radius(sigma_s, 1, iterations)) + 1;
    const size_t s0 = dt_window_smem(0, fl), s1 = dt_window_smem(1, fl);
    if (s1 > 227 * 1024 || s0 > 227 * 1024) return false;
    if (s0 > 48 * 1024)
        cudaFuncSetAttribute(k_dt_window<0, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s0);
    if (s1 > 48 * 1024) {
        cudaFuncSetAttribute(k_dt_window<1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s1);
        cudaFuncSetAttribute(k_dt_window<1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s1);
    }
    return cudaGetLastError() == cudaSuccess;
}

int launch_dt_filter(const DtParams& p, int iterations, double sigma_s, int nsm, cudaStream_t st)
{
    const dim3 gprep((unsigned)std::min(p.H, nsm * 2), p.slots);
    const dim3 grows((unsigned)((p.H + kLPW * kScanCta - 1) / (kLPW * kScanCta)), p.slots);
    const dim3 gcols((unsigned)((p.W + kLPW * kScanCta - 1) / (kLPW * kScanCta)), p.slots);
    const dim3 gw0((unsigned)((p.W + kWinRow - 1) / kWinRow),
                   (p.H + kWinRowsPerCta - 1) / kWinRowsPerCta, p.slots);
    const dim3 gw1((unsigned)((p.H + kWinRows - 1) / kWinRows), (p.W + kWinCols - 1) / kWinCols,
                   p.slots);
    k_dt_prep<<<gprep, 256, 0, st>>>(p);
    k_dt_rows_scan<0><<<grows, 32 * kScanCta, 0, st>>>(p);
    k_dt_cols_scan<0><<<gcols, 32 * kScanCta, 0, st>>>(p);
    int launches = 3;
    for (int it = 1; it <= iterations; ++it) {
        const double radius = nc_box_radius(sigma_s, it, iterations);
        const int fl = (int)std::floor(radius) + 1;  // window half-width bound (+1 margin)
        const size_t s0 = dt_window_smem(0, fl), s1 = dt_window_smem(1, fl);  // <= dt_configure's
        k_dt_rows_scan<1><<<grows, 32 * kScanCta, 0, st>>>(p);
        k_dt_window<0, false><<<gw0, 32 * kWinRowsPerCta, s0, st>>>(p, radius, fl);
        k_dt_cols_scan<1><<<gcols, 32 * kScanCta, 0, st>>>(p);
        if (it == iterations)
            k_dt_window<1, true><<<gw1, 256, s1, st>>>(p, radius, fl);
        else
            k_dt_window<1, false><<<gw1, 256, s1, st>>>(p, radius, fl);
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
