// k_blf_j8.cu -- shared-grayscale-guide brute-force BLF, eight outputs per
// thread (MODE 2: three image channels filtered with one guide, the joint
// variant of bilateral.cpp:28-77 as filter_gradients calls it per channel
// with the same guide, pipelines.cpp:33-53), one gradient axis per CTA,
// factorised exponents.
//
// What bounds k_blf_j3 (4 outputs per thread) at 0.82 of the MUFU.EX2 rate on
// c5 is shared memory, not the SFU: each source column (guide b + the four
// staged values {g0 B, g1 B}, {g2 B, B}, 20 bytes) is loaded per thread and
// serves at most 4 outputs, so the LDS traffic is 83% of the MUFU time and the
// MIO queue (LDS and MUFU share it) throttles the exponentials.  Here a thread
// owns 8 adjacent outputs of one row: a loaded column serves up to 8 outputs
// (LDS per tap halved, ~46% of the MUFU time), and the per-row partial sums of
// k_blf_j3 are replaced by scaling the loaded sources by the row factor wy
// (2 FMUL2 per column and row), so the 8 x 4 accumulators fit without spills.
//
// Per tap and output: MUFU.EX2 + 2 FFMA2 (numerators {g0, g1}, {g2, z} with
// the weight as broadcast operand) + half an FFMA2 (the exponents of two
// adjacent outputs: e = {2a_q, 2a_q+1} b + {cs|dx|, cs|dx-1|}).  Factorised
// exponent -(a - b)^2 = -a^2 + 2ab - b^2: exp2(-b^2) is folded into the staged
// sources of column t, exp2(-a^2) scales numerator and normaliser of output s
// alike and cancels; valid while 2 range_coef^2 <= 60 (launch_j8), else the
// difference form of k_blf_j3 runs.
//
// Tile: TH rows x 64 columns, 8 threads per row (a quarter-warp per row).
// Shared rows are 16-byte-chunk swizzled so the 8 lanes of a quarter-warp
// (8 columns apart) hit 8 distinct bank groups.
#include <algorithm>
#include <cstdint>

#include "blfls_internal.cuh"

namespace blfls {

#ifdef BLFLS_EXPERIMENTS  // measured slower than k_blf_j3 (see launch_grad_blf_j8)

namespace {

__device__ __forceinline__ float j8_ex2(float x)
{
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// d = {a, a} * b + c (f32x2, the weight as broadcast operand)
__device__ __forceinline__ unsigned long long j8_ffma2(float a, unsigned long long b, unsigned long long c)
{
    unsigned long long aa, d;
    asm("mov.b64 %0, {%1, %1};" : "=l"(aa) : "f"(a));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(aa), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ unsigned long long j8_fmul2(float a, unsigned long long b)
{
    unsigned long long aa, d;
    asm("mov.b64 %0, {%1, %1};" : "=l"(aa) : "f"(a));
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(aa), "l"(b));
    return d;
}
// exp2 of both lanes of an f32x2 pair on the FMA pipe: round-to-nearest
// split x = j + f (|f| <= 1/2) by the 1.5 * 2^23 shifter, degree-5 minimax
// polynomial for 2^f (rel. err 2.3e-7, the coefficients of k_blf.cu
// poly_ex2), 2^j by an exponent-field add.  The factorised exponents are
// within [-2 coef^2 + cs_min, 2 coef^2] subset of [-125, 60], no clamping.
__device__ __forceinline__ float2 j8_poly_ex2x2(unsigned long long x)
{
    unsigned long long t, jj, f, pp, magic, c;
    asm("mov.b64 %0, {%1, %1};" : "=l"(magic) : "f"(12582912.0f));
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(x), "l"(magic));
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(jj) : "l"(t), "l"(magic));
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(f) : "l"(x), "l"(jj));
    asm("mov.b64 %0, {%1, %1};" : "=l"(pp) : "f"(0.001327647129073739f));
    asm("mov.b64 %0, {%1, %1};" : "=l"(c) : "f"(0.009675541892647743f));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(pp) : "l"(pp), "l"(f), "l"(c));
    asm("mov.b64 %0, {%1, %1};" : "=l"(c) : "f"(0.05550713092088699f));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(pp) : "l"(pp), "l"(f), "l"(c));
    asm("mov.b64 %0, {%1, %1};" : "=l"(c) : "f"(0.24022120237350464f));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(pp) : "l"(pp), "l"(f), "l"(c));
    asm("mov.b64 %0, {%1, %1};" : "=l"(c) : "f"(0.6931469440460205f));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(pp) : "l"(pp), "l"(f), "l"(c));
    asm("mov.b64 %0, {%1, %1};" : "=l"(c) : "f"(1.0000001192092896f));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(pp) : "l"(pp), "l"(f), "l"(c));
    float2 tv, pv;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(tv.x), "=f"(tv.y) : "l"(t));
    asm("mov.b64 {%0, %1}, %2;" : "=f"(pv.x), "=f"(pv.y) : "l"(pp));
    return make_float2(__int_as_float(__float_as_int(pv.x) + (__float_as_int(tv.x) << 23)),
                       __int_as_float(__float_as_int(pv.y) + (__float_as_int(tv.y) << 23)));
}
__device__ __forceinline__ unsigned long long j8_pack(float x, float y)
{
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y));
    return r;
}
__device__ __forceinline__ float2 j8_unpack(unsigned long long r)
{
    float2 v;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r));
    return v;
}
// float2 column -> swizzled float2 slot (16-byte chunk k of two columns:
// k ^ ((k >> 3) & 3); lanes 8 columns apart read chunks 4 apart)
__device__ __forceinline__ int j8_ssw(int col)
{
    const int k = col >> 1;
    return ((k ^ ((k >> 3) & 3)) << 1) | (col & 1);
}
// float column -> swizzled float slot (16-byte chunk k of four columns:
// k ^ ((k >> 3) & 1); lanes 8 columns apart read chunks 2 apart)
__device__ __forceinline__ int j8_gsw(int col)
{
    const int k = col >> 2;
    return ((k ^ ((k >> 3) & 1)) << 2) | (col & 3);
}
__device__ __forceinline__ void j8_decode(const uint32_t* lohi, int b, float coef, float& s, float& range)
{
    const float lo = ordered_to_float(lohi[2 * b]);
    const float hi = ordered_to_float(lohi[2 * b + 1]);
    range = hi - lo;
    s = range > 0.f ? coef / range : coef;
}

}  // namespace

template <int R, int TH>
struct J8Geom {
    static constexpr int P = 8, TPR = 8, TW = P * TPR, NT = TPR * TH;
    static constexpr int ROWS = TH + 2 * R;
    static constexpr int COLS = TW + 2 * R;
    static constexpr int VN = P + 2 * R;                 // window columns per thread
    static constexpr int VN4 = (VN + 3) & ~3;            // rounded to column quads
    static constexpr int GP = (COLS + 31) & ~31;         // guide pitch (floats, whole swizzle groups)
    static constexpr int SP = (COLS + 15) & ~15;         // source pitch (float2, whole swizzle groups)
    static_assert((TPR - 1) * P + VN4 <= SP && (TPR - 1) * P + VN4 <= GP, "reads stay inside a row");
    static constexpr size_t smem_bytes()
    {
        return (size_t)ROWS * GP * sizeof(float) + (size_t)2 * ROWS * SP * sizeof(float2);
    }
};

// Stages one tile: this axis' circular gradients (image.cpp:72-95) of guide
// and channels into G / S01 / S2, a warp per tile row and a lane per column,
// by `nworkers` threads (worker = 0 .. nworkers - 1, whole warps).
// Out-of-image cells hold b = 0 and zero sources (weight 0: the clipped
// window, bilateral.cpp:56-57).
template <int R, int TH>
__device__ __forceinline__ void j8_stage(const BlfParams& p, float* G, float2* S01, float2* S2, int b, int axis,
                                         int tx0, int ty0, int worker, int nworkers)
{
    using Gm = J8Geom<R, TH>;
    constexpr int ROWS = Gm::ROWS, COLS = Gm::COLS, GP = Gm::GP, SP = Gm::SP;
    const int H = p.H, W = p.W;
    const size_t plane = (size_t)H * W;
    float sg, grange;
    j8_decode(p.glohi, b, p.range_coef, sg, grange);
    const float* fimg = p.f + (size_t)b * 3 * plane;
    const float* gimg = p.guide + (size_t)b * p.GC * plane;
    const int lane = worker & 31;
    for (int i = worker >> 5; i < ROWS; i += nworkers >> 5) {
        const int y = ty0 - R + i;
        const bool yin = y >= 0 && y < H;
        const int yn = axis == 0 ? y : (y + 1 == H ? 0 : y + 1);
        const size_t r0 = (size_t)(yin ? y : 0) * W, r1 = (size_t)(yin ? yn : 0) * W;
        float* grow = G + i * GP;
        float2* s01 = S01 + i * SP;
        float2* s2 = S2 + i * SP;
#pragma unroll
        for (int j = lane; j < COLS; j += 32) {
            const int x = tx0 - R + j;
            const int o = j8_ssw(j);
            if (yin && x >= 0 && x < W) {
                const int x1 = axis == 0 ? (x + 1 == W ? 0 : x + 1) : x;
                const float bb = (__ldg(gimg + r1 + x1) - __ldg(gimg + r0 + x)) * sg;
                grow[j8_gsw(j)] = bb;
                float g[3];
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const float* fc = fimg + (size_t)c * plane;
                    g[c] = __ldg(fc + r1 + x1) - __ldg(fc + r0 + x);
                }
                const float bw = j8_ex2(-bb * bb);  // exp2(-b^2) of column t
                s01[o] = make_float2(g[0] * bw, g[1] * bw);
                s2[o] = make_float2(g[2] * bw, bw);
            } else {
                grow[j8_gsw(j)] = 0.0f;
                s01[o] = make_float2(0.f, 0.f);
                s2[o] = make_float2(0.f, 0.f);
            }
        }
    }
}

// Filters one staged tile and stores its targets: thread tid in [0, NT)
// owns outputs (ty0 + tid / 8, tx0 + 8 (tid % 8) .. + 7).
// POLYK > 0: every POLYK-th exponent pair runs on the FMA pipe (j8_poly_ex2x2)
template <int R, int TH, int POLYK = 0>
__device__ __forceinline__ void j8_filter(const BlfParams& p, const float* G, const float2* S01, const float2* S2,
                                          int b, int axis, int tx0, int ty0, int tid)
{
    using Gm = J8Geom<R, TH>;
    constexpr int P = Gm::P, TPR = Gm::TPR, VN = Gm::VN, VN4 = Gm::VN4, GP = Gm::GP, SP = Gm::SP;
    const int H = p.H, W = p.W;
    const int tx = tid % TPR, ty = tid / TPR;
    const int ox = tx0 + tx * P, oy = ty0 + ty;
    unsigned long long acc01[P], acc2z[P], gsp[P / 2];
    {
        const float* grow = G + (ty + R) * GP;
#pragma unroll
        for (int h = 0; h < P / 2; ++h) {
            const float a0 = grow[j8_gsw(tx * P + 2 * h + R)], a1 = grow[j8_gsw(tx * P + 2 * h + 1 + R)];
            gsp[h] = j8_pack(2.0f * a0, 2.0f * a1);
        }
#pragma unroll
        for (int q = 0; q < P; ++q) {
            acc01[q] = 0ull;
            acc2z[q] = 0ull;
        }
    }
#pragma unroll 1
    for (int dy = -R; dy <= R; ++dy) {
        const float wy = p.wrow[dy < 0 ? -dy : dy];
        const float* grow = G + (ty + R + dy) * GP;
        const float2* s01 = S01 + (ty + R + dy) * SP;
        const float2* s2 = S2 + (ty + R + dy) * SP;
#pragma unroll
        for (int j4 = 0; j4 < VN4; j4 += 4) {
            const float4 g4 = *reinterpret_cast<const float4*>(grow + j8_gsw(tx * P + j4));
            const float gt[4] = {g4.x, g4.y, g4.z, g4.w};
            unsigned long long v01[4], v2z[4];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int pc = j8_ssw(tx * P + j4 + 2 * h);
                const float4 a = *reinterpret_cast<const float4*>(s01 + pc);
                const float4 c = *reinterpret_cast<const float4*>(s2 + pc);
                // the row factor exp2(cs[|dy|]) on the sources, once per column
                v01[2 * h] = j8_fmul2(wy, j8_pack(a.x, a.y));
                v01[2 * h + 1] = j8_fmul2(wy, j8_pack(a.z, a.w));
                v2z[2 * h] = j8_fmul2(wy, j8_pack(c.x, c.y));
                v2z[2 * h + 1] = j8_fmul2(wy, j8_pack(c.z, c.w));
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int j = j4 + u;
                if (j >= VN) break;
#pragma unroll
                for (int h = 0; h < P / 2; ++h) {
                    const int q0 = 2 * h, dx0 = j - q0 - R;
                    const bool ok0 = dx0 >= -R && dx0 <= R, ok1 = dx0 - 1 >= -R && dx0 - 1 <= R;
                    if (!ok0 && !ok1) continue;
                    unsigned long long gtt, ce, e;
                    asm("mov.b64 %0, {%1, %1};" : "=l"(gtt) : "f"(gt[u]));
                    asm("mov.b64 %0, {%1, %2};" : "=l"(ce) : "f"(p.cep[dx0 + R].x), "f"(p.cep[dx0 + R].y));
                    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(e) : "l"(gtt), "l"(gsp[h]), "l"(ce));
                    const bool poly = POLYK > 0 && ok0 && ok1 && (j * (P / 2) + h) % (POLYK > 0 ? POLYK : 1) ==
                                                                 (POLYK > 0 ? POLYK - 1 : 0);
                    float2 ww;
                    if (poly) {
                        ww = j8_poly_ex2x2(e);
                    } else {
                        const float2 ee = j8_unpack(e);
                        ww.x = ok0 ? j8_ex2(ee.x) : 0.f;
                        ww.y = ok1 ? j8_ex2(ee.y) : 0.f;
                    }
                    if (ok0) {
                        acc01[q0] = j8_ffma2(ww.x, v01[u], acc01[q0]);
                        acc2z[q0] = j8_ffma2(ww.x, v2z[u], acc2z[q0]);
                    }
                    if (ok1) {
                        acc01[q0 + 1] = j8_ffma2(ww.y, v01[u], acc01[q0 + 1]);
                        acc2z[q0 + 1] = j8_ffma2(ww.y, v2z[u], acc2z[q0 + 1]);
                    }
                }
            }
        }
    }

    // ---- epilogue: T = num / z per channel (z >= the centre weight > 0)
    if (oy < p.y1) {
        float s, range;
        j8_decode(p.lohi, b, p.range_coef, s, range);
        const float oscale = (p.normalized_out && range > 0.f) ? 1.f / range : 1.f;
        float* dst = axis == 0 ? p.tx : p.ty;
        const size_t pl = (size_t)p.out_rows * W;
        const size_t orow = (size_t)(oy - (p.out_rows == H ? 0 : p.y0)) * W;
        float t[3][P];
#pragma unroll
        for (int q = 0; q < P; ++q) {
            const float2 n01 = j8_unpack(acc01[q]);
            const float2 n2z = j8_unpack(acc2z[q]);
            const float inv = oscale / n2z.y;
            t[0][q] = n01.x * inv;
            t[1][q] = n01.y * inv;
            t[2][q] = n2z.x * inv;
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const size_t off = ((size_t)b * 3 + c) * pl + orow + ox;
            if (ox + P <= W && (off & 3) == 0) {
                *reinterpret_cast<float4*>(dst + off) = make_float4(t[c][0], t[c][1], t[c][2], t[c][3]);
                *reinterpret_cast<float4*>(dst + off + 4) = make_float4(t[c][4], t[c][5], t[c][6], t[c][7]);
            } else {
#pragma unroll
                for (int q = 0; q < P; ++q)
                    if (ox + q < W) dst[off + q] = t[c][q];
            }
        }
    }
}

// One CTA per tile: every thread stages, then filters.
template <int R, int TH, int MINB, int POLYK>
__global__ void __launch_bounds__(8 * TH, MINB) k_blf_j8(const BlfParams p)
{
    using Gm = J8Geom<R, TH>;
    extern __shared__ __align__(16) float smj8[];
    float* G = smj8;                                                        // [ROWS][GP] scaled guide b
    float2* S01 = reinterpret_cast<float2*>(smj8 + Gm::ROWS * Gm::GP);      // [ROWS][SP] {g0 B, g1 B}
    float2* S2 = S01 + Gm::ROWS * Gm::SP;                                   // [ROWS][SP] {g2 B, B}
    const int b = blockIdx.z >> 1, axis = blockIdx.z & 1;
    const int tx0 = blockIdx.x * Gm::TW, ty0 = p.y0 + blockIdx.y * TH;
    j8_stage<R, TH>(p, G, S01, S2, b, axis, tx0, ty0, threadIdx.x, Gm::NT);
    __syncthreads();
    j8_filter<R, TH, POLYK>(p, G, S01, S2, b, axis, tx0, ty0, threadIdx.x);
}

// Persistent, warp-specialised: NT filter threads (warps 0 .. NT/32 - 1) and
// NT staging threads (the other half) per CTA, two staged-tile buffers.  The
// stagers fill buffer k & 1 with tile k (global loads, gradients, exp2(-b^2))
// while the filter warps work on tile k - 1, so the filter warps never wait
// on global memory (in k_blf_j8 / k_blf_j3 the staging loads are the top
// warp stall, and all CTAs of an SM can be staging at once).  Handshake by
// named barriers (bar.arrive / bar.sync over all 2 NT threads): FULL[s] (1,
// 2) stagers -> filter, EMPTY[s] (3, 4) filter -> stagers.  Tiles in the
// order of k_blf_j8's grid (tile column, tile row, image x axis).
template <int R, int TH>
__global__ void __launch_bounds__(16 * TH, 2) k_blf_j8p(const BlfParams p, int ntx, int nty, int total)
{
    using Gm = J8Geom<R, TH>;
    constexpr int NT = Gm::NT;
    constexpr int BUF = Gm::ROWS * Gm::GP + 2 * 2 * Gm::ROWS * Gm::SP;  // floats per buffer
    extern __shared__ __align__(16) float smj8[];
    const int ntiles = total > (int)blockIdx.x ? (total - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    auto decode = [&](int t, int& b, int& axis, int& tx0, int& ty0) {
        const int cx = t % ntx, r = t / ntx, cy = r % nty, z = r / nty;
        b = z >> 1;
        axis = z & 1;
        tx0 = cx * Gm::TW;
        ty0 = p.y0 + cy * TH;
    };
    auto bufs = [&](int s, float*& G, float2*& S01, float2*& S2) {
        G = smj8 + s * BUF;
        S01 = reinterpret_cast<float2*>(G + Gm::ROWS * Gm::GP);
        S2 = S01 + Gm::ROWS * Gm::SP;
    };
    if ((int)threadIdx.x >= NT) {
        // stagers
        const int w = threadIdx.x - NT;
        for (int k = 0; k < ntiles; ++k) {
            const int s = k & 1;
            if (k >= 2) asm volatile("bar.sync %0, %1;" ::"r"(3 + s), "r"(2 * NT) : "memory");
            int b, axis, tx0, ty0;
            decode(blockIdx.x + k * gridDim.x, b, axis, tx0, ty0);
            float* G;
            float2 *S01, *S2;
            bufs(s, G, S01, S2);
            j8_stage<R, TH>(p, G, S01, S2, b, axis, tx0, ty0, w, NT);
            asm volatile("bar.arrive %0, %1;" ::"r"(1 + s), "r"(2 * NT) : "memory");
        }
    } else {
        // filter warps
        for (int k = 0; k < ntiles; ++k) {
            const int s = k & 1;
            asm volatile("bar.sync %0, %1;" ::"r"(1 + s), "r"(2 * NT) : "memory");
            int b, axis, tx0, ty0;
            decode(blockIdx.x + k * gridDim.x, b, axis, tx0, ty0);
            float* G;
            float2 *S01, *S2;
            bufs(s, G, S01, S2);
            j8_filter<R, TH>(p, G, S01, S2, b, axis, tx0, ty0, threadIdx.x);
            // the stagers wait for this buffer only before tile k + 2
            if (k + 2 < ntiles) asm volatile("bar.arrive %0, %1;" ::"r"(3 + s), "r"(2 * NT) : "memory");
        }
    }
}

template <int R, int TH, int MINB, int POLYK = 0>
static cudaError_t launch_j8_t(const BlfParams& p, int batch, cudaStream_t st)
{
    using Gm = J8Geom<R, TH>;
    constexpr size_t smem = Gm::smem_bytes();
    cudaError_t e = cudaFuncSetAttribute(k_blf_j8<R, TH, MINB, POLYK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    dim3 grid((p.W + Gm::TW - 1) / Gm::TW, (p.y1 - p.y0 + TH - 1) / TH, 2 * batch);
    k_blf_j8<R, TH, MINB, POLYK><<<grid, Gm::NT, smem, st>>>(p);
    return cudaGetLastError();
}

template <int R, int TH>
static cudaError_t launch_j8p_t(const BlfParams& p, int batch, int ctas_per_sm, cudaStream_t st)
{
    using Gm = J8Geom<R, TH>;
    constexpr size_t smem = 2 * Gm::smem_bytes();
    cudaError_t e = cudaFuncSetAttribute(k_blf_j8p<R, TH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const int ntx = (p.W + Gm::TW - 1) / Gm::TW, nty = (p.y1 - p.y0 + TH - 1) / TH;
    const long total = (long)ntx * nty * 2 * batch;
    if (total > INT32_MAX) return cudaErrorInvalidValue;
    const int grid = (int)std::min<long>(total, (long)ctas_per_sm * nsm);
    k_blf_j8p<R, TH><<<grid, 2 * Gm::NT, smem, st>>>(p, ntx, nty, (int)total);
    return cudaGetLastError();
}

// Shared-gray-guide filter with 8 outputs per thread: factorised exponents
// only (2 range_coef^2 <= 60) and no peer-storing epilogue; false otherwise
// (the caller runs k_blf_j3).  Experiments build only: on c5 (r02 B200,
// tools/ab_j8.sh) it measured 0.765 of the MUFU rate against k_blf_j3's
// 0.820 -- the LDS traffic halves (L1 48% vs 80% of peak) but 128 registers
// and 50 KB per 4-warp CTA leave 16 warps per SM, and the tile staging
// (global-load latency, 17% of the stall samples) is no longer hidden;
// 24 / 32-row tiles 0.81 / 0.80, every 4th..12th exponent pair on the FMA
// pipe 0.715..0.76, the persistent warp-specialised variant (stager warps
// fill the next tile while filter warps work) 0.65 at 8 filter warps per SM.
bool launch_grad_blf_j8(const BlfParams& p, int batch, cudaStream_t st, cudaError_t* err)
{
    static const int enabled = knob("BLFLS_J8", 0);
    static const int th = knob("BLFLS_J8_TH", 16);
    static const int persistent = knob("BLFLS_J8P", 0);
    static const int polyk = knob("BLFLS_J8_POLY", 0);
    if (!enabled || p.C != 3 || p.npeers > 0 || !(2.0f * p.range_coef * p.range_coef <= 60.0f)) return false;
#ifdef BLFLS_EXPERIMENTS
    if (persistent && p.radius == 7) {
        *err = launch_j8p_t<7, 16>(p, batch, 2, st);
        return true;
    }
    if (p.radius == 7 && polyk) {
        switch (polyk) {
            case 4: *err = th == 24 ? launch_j8_t<7, 24, 3, 4>(p, batch, st) : launch_j8_t<7, 16, 4, 4>(p, batch, st); return true;
            case 6: *err = th == 24 ? launch_j8_t<7, 24, 3, 6>(p, batch, st) : launch_j8_t<7, 16, 4, 6>(p, batch, st); return true;
            case 8: *err = th == 24 ? launch_j8_t<7, 24, 3, 8>(p, batch, st) : launch_j8_t<7, 16, 4, 8>(p, batch, st); return true;
            default: *err = th == 24 ? launch_j8_t<7, 24, 3, 12>(p, batch, st) : launch_j8_t<7, 16, 4, 12>(p, batch, st); return true;
        }
    }
#endif
    switch (p.radius) {
        case 7:
#ifdef BLFLS_EXPERIMENTS
            if (th == 24) { *err = launch_j8_t<7, 24, 3>(p, batch, st); return true; }
            if (th == 32) { *err = launch_j8_t<7, 32, 2>(p, batch, st); return true; }
#endif
            *err = launch_j8_t<7, 16, 4>(p, batch, st);
            return true;
        case 5: *err = launch_j8_t<5, 16, 4>(p, batch, st); return true;
        case 3: *err = launch_j8_t<3, 16, 4>(p, batch, st); return true;
        default: return false;
    }
    (void)th;
    (void)persistent;
    (void)polyk;
}

#else
bool launch_grad_blf_j8(const BlfParams&, int, cudaStream_t, cudaError_t*) { return false; }
#endif  // BLFLS_EXPERIMENTS

}  // namespace blfls
