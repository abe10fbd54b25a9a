// k_blf_j3.cu -- shared-grayscale-guide brute-force BLF (MODE 2: three image
// channels filtered with one guide, the joint variant of bilateral.cpp:28-77
// as filter_gradients calls it per channel with the same guide,
// pipelines.cpp:33-53), one gradient axis per CTA.
//
// One exponential per tap serves the three channels; the four sums it feeds
// (three numerators and the normaliser) are updated by two packed FFMA2
// (sm_100 f32x2 with the weight as a broadcast scalar operand): the sources
// are interleaved in shared memory as {g0, g1} and {g2, 1}.  Per tap:
//   FADD (guide difference), FFMA (exponent: cs[|dy|] + cs[|dx|] - d^2),
//   MUFU.EX2, 2 x FFMA2
// against FADD, FFMA, MUFU.EX2, FADD, 3 x FFMA in k_grad_blf<MODE 2>, which
// is issue-bound at ~8.8 instructions per MUFU.EX2.  The window is streamed
// column by column (LDS.128 = two columns of one interleaved array) instead
// of being held in registers, so the kernel stays at 4 CTAs per SM; the
// interleaved rows are chunk-swizzled (j3_sw) so the LDS.128 are conflict-free.
#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "blfls_internal.cuh"

namespace blfls {

namespace {

constexpr float kJ3Sentinel = 1.0e15f;

__device__ __forceinline__ float j3_ex2(float x)
{
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// d.xy = {a, a} * b.xy + c.xy
__device__ __forceinline__ unsigned long long j3_ffma2(float a, unsigned long long b, unsigned long long c)
{
    unsigned long long aa, d;
    asm("mov.b64 %0, {%1, %1};" : "=l"(aa) : "f"(a));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(aa), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ float2 j3_unpack(unsigned long long r)
{
    float2 v;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r));
    return v;
}
// exp2 of both lanes of an f32x2 pair on the FMA pipe (XF exponents lie in
// [-2 coef^2 + cs_min, 2 coef^2], inside [-125, 60]: no clamping): split
// x = j + f by the 1.5 * 2^23 shifter, degree-5 polynomial for 2^f (rel. err
// 2.3e-7, the coefficients of k_blf.cu poly_ex2), 2^j by an exponent add
__device__ __forceinline__ float2 j3_poly_ex2x2(unsigned long long x)
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
// 16-byte chunk swizzle of the interleaved source rows: a thread's 4 output
// columns make consecutive lanes read chunks 2 apart, so quarter-warps would
// hit each 128-byte bank line twice; flipping bit 0 of the chunk index in
// every odd group of 8 chunks spreads the 8 reads over the 8 bank groups
__device__ __forceinline__ int j3_sw(int col)
{
    const int k = col >> 1;
    return ((k ^ ((k >> 3) & 1)) << 1) | (col & 1);
}
__device__ __forceinline__ void j3_decode(const uint32_t* lohi, int b, float coef, float& s, float& range)
{
    const float lo = ordered_to_float(lohi[2 * b]);
    const float hi = ordered_to_float(lohi[2 * b + 1]);
    range = hi - lo;
    s = range > 0.f ? coef / range : coef;
}

}  // namespace

// TH output rows x 64 output columns, 16 threads per row, P = 4 columns per
// thread; blockIdx.z = image * 2 + axis
template <int R, int TH>
struct J3Geom {
    static constexpr int P = 4, TW = 64, NT = 16 * TH;
    static constexpr int ROWS = TH + 2 * R;
    static constexpr int COLS = TW + 2 * R;
    static constexpr int VN = P + 2 * R;                      // window columns per thread
    static constexpr int VN4 = (VN + 3) & ~3;                 // rounded to column quads
    static constexpr int GP = ((COLS + 3) & ~3) + 4;          // guide pitch (floats)
    static constexpr int SP = (COLS + 3 + 15) & ~15;          // source pitch (float2, 128-byte rows)
    static constexpr size_t smem_bytes()
    {
        return (size_t)ROWS * GP * sizeof(float) + (size_t)2 * ROWS * SP * sizeof(float2);
    }
};

// The filter of one staged tile (G: scaled guide gradients, S01 / S2: the
// interleaved channel gradients, all [ROWS] rows from tile row -R)
// and its epilogue: targets of output rows [ty0, ty0 + TH) x columns
// [tx0, tx0 + 64).  row_hook(i) runs at the start of window row i (the
// persistent kernel issues its next-tile copies there).
// XF (factorised exponent, PX only): -(a - b)^2 = -a^2 + 2ab - b^2; exp2(-b^2)
// is folded into the staged sources of column t (G holds b), exp2(-a^2)
// multiplies numerator and normaliser of output s alike and cancels, so one
// FFMA2 per output pair and tap forms both exponents: e = {2a_q, 2a_q+1} b + cs
template <int R, int TH, bool PEERS, bool PX, bool XF, int POLYK, class Hook>
__device__ __forceinline__ void j3_filter_tile(const BlfParams& p, const float* __restrict__ G,
                                               const float2* __restrict__ S01, const float2* __restrict__ S2,
                                               int b, int axis, int tx0, int ty0, float range, Hook&& row_hook)
{
    using Gm = J3Geom<R, TH>;
    constexpr int P = Gm::P, VN = Gm::VN, VN4 = Gm::VN4, GP = Gm::GP, SP = Gm::SP;
    const int H = p.H, W = p.W;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int ox = tx0 + tx * P, oy = ty0 + ty;
    float gs[P];
    unsigned long long acc01[P], acc2z[P];
#pragma unroll
    for (int q = 0; q < P; ++q) {
        gs[q] = G[(ty + R) * GP + tx * P + q + R];
        acc01[q] = 0ull;
        acc2z[q] = 0ull;
    }
    if constexpr (PX) {
        unsigned long long gsp[2], m1;
        const float xs = XF ? 2.0f : 1.0f;
        asm("mov.b64 %0, {%1, %2};" : "=l"(gsp[0]) : "f"(xs * gs[0]), "f"(xs * gs[1]));
        asm("mov.b64 %0, {%1, %2};" : "=l"(gsp[1]) : "f"(xs * gs[2]), "f"(xs * gs[3]));
        asm("mov.b64 %0, {%1, %1};" : "=l"(m1) : "f"(-1.0f));
#pragma unroll 1
        for (int dy = -R; dy <= R; ++dy) {
            row_hook(dy + R);
            const float* grow = G + (ty + R + dy) * GP + tx * P;
            const float2* s01 = S01 + (ty + R + dy) * SP;
            const float2* s2 = S2 + (ty + R + dy) * SP;
            unsigned long long r01[P], r2z[P];
#pragma unroll
            for (int q = 0; q < P; ++q) {
                r01[q] = 0ull;
                r2z[q] = 0ull;
            }
#pragma unroll
            for (int j4 = 0; j4 < VN4; j4 += 4) {
                const float4 g4 = *reinterpret_cast<const float4*>(grow + j4);
                const float gt[4] = {g4.x, g4.y, g4.z, g4.w};
                unsigned long long v01[4], v2z[4];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int pc = j3_sw(tx * P + j4 + 2 * h);
                    const float4 a = *reinterpret_cast<const float4*>(s01 + pc);
                    const float4 c = *reinterpret_cast<const float4*>(s2 + pc);
                    asm("mov.b64 %0, {%1, %2};" : "=l"(v01[2 * h]) : "f"(a.x), "f"(a.y));
                    asm("mov.b64 %0, {%1, %2};" : "=l"(v01[2 * h + 1]) : "f"(a.z), "f"(a.w));
                    asm("mov.b64 %0, {%1, %2};" : "=l"(v2z[2 * h]) : "f"(c.x), "f"(c.y));
                    asm("mov.b64 %0, {%1, %2};" : "=l"(v2z[2 * h + 1]) : "f"(c.z), "f"(c.w));
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
                        unsigned long long gtt, d, nd, ce, e;
                        asm("mov.b64 %0, {%1, %1};" : "=l"(gtt) : "f"(gt[u]));
                        asm("mov.b64 %0, {%1, %2};" : "=l"(ce) : "f"(p.cep[dx0 + R].x), "f"(p.cep[dx0 + R].y));
                        if constexpr (XF) {
                            asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(e) : "l"(gtt), "l"(gsp[h]), "l"(ce));
                        } else {
                            asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(gtt), "l"(m1), "l"(gsp[h]));
                            const float2 dd = j3_unpack(d);
                            asm("mov.b64 %0, {%1, %2};" : "=l"(nd) : "f"(-dd.x), "f"(-dd.y));
                            asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(e) : "l"(nd), "l"(d), "l"(ce));
                        }
                        // POLYK > 0 (XF): every POLYK-th exponent pair on the FMA pipe
                        constexpr int PK = POLYK > 0 ? POLYK : 1;
                        const bool poly = XF && POLYK > 0 && ok0 && ok1 && (j * (P / 2) + h) % PK == PK - 1;
                        float2 ww;
                        if (poly) {
                            ww = j3_poly_ex2x2(e);
                        } else {
                            const float2 ee = j3_unpack(e);
                            ww.x = ok0 ? j3_ex2(ee.x) : 0.f;
                            ww.y = ok1 ? j3_ex2(ee.y) : 0.f;
                        }
                        if (ok0) {
                            r01[q0] = j3_ffma2(ww.x, v01[u], r01[q0]);
                            r2z[q0] = j3_ffma2(ww.x, v2z[u], r2z[q0]);
                        }
                        if (ok1) {
                            r01[q0 + 1] = j3_ffma2(ww.y, v01[u], r01[q0 + 1]);
                            r2z[q0 + 1] = j3_ffma2(ww.y, v2z[u], r2z[q0 + 1]);
                        }
                    }
                }
            }
            const float wy = p.wrow[dy < 0 ? -dy : dy];
#pragma unroll
            for (int q = 0; q < P; ++q) {
                acc01[q] = j3_ffma2(wy, r01[q], acc01[q]);
                acc2z[q] = j3_ffma2(wy, r2z[q], acc2z[q]);
            }
        }
    } else {
#pragma unroll 1
        for (int dy = -R; dy <= R; ++dy) {
            row_hook(dy + R);
            const int ady = dy < 0 ? -dy : dy;
            float ce[R + 1];  // log2 spatial weight of (dy, |dx|)
    #pragma unroll
            for (int k = 0; k <= R; ++k) ce[k] = p.cs[ady] + p.cs[k];
            const float* grow = G + (ty + R + dy) * GP + tx * P;
            const float2* s01 = S01 + (ty + R + dy) * SP;
            const float2* s2 = S2 + (ty + R + dy) * SP;
    #pragma unroll
            for (int j4 = 0; j4 < VN4; j4 += 4) {
                const float4 g4 = *reinterpret_cast<const float4*>(grow + j4);
                const float gt[4] = {g4.x, g4.y, g4.z, g4.w};
                unsigned long long v01[4], v2z[4];
    #pragma unroll
                for (int h = 0; h < 2; ++h) {
                    // columns tx P + j4 + 2h, + 1: one swizzled 16-byte chunk per array
                    const int pc = j3_sw(tx * P + j4 + 2 * h);
                    const float4 a = *reinterpret_cast<const float4*>(s01 + pc);
                    const float4 c = *reinterpret_cast<const float4*>(s2 + pc);
                    asm("mov.b64 %0, {%1, %2};" : "=l"(v01[2 * h]) : "f"(a.x), "f"(a.y));
                    asm("mov.b64 %0, {%1, %2};" : "=l"(v01[2 * h + 1]) : "f"(a.z), "f"(a.w));
                    asm("mov.b64 %0, {%1, %2};" : "=l"(v2z[2 * h]) : "f"(c.x), "f"(c.y));
                    asm("mov.b64 %0, {%1, %2};" : "=l"(v2z[2 * h + 1]) : "f"(c.z), "f"(c.w));
                }
    #pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int j = j4 + u;
                    if (j >= VN) break;
    #pragma unroll
                    for (int q = 0; q < P; ++q) {
                        const int dx = j - q - R;
                        if (dx < -R || dx > R) continue;
                        const float d = gs[q] - gt[u];
                        const float w = j3_ex2(fmaf(-d, d, ce[dx < 0 ? -dx : dx]));
                        acc01[q] = j3_ffma2(w, v01[u], acc01[q]);
                        acc2z[q] = j3_ffma2(w, v2z[u], acc2z[q]);
                    }
                }
            }
        }
    }
    if (oy < p.y1) {
        const float oscale = (p.normalized_out && range > 0.f) ? 1.f / range : 1.f;
        float* dst = axis == 0 ? p.tx : p.ty;
        const size_t pl = (size_t)p.out_rows * W;
        const size_t orow = (size_t)(oy - (p.out_rows == H ? 0 : p.y0)) * W;
        float t[3][P];
#pragma unroll
        for (int q = 0; q < P; ++q) {
            const float2 n01 = j3_unpack(acc01[q]);
            const float2 n2z = j3_unpack(acc2z[q]);
            const float inv = oscale / n2z.y;
            t[0][q] = n01.x * inv;
            t[1][q] = n01.y * inv;
            t[2][q] = n2z.x * inv;
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const size_t off = ((size_t)b * 3 + c) * pl + orow + ox;
            if constexpr (PEERS) {
                const bool vec = ox + P <= W && (off & 3) == 0;  // 16-byte peer stores
                for (int k = 0; k < p.npeers; ++k) {
                    float* d = (axis == 0 ? p.peer_tx[k] : p.peer_ty[k]) + off;
                    if (vec)
                        *reinterpret_cast<float4*>(d) = make_float4(t[c][0], t[c][1], t[c][2], t[c][3]);
                    else
                        for (int q = 0; q < P && ox + q < W; ++q) d[q] = t[c][q];
                }
            } else if (ox + P <= W && (off & 3) == 0) {
                *reinterpret_cast<float4*>(dst + off) = make_float4(t[c][0], t[c][1], t[c][2], t[c][3]);
            } else {
#pragma unroll
                for (int q = 0; q < P; ++q)
                    if (ox + q < W) dst[off + q] = t[c][q];
            }
        }
    }
}

// PEERS: fused band exchange (multi-GPU row bands): every target is stored
// into the full-height buffers of all p.npeers ranks (NVLink peer pointers)
// PX: guide difference and exponent of two adjacent outputs as one FFMA2
// each (column-spatial pair table p.cep, row factor on per-row partial sums)
template <int R, int TH, bool PEERS, int MINB, bool PX = false, bool XF = false, int POLYK = 0>
__global__ void __launch_bounds__(16 * TH, MINB) k_blf_j3(const BlfParams p)
{
    using Gm = J3Geom<R, TH>;
    constexpr int P = Gm::P, TW = Gm::TW, NT = Gm::NT, ROWS = Gm::ROWS, COLS = Gm::COLS;
    constexpr int VN = Gm::VN, VN4 = Gm::VN4, GP = Gm::GP, SP = Gm::SP;
    extern __shared__ __align__(16) float smj[];
    float* G = smj;                                                   // [ROWS][GP]
    float2* S01 = reinterpret_cast<float2*>(smj + ROWS * GP);         // [ROWS][SP] {g0, g1}
    float2* S2 = S01 + ROWS * SP;                                     // [ROWS][SP] {g2, 1}

    const int H = p.H, W = p.W;
    const int b = blockIdx.z >> 1, axis = blockIdx.z & 1;
    const int tx0 = blockIdx.x * TW;
    const int ty0 = p.y0 + blockIdx.y * TH;
    const size_t plane = (size_t)H * W;
    float s, range, sg, grange;
    j3_decode(p.lohi, b, p.range_coef, s, range);
    j3_decode(p.glohi, b, p.range_coef, sg, grange);
    const float* fimg = p.f + (size_t)b * 3 * plane;
    const float* gimg = p.guide + (size_t)b * p.GC * plane;

    // ---- prologue: this axis' circular gradients of guide and channels
    // staging: warp per tile row, lane per column
    {
        const int lane = threadIdx.x & 31;
        for (int i = threadIdx.x >> 5; i < ROWS; i += NT / 32) {
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
                const int o = j3_sw(j);
                if (yin && x >= 0 && x < W) {
                    const int x1 = axis == 0 ? (x + 1 == W ? 0 : x + 1) : x;
                    const float b = (__ldg(gimg + r1 + x1) - __ldg(gimg + r0 + x)) * sg;
                    grow[j] = b;
                    float g[3];
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        const float* fc = fimg + (size_t)c * plane;
                        g[c] = __ldg(fc + r1 + x1) - __ldg(fc + r0 + x);
                    }
                    const float bw = XF ? j3_ex2(-b * b) : 1.0f;  // exp2(-b^2) of column t
                    s01[o] = make_float2(g[0] * bw, g[1] * bw);
                    s2[o] = make_float2(g[2] * bw, bw);
                } else {
                    grow[j] = XF ? 0.0f : kJ3Sentinel;  // XF: b = 0, zero sources: weight 0
                    s01[o] = make_float2(0.f, 0.f);
                    s2[o] = make_float2(0.f, 0.f);
                }
            }
        }
    }
    __syncthreads();

    j3_filter_tile<R, TH, PEERS, PX, XF, POLYK>(p, G, S01, S2, b, axis, tx0, ty0, range, [](int) {});
}

template <int R, int TH, bool PEERS, int MINB, bool PX = false, bool XF = false, int POLYK = 0>
static cudaError_t launch_j3_t(const BlfParams& p, int batch, cudaStream_t st)
{
    using Gm = J3Geom<R, TH>;
    constexpr size_t smem = Gm::smem_bytes();
    cudaError_t e = cudaFuncSetAttribute(k_blf_j3<R, TH, PEERS, MINB, PX, XF, POLYK>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dim3 grid((p.W + Gm::TW - 1) / Gm::TW, (p.y1 - p.y0 + TH - 1) / TH, 2 * batch);
    k_blf_j3<R, TH, PEERS, MINB, PX, XF, POLYK><<<grid, Gm::NT, smem, st>>>(p);
    return cudaGetLastError();
}

template <int R, int TH>
static cudaError_t launch_j3(const BlfParams& p, int batch, cudaStream_t st)
{
    // register cap: 3 CTAs per SM (no spills; c5 0.764 of MUFU) or 4 (64
    // registers, a few spills; 0.755)
    static const int minb = knob("BLFLS_J3_MINB", 3);
    static const int px = knob("BLFLS_J3X", 2);  // 0: per-tap exponents (A/B)
    // difference form (when XF does not apply): pair exponents at 2 CTAs per
    // SM (c5: 0.786 of the MUFU peak, 0.781 at 3 CTAs, 0.765 without); the
    // peer-storing epilogue uses the same arithmetic so band exchange targets
    // match the plain band filter.  (A persistent variant that prefetched the
    // next tile by cp.async measured 0.698 / 0.587: removed in r02.)
    // factorised exponents (XF) whenever exp2(2ab) cannot overflow: |a|, |b| <=
    // range_coef (gradients of an image spanning [lo, hi] are at most hi - lo),
    // so the largest argument is 2 coef^2 (c5, sigma_r = 0.1: 36) and
    // exp2(-b^2) >= 2^-30 keeps the staged sources normal.  XF needs fewer
    // registers, so it runs at 4 CTAs per SM (64 registers): c5 0.778 -> 0.818
    // of the MUFU peak (r01 B200; XF at 2 CTAs per SM: 0.748, at 3: 0.802).
    // BLFLS_J3_XF=0 keeps the difference form.  The peer-storing band
    // epilogue uses the same arithmetic as the plain band filter.
    static const int xf = knob("BLFLS_J3_XF", 1);
    const bool use_xf = xf != 0 && px == 2 && 2.0f * p.range_coef * p.range_coef <= 60.0f;
    if (p.npeers > 0 && use_xf) return launch_j3_t<R, TH, true, TH >= 32 ? 2 : 4, true, true>(p, batch, st);
#ifdef BLFLS_EXPERIMENTS
    static const int polyk = knob("BLFLS_J3_POLY", 0);
    if (use_xf && polyk) {
        switch (polyk) {
            case 4: return launch_j3_t<R, TH, false, 4, true, true, 4>(p, batch, st);
            case 6: return launch_j3_t<R, TH, false, 4, true, true, 6>(p, batch, st);
            case 8: return launch_j3_t<R, TH, false, 4, true, true, 8>(p, batch, st);
            case 12: return launch_j3_t<R, TH, false, 4, true, true, 12>(p, batch, st);
            default: return launch_j3_t<R, TH, false, 3, true, true, 6>(p, batch, st);  // 3 CTAs/SM
        }
    }
#endif
    // 4 CTAs of 16 rows (256 threads) per SM at 64 registers; 32-row tiles
    // (2 CTAs of 512 threads, the halo staged once per 32 output rows) below
    constexpr int XMINB = TH >= 32 ? 2 : 4;
    if (use_xf) return launch_j3_t<R, TH, false, XMINB, true, true>(p, batch, st);
    if (p.npeers > 0) return launch_j3_t<R, TH, true, 2, true>(p, batch, st);
#ifdef BLFLS_EXPERIMENTS
    if (px == 3) return launch_j3_t<R, TH, false, 3, true>(p, batch, st);
    if (px == 0) return minb == 3 ? launch_j3_t<R, TH, false, 3>(p, batch, st) : launch_j3_t<R, TH, false, 4>(p, batch, st);
#endif
    return launch_j3_t<R, TH, false, 2, true>(p, batch, st);
}

// Shared-gray-guide filter (mode 2) on the packed kernel at the radii it is
// instantiated for; false otherwise (the caller runs k_grad_blf<MODE 2>).
// BLFLS_J3=0 selects the unpacked kernel (A/B experiments).
bool launch_grad_blf_j3(const BlfParams& p, int batch, cudaStream_t st, cudaError_t* err)
{
    static const bool enabled = (knob("BLFLS_J3", 1) != 0);
    if (!enabled || p.C != 3) return false;
    switch (p.radius) {
        case 3: *err = launch_j3<3, 16>(p, batch, st); return true;
        case 5: *err = launch_j3<5, 16>(p, batch, st); return true;
        case 7:
            // 32-row tiles when the factorised form runs (2 CTAs of 512
            // threads per SM, the 2R halo rows staged once per 32 output rows
            // instead of 16): c5 0.817 -> 0.831 of the MUFU rate (r02 B200,
            // tools/ab_j3th.sh); the difference form keeps 16 rows
            if (2.0f * p.range_coef * p.range_coef <= 60.0f && knob("BLFLS_J3_TH", 32) == 32) {
                *err = launch_j3<7, 32>(p, batch, st);
                return true;
            }
            *err = launch_j3<7, 16>(p, batch, st);
            return true;
        case 15: *err = launch_j3<15, 16>(p, batch, st); return true;
        default: return false;
    }
}

}  // namespace blfls
