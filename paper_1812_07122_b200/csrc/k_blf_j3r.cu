// k_blf_j3r.cu -- shared-grayscale-guide brute-force BLF (the joint filter of
// bilateral.cpp:28-77 as filter_gradients applies it to the three channels
// with one guide, pipelines.cpp:33-53), TWO output rows x four columns per
// thread.
//
// k_blf_j3 (one row x four columns per thread) is co-limited by shared-memory
// bandwidth: every thread re-reads its 20 staged source columns for each of
// its window rows, 100 wavefronts per 60 warp-MUFU.EX2, i.e. 83% of the
// shared pipe at the MUFU bound (ncu: mio_throttle the top stall).  Here a
// staged source row r serves the output rows y and y + 1 of the thread
// (dy = r - y and r - y - 1), so the same loads feed twice the taps.
//
// Registers for eight outputs come from dropping the per-row partial sums:
// the row factor wy(dy) is folded into the accumulators themselves.  Before
// the taps of window row dy are added (with the weight exp2(2ab + cs[|dx|]),
// no row term), the accumulators are multiplied by wy(dy - 1) / wy(dy); after
// the last row they hold sum_dy wy(dy) / wy(R) * (row sum), and the common
// 1 / wy(R) cancels between numerator and normaliser.  Same factorised
// exponent as k_blf_j3<XF>: exp2(-b^2) is folded into the staged sources,
// exp2(-a^2) cancels.
//
// 32 x 64 output tiles, 256 threads (16 x 16), 73.6 KB of staged sources, 85
// registers: 3 CTAs = 24 warps per SM.
#include <algorithm>
#include <cstdint>

#include "blfls_internal.cuh"

namespace blfls {

namespace {

__device__ __forceinline__ float r_ex2(float x)
{
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// d.xy = {a, a} * b.xy + c.xy
__device__ __forceinline__ unsigned long long r_ffma2(float a, unsigned long long b, unsigned long long c)
{
    unsigned long long aa, d;
    asm("mov.b64 %0, {%1, %1};" : "=l"(aa) : "f"(a));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(aa), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ unsigned long long r_fmul2(float a, unsigned long long b)
{
    unsigned long long aa, d;
    asm("mov.b64 %0, {%1, %1};" : "=l"(aa) : "f"(a));
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(aa), "l"(b));
    return d;
}
__device__ __forceinline__ float2 r_unpack(unsigned long long r)
{
    float2 v;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r));
    return v;
}
// exp2 of both lanes of an f32x2 pair on the FMA pipe (factorised exponents lie
// in [-2 coef^2 + cs_min, 2 coef^2], inside [-125, 60]: no clamping): split
// x = j + f by the 1.5 * 2^23 shifter, degree-5 polynomial for 2^f (rel. err
// 2.3e-7, the coefficients of k_blf.cu poly_ex2), 2^j by an exponent add
__device__ __forceinline__ float2 r_poly_ex2x2(unsigned long long x)
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
// 16-byte chunk swizzle of the interleaved source rows (k_blf_j3.cu j3_sw)
__device__ __forceinline__ int r_sw(int col)
{
    const int k = col >> 1;
    return ((k ^ ((k >> 3) & 1)) << 1) | (col & 1);
}
__device__ __forceinline__ void r_decode(const uint32_t* lohi, int b, float coef, float& s, float& range)
{
    const float lo = ordered_to_float(lohi[2 * b]);
    const float hi = ordered_to_float(lohi[2 * b + 1]);
    range = hi - lo;
    s = range > 0.f ? coef / range : coef;
}

template <int R>
struct J3rGeom {
    static constexpr int P = 4, TW = 64, TH = 32, NT = 256;
    static constexpr int ROWS = TH + 2 * R;
    // the staged tile starts OX columns left of the outputs, a multiple of 4,
    // so aligned column quads of the image map to aligned quads of the tile
    static constexpr int OX = (R + 3) & ~3;
    static constexpr int J0 = OX - R;             // first window column of thread column 0
    static constexpr int VN = P + 2 * R;          // window columns per thread: [J0, J0 + VN)
    static constexpr int VN4 = (J0 + VN + 3) & ~3;  // aligned quads covering the window
    static constexpr int COLS = TW - P + VN4;     // staged columns (a multiple of 4)
    static constexpr int GP = COLS;
    static constexpr int SP = COLS;
    static constexpr size_t smem_bytes()
    {
        return (size_t)ROWS * GP * sizeof(float) + (size_t)2 * ROWS * SP * sizeof(float2);
    }
};

// the taps of one staged source row for the output rows in MASK (bit k: row k)
template <int R, int MASK, int POLYK>
__device__ __forceinline__ void j3r_row(const BlfParams& p, const float* __restrict__ grow,
                                        const float2* __restrict__ s01, const float2* __restrict__ s2, int tx,
                                        const unsigned long long (&gsp)[2][2], unsigned long long (&a01)[2][4],
                                        unsigned long long (&a2z)[2][4])
{
    using Gm = J3rGeom<R>;
    constexpr int P = Gm::P, VN = Gm::VN, VN4 = Gm::VN4;
#pragma unroll
    for (int j4 = 0; j4 < VN4; j4 += 4) {
        const float4 g4 = *reinterpret_cast<const float4*>(grow + j4);
        const float gt[4] = {g4.x, g4.y, g4.z, g4.w};
        unsigned long long v01[4], v2z[4];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int pc = r_sw(tx * P + j4 + 2 * h);
            const float4 a = *reinterpret_cast<const float4*>(s01 + pc);
            const float4 c = *reinterpret_cast<const float4*>(s2 + pc);
            asm("mov.b64 %0, {%1, %2};" : "=l"(v01[2 * h]) : "f"(a.x), "f"(a.y));
            asm("mov.b64 %0, {%1, %2};" : "=l"(v01[2 * h + 1]) : "f"(a.z), "f"(a.w));
            asm("mov.b64 %0, {%1, %2};" : "=l"(v2z[2 * h]) : "f"(c.x), "f"(c.y));
            asm("mov.b64 %0, {%1, %2};" : "=l"(v2z[2 * h + 1]) : "f"(c.z), "f"(c.w));
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int j = j4 + u - Gm::J0;  // window column
            if (j < 0 || j >= VN) continue;
            unsigned long long gtt;
            asm("mov.b64 %0, {%1, %1};" : "=l"(gtt) : "f"(gt[u]));
#pragma unroll
            for (int h = 0; h < P / 2; ++h) {
                const int q0 = 2 * h, dx0 = j - q0 - R;
                const bool ok0 = dx0 >= -R && dx0 <= R, ok1 = dx0 - 1 >= -R && dx0 - 1 <= R;
                if (!ok0 && !ok1) continue;
                unsigned long long ce;
                asm("mov.b64 %0, {%1, %2};" : "=l"(ce) : "f"(p.cep[dx0 + R].x), "f"(p.cep[dx0 + R].y));
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    if (!((MASK >> k) & 1)) continue;
                    unsigned long long e;
                    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(e) : "l"(gtt), "l"(gsp[k][h]), "l"(ce));
                    // POLYK > 0: every POLYK-th exponent pair of the row on the FMA pipe
                    constexpr int PK = POLYK > 0 ? POLYK : 1;
                    const bool poly = POLYK > 0 && ok0 && ok1 && ((j * (P / 2) + h) * 2 + k) % PK == PK - 1;
                    float2 ww;
                    if (poly) {
                        ww = r_poly_ex2x2(e);
                    } else {
                        const float2 ee = r_unpack(e);
                        ww.x = ok0 ? r_ex2(ee.x) : 0.f;
                        ww.y = ok1 ? r_ex2(ee.y) : 0.f;
                    }
                    if (ok0) {
                        a01[k][q0] = r_ffma2(ww.x, v01[u], a01[k][q0]);
                        a2z[k][q0] = r_ffma2(ww.x, v2z[u], a2z[k][q0]);
                    }
                    if (ok1) {
                        a01[k][q0 + 1] = r_ffma2(ww.y, v01[u], a01[k][q0 + 1]);
                        a2z[k][q0 + 1] = r_ffma2(ww.y, v2z[u], a2z[k][q0 + 1]);
                    }
                }
            }
        }
    }
}

}  // namespace

// blockIdx.y = tile row * 2 + axis, blockIdx.z = image: the two axis CTAs of a
// tile row are neighbours in launch order, so they run at the same time on
// different SMs and the second one's staging loads find the raw rows in L2
// (ROWMAJ = false: blockIdx.z = image * 2 + axis, the r01 order, experiments).
// PEERS: fused band exchange (k_blf_j3.cu)
template <int R, bool PEERS, int POLYK, bool ROWMAJ = true>
__global__ void __launch_bounds__(256, 3) k_blf_j3r(const BlfParams p)
{
    using Gm = J3rGeom<R>;
    constexpr int P = Gm::P, TW = Gm::TW, TH = Gm::TH, NT = Gm::NT, ROWS = Gm::ROWS, COLS = Gm::COLS;
    static_assert(COLS % 4 == 0 && TW % 4 == 0, "aligned quads");
    constexpr int GP = Gm::GP, SP = Gm::SP;
    extern __shared__ __align__(16) float smr[];
    float* G = smr;                                               // [ROWS][GP]  b (scaled guide gradient)
    float2* S01 = reinterpret_cast<float2*>(smr + ROWS * GP);     // [ROWS][SP] {g0 B, g1 B}
    float2* S2 = S01 + ROWS * SP;                                 // [ROWS][SP] {g2 B, B}, B = exp2(-b^2)

    const int H = p.H, W = p.W;
    const int b = ROWMAJ ? blockIdx.z : blockIdx.z >> 1;
    const int axis = ROWMAJ ? blockIdx.y & 1 : blockIdx.z & 1;
    const int tx0 = blockIdx.x * TW;
    const int ty0 = p.y0 + (ROWMAJ ? blockIdx.y >> 1 : blockIdx.y) * TH;
    const size_t plane = (size_t)H * W;
    float s, range, sg, grange;
    r_decode(p.lohi, b, p.range_coef, s, range);
    r_decode(p.glohi, b, p.range_coef, sg, grange);
    const float* fimg = p.f + (size_t)b * 3 * plane;
    const float* gimg = p.guide + (size_t)b * p.GC * plane;

    // ---- staging: this axis' circular gradients of guide and channels.
    // Cells outside the image: b = 0 and zero sources (no weight reaches the sums).
    if ((W & 3) == 0 && ((reinterpret_cast<uintptr_t>(p.f) | reinterpret_cast<uintptr_t>(p.guide)) & 15) == 0) {
        // aligned column quads: one task = 4 staged cells of one row from 16-byte
        // loads (8-9 load instructions per 4 cells instead of 8 per cell, ~4
        // dependent rounds per thread instead of ~17)
        constexpr int QPR = COLS / 4, NTASK = ROWS * QPR;
        struct Quad {
            float4 v0[4], v1[4];  // guide, c0, c1, c2: the cells and (axis 1) their +1 row / (axis 0, .x) the cell after
            bool in;
        };
        auto qload = [&](int t, Quad& q) {
            const int i = t / QPR, c = t - i * QPR;
            const int y = ty0 - R + i, x = tx0 - Gm::OX + 4 * c;
            q.in = y >= 0 && y < H && x >= 0 && x < W;
            if (!q.in) return;
            const int r0 = y * W + x;  // offsets within a plane fit 32 bits
            if (axis == 0) {
                const int rn = y * W + (x + 4 == W ? 0 : x + 4);
                q.v0[0] = __ldg(reinterpret_cast<const float4*>(gimg + r0));
                q.v1[0].x = __ldg(gimg + rn);
#pragma unroll
                for (int ch = 0; ch < 3; ++ch) {
                    q.v0[ch + 1] = __ldg(reinterpret_cast<const float4*>(fimg + ch * plane + r0));
                    q.v1[ch + 1].x = __ldg(fimg + ch * plane + rn);
                }
            } else {
                const int r1 = (y + 1 == H ? 0 : y + 1) * W + x;
                q.v0[0] = __ldg(reinterpret_cast<const float4*>(gimg + r0));
                q.v1[0] = __ldg(reinterpret_cast<const float4*>(gimg + r1));
#pragma unroll
                for (int ch = 0; ch < 3; ++ch) {
                    q.v0[ch + 1] = __ldg(reinterpret_cast<const float4*>(fimg + ch * plane + r0));
                    q.v1[ch + 1] = __ldg(reinterpret_cast<const float4*>(fimg + ch * plane + r1));
                }
            }
        };
        auto qstore = [&](int t, const Quad& q) {
            const int i = t / QPR, c = t - i * QPR;
            float4 bq = make_float4(0.f, 0.f, 0.f, 0.f), sa = bq, sb = bq, sc = bq, sd = bq;
            if (q.in) {
                float4 d[4];  // gradients of guide, c0, c1, c2
#pragma unroll
                for (int ch = 0; ch < 4; ++ch) {
                    const float4 a = q.v0[ch];
                    const float4 n = axis == 0 ? make_float4(a.y, a.z, a.w, q.v1[ch].x) : q.v1[ch];
                    d[ch] = make_float4(n.x - a.x, n.y - a.y, n.z - a.z, n.w - a.w);
                }
                bq = make_float4(d[0].x * sg, d[0].y * sg, d[0].z * sg, d[0].w * sg);
                const float w0 = r_ex2(-bq.x * bq.x), w1 = r_ex2(-bq.y * bq.y);
                const float w2 = r_ex2(-bq.z * bq.z), w3 = r_ex2(-bq.w * bq.w);
                sa = make_float4(d[1].x * w0, d[2].x * w0, d[1].y * w1, d[2].y * w1);
                sb = make_float4(d[1].z * w2, d[2].z * w2, d[1].w * w3, d[2].w * w3);
                sc = make_float4(d[3].x * w0, w0, d[3].y * w1, w1);
                sd = make_float4(d[3].z * w2, w2, d[3].w * w3, w3);
            }
            // chunks 2c, 2c + 1 of the interleaved rows (r_sw: swapped in odd groups of 8 chunks)
            const int k0 = (2 * c) ^ ((c >> 2) & 1), k1 = k0 ^ 1;
            *reinterpret_cast<float4*>(G + i * GP + 4 * c) = bq;
            *reinterpret_cast<float4*>(S01 + i * SP + 2 * k0) = sa;
            *reinterpret_cast<float4*>(S01 + i * SP + 2 * k1) = sb;
            *reinterpret_cast<float4*>(S2 + i * SP + 2 * k0) = sc;
            *reinterpret_cast<float4*>(S2 + i * SP + 2 * k1) = sd;
        };
        // (two tasks in flight per thread need > 80 registers: the spills cost
        // more than the second round of loads hides, 0.862 vs 0.872 of MUFU)
        for (int t = threadIdx.x; t < NTASK; t += NT) {
            Quad q;
            qload(t, q);
            qstore(t, q);
        }
    } else {
        // any width: warp per tile row, lane per column
        const int lane = threadIdx.x & 31;
        for (int i = threadIdx.x >> 5; i < ROWS; i += NT / 32) {
            const int y = ty0 - R + i;
            const bool yin = y >= 0 && y < H;
            const int yn = axis == 0 ? y : (y + 1 == H ? 0 : y + 1);
            const size_t r0 = (size_t)(yin ? y : 0) * W, r1 = (size_t)(yin ? yn : 0) * W;
            float* grow = G + i * GP;
            float2* s01 = S01 + i * SP;
            float2* s2 = S2 + i * SP;
            for (int j = lane; j < COLS; j += 32) {
                const int x = tx0 - Gm::OX + j;
                const int o = r_sw(j);
                if (yin && x >= 0 && x < W) {
                    const int x1 = axis == 0 ? (x + 1 == W ? 0 : x + 1) : x;
                    const float bb = (__ldg(gimg + r1 + x1) - __ldg(gimg + r0 + x)) * sg;
                    grow[j] = bb;
                    float g[3];
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        const float* fc = fimg + (size_t)c * plane;
                        g[c] = __ldg(fc + r1 + x1) - __ldg(fc + r0 + x);
                    }
                    const float bw = r_ex2(-bb * bb);
                    s01[o] = make_float2(g[0] * bw, g[1] * bw);
                    s2[o] = make_float2(g[2] * bw, bw);
                } else {
                    grow[j] = 0.0f;
                    s01[o] = make_float2(0.f, 0.f);
                    s2[o] = make_float2(0.f, 0.f);
                }
            }
        }
    }
    __syncthreads();

    const int tx = threadIdx.x & 15, typ = threadIdx.x >> 4;
    unsigned long long gsp[2][2], a01[2][4], a2z[2][4];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const float* ga = G + (2 * typ + k + R) * GP + tx * P + Gm::OX;
        asm("mov.b64 %0, {%1, %2};" : "=l"(gsp[k][0]) : "f"(2.0f * ga[0]), "f"(2.0f * ga[1]));
        asm("mov.b64 %0, {%1, %2};" : "=l"(gsp[k][1]) : "f"(2.0f * ga[2]), "f"(2.0f * ga[3]));
#pragma unroll
        for (int q = 0; q < P; ++q) {
            a01[k][q] = 0ull;
            a2z[k][q] = 0ull;
        }
    }
    // staged row 2 typ + i holds source row (output row 0) - R + i
    const float* grow = G + (2 * typ) * GP + tx * P;
    const float2* s01 = S01 + (2 * typ) * SP;
    const float2* s2 = S2 + (2 * typ) * SP;
    j3r_row<R, 1, POLYK>(p, grow, s01, s2, tx, gsp, a01, a2z);
#pragma unroll 1
    for (int i = 1; i <= 2 * R; ++i) {
        grow += GP;
        s01 += SP;
        s2 += SP;
        const float f0 = p.rfold[i], f1 = p.rfold[i - 1];
#pragma unroll
        for (int q = 0; q < P; ++q) {
            a01[0][q] = r_fmul2(f0, a01[0][q]);
            a2z[0][q] = r_fmul2(f0, a2z[0][q]);
            a01[1][q] = r_fmul2(f1, a01[1][q]);
            a2z[1][q] = r_fmul2(f1, a2z[1][q]);
        }
        j3r_row<R, 3, POLYK>(p, grow, s01, s2, tx, gsp, a01, a2z);
    }
    {
        const float f1 = p.rfold[2 * R];
#pragma unroll
        for (int q = 0; q < P; ++q) {
            a01[1][q] = r_fmul2(f1, a01[1][q]);
            a2z[1][q] = r_fmul2(f1, a2z[1][q]);
        }
        j3r_row<R, 2, POLYK>(p, grow + GP, s01 + SP, s2 + SP, tx, gsp, a01, a2z);
    }

    const int ox = tx0 + tx * P;
    const float oscale = (p.normalized_out && range > 0.f) ? 1.f / range : 1.f;
    float* dst = axis == 0 ? p.tx : p.ty;
    const size_t pl = (size_t)p.out_rows * W;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const int oy = ty0 + 2 * typ + k;
        if (oy >= p.y1) continue;
        const size_t orow = (size_t)(oy - (p.out_rows == H ? 0 : p.y0)) * W;
        float t[3][P];
#pragma unroll
        for (int q = 0; q < P; ++q) {
            const float2 n01 = r_unpack(a01[k][q]);
            const float2 n2z = r_unpack(a2z[k][q]);
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
                for (int n = 0; n < p.npeers; ++n) {
                    float* d = (axis == 0 ? p.peer_tx[n] : p.peer_ty[n]) + off;
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

template <int R, bool PEERS, int POLYK, bool ROWMAJ = true>
static cudaError_t launch_j3r_t(const BlfParams& p, int batch, cudaStream_t st)
{
    using Gm = J3rGeom<R>;
    constexpr size_t smem = Gm::smem_bytes();
    cudaError_t e =
        cudaFuncSetAttribute(k_blf_j3r<R, PEERS, POLYK, ROWMAJ>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int gy = (p.y1 - p.y0 + Gm::TH - 1) / Gm::TH;
    dim3 grid((p.W + Gm::TW - 1) / Gm::TW, ROWMAJ ? 2 * gy : gy, ROWMAJ ? batch : 2 * batch);
    k_blf_j3r<R, PEERS, POLYK, ROWMAJ><<<grid, Gm::NT, smem, st>>>(p);
    return cudaGetLastError();
}

// Two-row shared-gray-guide filter where it applies: three channels, r = 7,
// factorised exponents cannot overflow (2 coef^2 <= 60, k_blf_j3.cu) and the
// folded row factors stay in range (1 / wy(R) <= 2^57).  false: not covered.
bool launch_grad_blf_j3r(const BlfParams& p, int batch, cudaStream_t st, cudaError_t* err)
{
    if (knob("BLFLS_J3R", 1) == 0) return false;
    if (p.C != 3 || (p.radius != 7 && p.radius != 5 && p.radius != 3)) return false;
    if (2.0f * p.range_coef * p.range_coef > 60.0f || -p.cs[p.radius] > 57.0f) return false;
    // every 12th exponent pair of a window row runs on the FMA pipe (f32x2
    // polynomial exp2): the FMA pipe is ~60% busy at the MUFU bound, so the
    // freed MUFU slots pay (c5 r02: 0.870 -> 0.891 of the MUFU rate; periods
    // 24 / 16 / 10 / 8 / 6: 0.887 / 0.887 / 0.889 / 0.887 / 0.872).  The
    // peer-storing band epilogue uses the same arithmetic.
    // Measured and removed (profiles/r02_ab_summary.md): the same loop without
    // its source loads reaches 0.925 (the LDS traffic costs ~5 points through
    // the shared MIO queue); an L2 prefetch of a later tile's raw rows 0.891;
    // two staging tasks in flight per thread (spills at 80 registers) 0.862.
#ifdef BLFLS_EXPERIMENTS
    if (p.radius == 7 && p.npeers == 0 && knob("BLFLS_J3R_ROWMAJ", 1) == 0) {
        *err = launch_j3r_t<7, false, 12, false>(p, batch, st);
        return true;
    }
    switch (p.npeers > 0 || p.radius != 7 ? 12 : knob("BLFLS_J3R_POLY", 12)) {
        case 0: *err = launch_j3r_t<7, false, 0>(p, batch, st); return true;
        case 6: *err = launch_j3r_t<7, false, 6>(p, batch, st); return true;
        case 8: *err = launch_j3r_t<7, false, 8>(p, batch, st); return true;
        case 10: *err = launch_j3r_t<7, false, 10>(p, batch, st); return true;
        case 16: *err = launch_j3r_t<7, false, 16>(p, batch, st); return true;
        case 24: *err = launch_j3r_t<7, false, 24>(p, batch, st); return true;
        default: break;
    }
#endif
    // r = 5 and r = 3 windows start 3 / 1 columns into an aligned quad (r = 5 reads 20
    // instead of 16 staged columns per row, still half of k_blf_j3's per exponential);
    // r = 15 tiles (62 x 96 staged cells) would leave one CTA per SM: k_blf_j3
    if (p.radius == 5) {
        *err = p.npeers > 0 ? launch_j3r_t<5, true, 12>(p, batch, st) : launch_j3r_t<5, false, 12>(p, batch, st);
        return true;
    }
    if (p.radius == 3) {
        *err = p.npeers > 0 ? launch_j3r_t<3, true, 12>(p, batch, st) : launch_j3r_t<3, false, 12>(p, batch, st);
        return true;
    }
    *err = p.npeers > 0 ? launch_j3r_t<7, true, 12>(p, batch, st) : launch_j3r_t<7, false, 12>(p, batch, st);
    return true;
}

}  // namespace blfls
