// k_blf_p2.cu -- self-guided / per-channel-joint brute-force BLF (MODE 0 / 1)
// with packed accumulation, one gradient axis per CTA (bilateral.cpp:28-77
// semantics, driven per channel and axis as filter_gradients does,
// pipelines.cpp:33-53).
//
// The two sums of an output (numerator and normaliser) are one f32x2 pair
// updated by a single FFMA2 with the weight as broadcast scalar: the source
// is staged interleaved as {v, 1}, so per tap
//   FADD (guide difference), FFMA (exponent cs[|dy|] + cs[|dx|] - d^2),
//   MUFU.EX2, FFMA2
// four instructions against five in k_grad_blf (FADD, FFMA, MUFU, FADD,
// FFMA).  The freed issue slots let every POLY-th exponential run on the FMA
// pipe (poly_ex2 of k_blf.cu) next to MUFU.EX2.  Rows of {v, 1} are
// chunk-swizzled like k_blf_j3.cu so the LDS.128 of a quarter-warp (8 lanes,
// each 4 columns apart) hit 8 different bank groups.
#include <cstdlib>

#include "blfls_internal.cuh"

#ifndef BLFLS_P2_QUAD5
// quad staging for the r = 5 self-guided tiles too: their window starts 3 columns
// into an aligned quad, so a window row reads 20 instead of 16 staged columns,
// and still c1 BLF 25.5 -> 24.3 us, c3 1.095 -> 1.081 ms per step (r02)
#define BLFLS_P2_QUAD5 1
#endif

namespace blfls {

namespace {

constexpr float kP2Sentinel = 1.0e15f;

__device__ __forceinline__ float p2_ex2(float x)
{
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// exp2 on the FMA pipe (same polynomial as k_blf.cu poly_ex2)
__device__ __forceinline__ float p2_poly_ex2(float x)
{
    x = fmaxf(x, -125.0f);
    const float t = x + 12582912.0f;
    const float j = t - 12582912.0f;
    const float f = x - j;
    float p = fmaf(0.001327647129073739f, f, 0.009675541892647743f);
    p = fmaf(p, f, 0.05550713092088699f);
    p = fmaf(p, f, 0.24022120237350464f);
    p = fmaf(p, f, 0.6931469440460205f);
    p = fmaf(p, f, 1.0000001192092896f);
    return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}
__device__ __forceinline__ unsigned long long p2_ffma2(float a, unsigned long long b, unsigned long long c)
{
    unsigned long long aa, d;
    asm("mov.b64 %0, {%1, %1};" : "=l"(aa) : "f"(a));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(aa), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ float2 p2_unpack(unsigned long long r)
{
    float2 v;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r));
    return v;
}
__device__ __forceinline__ int p2_sw(int col)
{
    const int k = col >> 1;
    return ((k ^ ((k >> 3) & 1)) << 1) | (col & 1);
}
__device__ __forceinline__ void p2_decode(const uint32_t* lohi, int b, float coef, float& s, float& range)
{
    const float lo = ordered_to_float(lohi[2 * b]);
    const float hi = ordered_to_float(lohi[2 * b + 1]);
    range = hi - lo;
    s = range > 0.f ? coef / range : coef;
}

}  // namespace

template <int R, int TH, int MODE, bool XF = false, bool PX = true>
struct P2Geom {
    static constexpr int P = 4, TW = 64, NT = 16 * TH;
    static constexpr int ROWS = TH + 2 * R;
    static constexpr int VN = P + 2 * R;
    // QUAD (factorised form, radii whose window starts one column after an
    // aligned quad): the staged tile starts OX columns left of the outputs, a
    // multiple of 4, so 16-byte image loads map to 16-byte shared stores
    // (k_blf_j3r.cu); r = 5 would read 20 instead of 16 columns per window row
    static constexpr bool QUAD = PX && ((XF && (R == 7 || R == 15)) || (BLFLS_P2_QUAD5 && R == 5 && MODE == 0));
    static constexpr int OX = QUAD ? ((R + 3) & ~3) : R;
    static constexpr int J0 = OX - R;                    // first window column of thread column 0
    static constexpr int VN4 = (J0 + VN + 3) & ~3;
    static constexpr int COLS = QUAD ? TW - P + VN4 : TW + 2 * R;
    static constexpr int GP = !(MODE == 1 || XF) ? 0 : (QUAD ? COLS : ((COLS + 3) & ~3) + 4);  // planar guide (MODE 1, XF)
    static constexpr int SP = QUAD ? COLS : (COLS + 3 + 15) & ~15;    // {v, 1} pitch (float2)
    static constexpr size_t smem_bytes()
    {
        return (size_t)ROWS * GP * sizeof(float) + (size_t)ROWS * SP * sizeof(float2);
    }
};

// blockIdx.z = plane * 2 + axis, plane = image * C + channel
// PX: the guide difference and exponent of two adjacent outputs (q, q + 1)
// at one source column as one FFMA2 each (the weight's column-spatial term
// from the cep pair table; the row term applied to per-row partial sums), so
// a tap costs 1 + 0.5 + 0.5 instructions next to its MUFU.EX2
// XF (with PX): factorised exponent, as k_blf_j3.cu: -(a - b)^2 = -a^2 + 2ab -
// b^2, exp2(-b^2) folded into the staged source {v B, B} of column t (the
// guide b then lives in the planar G array for both modes), exp2(-a^2)
// cancels between numerator and normaliser: one FFMA2 {2a_q, 2a_q+1} b + cs
// per output pair and tap
template <int R, int TH, int MODE, int POLY, bool PEERS, int MINB, bool PX = false, bool XF = false>
__global__ void __launch_bounds__(16 * TH, MINB) k_blf_p2(const BlfParams p)
{
    using Gm = P2Geom<R, TH, MODE, XF, PX>;
    constexpr int P = Gm::P, TW = Gm::TW, NT = Gm::NT, ROWS = Gm::ROWS, COLS = Gm::COLS;
    constexpr int VN = Gm::VN, VN4 = Gm::VN4, GP = Gm::GP, SP = Gm::SP;
    extern __shared__ __align__(16) float smp[];
    float* G = smp;                                                  // [ROWS][GP] (MODE 1)
    float2* SV = reinterpret_cast<float2*>(smp + ROWS * GP);         // [ROWS][SP] {v, 1}

    const int H = p.H, W = p.W, C = p.C;
    const int pl = blockIdx.z >> 1, axis = blockIdx.z & 1;
    const int b = pl / C, c0 = pl - (pl / C) * C;
    const int tx0 = blockIdx.x * TW;
    const int ty0 = p.y0 + blockIdx.y * TH;
    const size_t plane = (size_t)H * W;
    float s, range;
    p2_decode(p.lohi, b, p.range_coef, s, range);
    float sg = s, grange = range;
    if (MODE == 1) p2_decode(p.glohi, b, p.range_coef, sg, grange);
    const float* fimg = p.f + ((size_t)b * C + c0) * plane;
    const float* gimg = MODE == 0 ? fimg : p.guide + ((size_t)b * p.GC + (p.GC == 1 ? 0 : c0)) * plane;

    // staging
    bool quads = false;
    if constexpr (Gm::QUAD)
        quads = (W & 3) == 0 &&
                ((reinterpret_cast<uintptr_t>(fimg) | reinterpret_cast<uintptr_t>(gimg)) & 15) == 0;
    if (quads) {
        // aligned column quads (k_blf_j3r.cu): one task = 4 staged cells of one
        // row from 16-byte loads
        constexpr int QPR = COLS / 4;
        for (int t = threadIdx.x; t < ROWS * QPR; t += NT) {
            const int i = t / QPR, c = t - i * QPR;
            const int y = ty0 - R + i, x = tx0 - Gm::OX + 4 * c;
            float4 bq = make_float4(0.f, 0.f, 0.f, 0.f), sa = bq, sb = bq;
            if (y >= 0 && y < H && x >= 0 && x < W) {
                const int r0 = y * W + x;
                float4 a = __ldg(reinterpret_cast<const float4*>(fimg + r0)), n, ga = a, gn;
                if (axis == 0) {
                    const int rn = y * W + (x + 4 == W ? 0 : x + 4);
                    n = make_float4(a.y, a.z, a.w, __ldg(fimg + rn));
                    if (MODE == 1) {
                        ga = __ldg(reinterpret_cast<const float4*>(gimg + r0));
                        gn = make_float4(ga.y, ga.z, ga.w, __ldg(gimg + rn));
                    }
                } else {
                    const int r1 = (y + 1 == H ? 0 : y + 1) * W + x;
                    n = __ldg(reinterpret_cast<const float4*>(fimg + r1));
                    if (MODE == 1) {
                        ga = __ldg(reinterpret_cast<const float4*>(gimg + r0));
                        gn = __ldg(reinterpret_cast<const float4*>(gimg + r1));
                    }
                }
                const float4 v = make_float4(n.x - a.x, n.y - a.y, n.z - a.z, n.w - a.w);
                if (MODE == 0)
                    bq = make_float4(v.x * s, v.y * s, v.z * s, v.w * s);
                else
                    bq = make_float4((gn.x - ga.x) * sg, (gn.y - ga.y) * sg, (gn.z - ga.z) * sg, (gn.w - ga.w) * sg);
                const float4 u = MODE == 0 ? bq : v;  // MODE 0: the source is the scaled gradient
                if constexpr (XF) {
                    const float w0 = p2_ex2(-bq.x * bq.x), w1 = p2_ex2(-bq.y * bq.y);
                    const float w2 = p2_ex2(-bq.z * bq.z), w3 = p2_ex2(-bq.w * bq.w);
                    sa = make_float4(u.x * w0, w0, u.y * w1, w1);
                    sb = make_float4(u.z * w2, w2, u.w * w3, w3);
                } else {
                    sa = make_float4(u.x, 1.0f, u.y, 1.0f);
                    sb = make_float4(u.z, 1.0f, u.w, 1.0f);
                }
            } else if constexpr (!XF) {  // difference form: a sentinel guide value gives weight 0
                sa = sb = make_float4(MODE == 0 ? kP2Sentinel : 0.f, 0.f, MODE == 0 ? kP2Sentinel : 0.f, 0.f);
                bq = make_float4(kP2Sentinel, kP2Sentinel, kP2Sentinel, kP2Sentinel);
            }
            const int k0 = (2 * c) ^ ((c >> 2) & 1), k1 = k0 ^ 1;  // p2_sw of chunks 2c, 2c + 1
            if constexpr (MODE == 1 || XF) *reinterpret_cast<float4*>(G + i * GP + 4 * c) = bq;
            *reinterpret_cast<float4*>(SV + i * SP + 2 * k0) = sa;
            *reinterpret_cast<float4*>(SV + i * SP + 2 * k1) = sb;
        }
    } else
    // staging: warp per tile row, lane per column (no per-element division;
    // the row's base pointer and wrap row are computed once)
    {
        const int lane = threadIdx.x & 31;
        for (int i = threadIdx.x >> 5; i < ROWS; i += NT / 32) {
            const int y = ty0 - R + i;
            const bool yin = y >= 0 && y < H;
            const int yn = axis == 0 ? y : (y + 1 == H ? 0 : y + 1);
            const float* f0 = fimg + (size_t)(yin ? y : 0) * W;
            const float* f1 = fimg + (size_t)(yin ? yn : 0) * W;
            const float* g0 = gimg + (size_t)(yin ? y : 0) * W;
            const float* g1 = gimg + (size_t)(yin ? yn : 0) * W;
            float2* srow = SV + i * SP;
#pragma unroll
            for (int j = lane; j < COLS; j += 32) {
                const int x = tx0 - Gm::OX + j;
                if (yin && x >= 0 && x < W) {
                    const int x1 = axis == 0 ? (x + 1 == W ? 0 : x + 1) : x;
                    const float v = __ldg(f1 + x1) - __ldg(f0 + x);
                    if constexpr (XF) {
                        const float bb = MODE == 0 ? v * s : (__ldg(g1 + x1) - __ldg(g0 + x)) * sg;
                        const float bw = p2_ex2(-bb * bb);  // exp2(-b^2) of column t
                        G[i * GP + j] = bb;
                        srow[p2_sw(j)] = make_float2((MODE == 0 ? v * s : v) * bw, bw);
                    } else if (MODE == 0) {
                        srow[p2_sw(j)] = make_float2(v * s, 1.0f);  // source = guide (scaled)
                    } else {
                        G[i * GP + j] = (__ldg(g1 + x1) - __ldg(g0 + x)) * sg;
                        srow[p2_sw(j)] = make_float2(v, 1.0f);
                    }
                } else if constexpr (XF) {
                    srow[p2_sw(j)] = make_float2(0.f, 0.f);  // weight 0, finite exponent
                    G[i * GP + j] = 0.f;
                } else {
                    srow[p2_sw(j)] = make_float2(MODE == 0 ? kP2Sentinel : 0.f, 0.f);
                    if (MODE == 1) G[i * GP + j] = kP2Sentinel;
                }
            }
        }
    }
    __syncthreads();

    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int ox = tx0 + tx * P, oy = ty0 + ty;
    float gs[P];
    unsigned long long acc[P];
#pragma unroll
    for (int q = 0; q < P; ++q) {
        gs[q] = (MODE == 0 && !XF) ? SV[(ty + R) * SP + p2_sw(tx * P + q + Gm::OX)].x
                                   : G[(ty + R) * GP + tx * P + q + Gm::OX];
        acc[q] = 0ull;
    }
    if constexpr (PX) {
        unsigned long long gsp[2];
        const float xs = XF ? 2.0f : 1.0f;
        asm("mov.b64 %0, {%1, %2};" : "=l"(gsp[0]) : "f"(xs * gs[0]), "f"(xs * gs[1]));
        asm("mov.b64 %0, {%1, %2};" : "=l"(gsp[1]) : "f"(xs * gs[2]), "f"(xs * gs[3]));
        unsigned long long m1;
        asm("mov.b64 %0, {%1, %1};" : "=l"(m1) : "f"(-1.0f));
#pragma unroll 1
        for (int dy = -R; dy <= R; ++dy) {
            const float2* sv = SV + (ty + R + dy) * SP;
            const float* grow = G + (ty + R + dy) * GP + tx * P;
            unsigned long long accr[P];
#pragma unroll
            for (int q = 0; q < P; ++q) accr[q] = 0ull;
#pragma unroll
            for (int j4 = 0; j4 < VN4; j4 += 4) {
                float gt[4];
                unsigned long long v1[4];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const float4 a = *reinterpret_cast<const float4*>(sv + p2_sw(tx * P + j4 + 2 * h));
                    asm("mov.b64 %0, {%1, %2};" : "=l"(v1[2 * h]) : "f"(a.x), "f"(a.y));
                    asm("mov.b64 %0, {%1, %2};" : "=l"(v1[2 * h + 1]) : "f"(a.z), "f"(a.w));
                    if (MODE == 0 && !XF) {
                        gt[2 * h] = a.x;
                        gt[2 * h + 1] = a.z;
                    }
                }
                if (MODE == 1 || XF) {
                    const float4 g4 = *reinterpret_cast<const float4*>(grow + j4);
                    gt[0] = g4.x;
                    gt[1] = g4.y;
                    gt[2] = g4.z;
                    gt[3] = g4.w;
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int j = j4 + u - Gm::J0;  // window column
                    if (j < 0 || j >= VN) continue;
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
                            const float2 dd = p2_unpack(d);
                            asm("mov.b64 %0, {%1, %2};" : "=l"(nd) : "f"(-dd.x), "f"(-dd.y));
                            asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(e) : "l"(nd), "l"(d), "l"(ce));
                        }
                        const float2 ee = p2_unpack(e);
                        if (ok0) {
                            const int tap = (dx0 + R) * P + q0;
                            const float w = (POLY > 0 && tap % POLY == POLY - 1) ? p2_poly_ex2(ee.x) : p2_ex2(ee.x);
                            accr[q0] = p2_ffma2(w, v1[u], accr[q0]);
                        }
                        if (ok1) {
                            const int tap = (dx0 - 1 + R) * P + q0 + 1;
                            const float w = (POLY > 0 && tap % POLY == POLY - 1) ? p2_poly_ex2(ee.y) : p2_ex2(ee.y);
                            accr[q0 + 1] = p2_ffma2(w, v1[u], accr[q0 + 1]);
                        }
                    }
                }
            }
            const float wy = p.wrow[dy < 0 ? -dy : dy];
#pragma unroll
            for (int q = 0; q < P; ++q) acc[q] = p2_ffma2(wy, accr[q], acc[q]);
        }
    } else {
#pragma unroll 1
        for (int dy = -R; dy <= R; ++dy) {
            const int ady = dy < 0 ? -dy : dy;
            float ce[R + 1];
    #pragma unroll
            for (int k = 0; k <= R; ++k) ce[k] = p.cs[ady] + p.cs[k];
            const float2* sv = SV + (ty + R + dy) * SP;
            const float* grow = G + (ty + R + dy) * GP + tx * P;
    #pragma unroll
            for (int j4 = 0; j4 < VN4; j4 += 4) {
                float gt[4];
                unsigned long long v1[4];
    #pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const float4 a = *reinterpret_cast<const float4*>(sv + p2_sw(tx * P + j4 + 2 * h));
                    asm("mov.b64 %0, {%1, %2};" : "=l"(v1[2 * h]) : "f"(a.x), "f"(a.y));
                    asm("mov.b64 %0, {%1, %2};" : "=l"(v1[2 * h + 1]) : "f"(a.z), "f"(a.w));
                    if (MODE == 0) {
                        gt[2 * h] = a.x;
                        gt[2 * h + 1] = a.z;
                    }
                }
                if (MODE == 1) {
                    const float4 g4 = *reinterpret_cast<const float4*>(grow + j4);
                    gt[0] = g4.x;
                    gt[1] = g4.y;
                    gt[2] = g4.z;
                    gt[3] = g4.w;
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
                        const float e = fmaf(-d, d, ce[dx < 0 ? -dx : dx]);
                        const int tap = (dx + R) * P + q;
                        const float w = (POLY > 0 && tap % POLY == POLY - 1) ? p2_poly_ex2(e) : p2_ex2(e);
                        acc[q] = p2_ffma2(w, v1[u], acc[q]);
                    }
                }
            }
        }
    }
    if (oy < p.y1) {
        float oscale;
        if (MODE == 0)
            oscale = p.normalized_out ? 1.f / p.range_coef : 1.f / s;
        else
            oscale = (p.normalized_out && range > 0.f) ? 1.f / range : 1.f;
        float t[P];
#pragma unroll
        for (int q = 0; q < P; ++q) {
            const float2 nz = p2_unpack(acc[q]);
            t[q] = nz.x / nz.y * oscale;
        }
        const size_t off = ((size_t)b * C + c0) * ((size_t)p.out_rows * W) +
                           (size_t)(oy - (p.out_rows == H ? 0 : p.y0)) * W + ox;
        if constexpr (PEERS) {
            // one 16-byte store per peer (NVLink writes of whole 16-byte
            // chunks; P = 4 outputs per thread) where aligned and in range
            const bool vec = ox + P <= W && (off & 3) == 0;
            for (int k = 0; k < p.npeers; ++k) {
                float* d = (axis == 0 ? p.peer_tx[k] : p.peer_ty[k]) + off;
                if (vec)
                    *reinterpret_cast<float4*>(d) = make_float4(t[0], t[1], t[2], t[3]);
                else
                    for (int q = 0; q < P && ox + q < W; ++q) d[q] = t[q];
            }
        } else {
            float* dst = (axis == 0 ? p.tx : p.ty) + off;
            if (ox + P <= W && (off & 3) == 0) {
                *reinterpret_cast<float4*>(dst) = make_float4(t[0], t[1], t[2], t[3]);
            } else {
#pragma unroll
                for (int q = 0; q < P; ++q)
                    if (ox + q < W) dst[q] = t[q];
            }
        }
    }
}

template <int R, int TH, int MODE, int POLY, bool PEERS, int MINB, bool PX, bool XF = false>
static cudaError_t launch_p2_t(const BlfParams& p, int nplanes, cudaStream_t st)
{
    using Gm = P2Geom<R, TH, MODE, XF, PX>;
    constexpr size_t smem = Gm::smem_bytes();
    cudaError_t e = cudaFuncSetAttribute(k_blf_p2<R, TH, MODE, POLY, PEERS, MINB, PX, XF>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dim3 grid((p.W + Gm::TW - 1) / Gm::TW, (p.y1 - p.y0 + TH - 1) / TH, 2 * nplanes);
    k_blf_p2<R, TH, MODE, POLY, PEERS, MINB, PX, XF><<<grid, Gm::NT, smem, st>>>(p);
    return cudaGetLastError();
}

template <int R, int MODE, int POLY, bool PX, bool XF = false>
static cudaError_t launch_p2_sized(const BlfParams& p, int nplanes, cudaStream_t st)
{
    // tile height: 32 rows (512 threads, 2 CTAs per SM: the staged halo rows
    // amortised over more outputs; c2 -1%) when that grid still fills ~6
    // waves, else 16, else 8 (small images: c1)
    const long ctas16 = (long)((p.W + 63) / 64) * ((p.y1 - p.y0 + 15) / 16) * 2 * nplanes;
    const long ctas32 = (long)((p.W + 63) / 64) * ((p.y1 - p.y0 + 31) / 32) * 2 * nplanes;
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    static const int th = knob("BLFLS_P2_TH", 0);
    if (PX && (th == 32 || (th == 0 && ctas32 >= 6L * 2 * nsm)))
        return launch_p2_t<R, 32, MODE, POLY, false, 2, PX, XF>(p, nplanes, st);
    if (th == 8 || (th == 0 && ctas16 < 6L * 4 * nsm))
        return launch_p2_t<R, 8, MODE, POLY, false, 8, PX, XF>(p, nplanes, st);
    return launch_p2_t<R, 16, MODE, POLY, false, 4, PX, XF>(p, nplanes, st);
}

// default FMA-pipe exp2 period of the pair-exponent kernel per radius (r01
// B200 sweeps, BLFLS_P2_POLY: r = 5 every 10th tap (c3), r = 7 every 7th
// (c2: 0.942 vs 0.939 at 8, 0.902 at 6), r = 15 every 8th (c4: 1.040 vs
// 1.030 at 7)); the peer-storing band epilogue uses the same period so its
// targets equal the plain band filter's bit for bit
template <int R>
constexpr int kP2DefaultPoly()
{
    return R == 5 ? 10 : (R == 15 ? 8 : 7);
}
// ... and of the factorised-exponent kernel, whose exponents cost half the
// FFMA2 so more of them fit on the FMA pipe (r02, with the quad staging: c2
// 0.985 / 1.000 / 0.994 / 0.984 at 5 / 6 / 7 / 8; c4 1.103 / 1.084 / 1.075 at
// 5 / 6 / 8)
template <int R>
constexpr int kP2XfPoly()
{
    return R == 5 ? 10 : (R == 15 ? 5 : 6);
}

template <int R, int MODE>
static cudaError_t launch_p2(const BlfParams& p, int nplanes, cudaStream_t st)
{
    // default: every 7th exponential on the FMA pipe for the large window
    // (r = 15: c4 0.973 of MUFU against 0.945 unpacked), none otherwise
    static const int poly_env = knob("BLFLS_P2_POLY", -1);
    static const int px = knob("BLFLS_P2X", 1);
    // pair exponents (PX) free enough issue slots for the offload at r = 7 too
    // (r = 5: every 10th; with 32-row tiles it ties the unpacked kernel at
    // c3 and beats it at c1)
    const int poly = poly_env >= 0 ? poly_env : (px ? kP2DefaultPoly<R>() : (R >= 12 ? 7 : 0));
    // factorised exponents (k_blf_j3.cu) for self-guided filtering whenever
    // exp2(2ab) cannot overflow (2 coef^2 <= 60: sigma_r >~ 0.07; c2 and c4,
    // not c1 / c3 at sigma_r = 0.05): c2 0.945 -> 0.976 of the MUFU peak, c4
    // 1.039 -> 1.098 (r01 B200, tools/p2_xf_ab2.sh); BLFLS_P2_XF=0 keeps the
    // difference form.  Same tile geometry: the higher-occupancy variants
    // (16 rows x 6 CTAs or 32 rows x 3 CTAs per SM at 40 registers) spill
    // and measured 0.91-0.94 at c2.
    static const int xf = knob("BLFLS_P2_XF", 1);
    const bool use_xf = MODE == 0 && xf != 0 && px && 2.0f * p.range_coef * p.range_coef <= 60.0f;
    if constexpr (MODE == 0) {
        if (use_xf && p.npeers > 0)
            return launch_p2_t<R, 16, MODE, kP2XfPoly<R>(), true, 3, true, true>(p, nplanes, st);
#ifdef BLFLS_EXPERIMENTS
        if (use_xf && poly_env >= 0) {
            switch (poly_env) {
                case 5: return launch_p2_sized<R, MODE, 5, true, true>(p, nplanes, st);
                case 6: return launch_p2_sized<R, MODE, 6, true, true>(p, nplanes, st);
                case 8: return launch_p2_sized<R, MODE, 8, true, true>(p, nplanes, st);
                case 10: return launch_p2_sized<R, MODE, 10, true, true>(p, nplanes, st);
                default: return launch_p2_sized<R, MODE, 0, true, true>(p, nplanes, st);
            }
        }
#endif
        if (use_xf) return launch_p2_sized<R, MODE, kP2XfPoly<R>(), true, true>(p, nplanes, st);
    }
    // peer-storing epilogue (fused band exchange) with the default offload, so
    // its targets equal the plain band filter's bit for bit
    if (p.npeers > 0) return launch_p2_t<R, 16, MODE, kP2DefaultPoly<R>(), true, 3, true>(p, nplanes, st);
#ifdef BLFLS_EXPERIMENTS
    if (px && poly != kP2DefaultPoly<R>()) {
        switch (poly) {
            case 5: return launch_p2_sized<R, MODE, 5, true>(p, nplanes, st);
            case 6: return launch_p2_sized<R, MODE, 6, true>(p, nplanes, st);
            case 8: return launch_p2_sized<R, MODE, 8, true>(p, nplanes, st);
            case 12: return launch_p2_sized<R, MODE, 12, true>(p, nplanes, st);
            default: return launch_p2_sized<R, MODE, 0, true>(p, nplanes, st);
        }
    }
    if (!px) {
        if (poly == 7) return launch_p2_sized<R, MODE, 7, false>(p, nplanes, st);
        return launch_p2_sized<R, MODE, 0, false>(p, nplanes, st);
    }
#endif
    return launch_p2_sized<R, MODE, kP2DefaultPoly<R>(), true>(p, nplanes, st);
}

// Packed self / per-channel-joint filter; false when not selected (the caller
// runs k_grad_blf).  Default: self-guided r = 5, 7, 15 with pair exponents
// and the FMA-pipe exp2 offload (r01 B200 A/B, tools/p2_ab.sh, p2x_ab.sh:
// c2 BLF 1.062 -> 0.970 ms per 3 iterations, c4 14.72 -> 13.50 ms, c1
// 28.2 -> 25.8 us, c3 tie).  BLFLS_P2=1 forces it for every instantiated
// radius and both modes, BLFLS_P2=0 disables it.
bool launch_grad_blf_p2(const BlfParams& p, int mode, int batch, cudaStream_t st, cudaError_t* err)
{
    const int np = batch * p.C;
#ifdef BLFLS_EXPERIMENTS
    static const int sel = knob("BLFLS_P2", -1);
    if (sel == 0 || mode == 2) return false;
    if (sel > 0) {
        switch (p.radius) {
            case 3: *err = mode == 0 ? launch_p2<3, 0>(p, np, st) : launch_p2<3, 1>(p, np, st); return true;
            case 5: *err = mode == 0 ? launch_p2<5, 0>(p, np, st) : launch_p2<5, 1>(p, np, st); return true;
            case 7: *err = mode == 0 ? launch_p2<7, 0>(p, np, st) : launch_p2<7, 1>(p, np, st); return true;
            case 15: *err = mode == 0 ? launch_p2<15, 0>(p, np, st) : launch_p2<15, 1>(p, np, st); return true;
            default: return false;
        }
    }
#endif
    if (mode != 0) return false;
    {
        int dev = 0, nsm = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        if (launch_grad_blf_p2r(p, np, nsm, st, err)) return true;
    }
    switch (p.radius) {
        case 5: *err = launch_p2<5, 0>(p, np, st); return true;
        case 7: *err = launch_p2<7, 0>(p, np, st); return true;
        case 15: *err = launch_p2<15, 0>(p, np, st); return true;
        default: return false;
    }
}

}  // namespace blfls
