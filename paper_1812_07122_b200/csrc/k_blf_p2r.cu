// k_blf_p2r.cu -- self-guided brute-force BLF of one gradient field (the
// bilateral.cpp:28-77 filter as filter_gradients applies it per channel and
// axis with the field as its own range image, pipelines.cpp:33-53), TWO output
// rows x four columns per thread: k_blf_j3r's scheme for the one-channel case.
//
// Per tap k_blf_p2 spends 1 MUFU.EX2 + 1.5 FFMA2 and re-reads its 20 (r = 7)
// or 36 (r = 15) staged columns for every output row.  Here a staged source row
// serves the thread's output rows y and y + 1, the row factor is folded into
// the sums (the accumulators are multiplied by wy(dy - 1) / wy(dy) before
// window row dy is added; the common 1 / wy(R) cancels in the ratio), so eight
// outputs take 16 accumulator registers and the kernel fits 64 (r = 7: 4 CTAs
// of 256 threads per SM) or 80 registers (r = 15: 3 CTAs).  With one packed
// accumulation per tap the FMA pipe is ~40% busy at the MUFU bound: every
// POLYK-th exponent pair of a window row runs there (f32x2 polynomial exp2).
// Factorised exponents (2 coef^2 <= 60), tiles staged by aligned column quads,
// both axis CTAs of a tile row adjacent in launch order (k_blf_j3r.cu).
#include <algorithm>
#include <cstdint>

#include "blfls_internal.cuh"

namespace blfls {

namespace {

__device__ __forceinline__ float q_ex2(float x)
{
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// d.xy = {a, a} * b.xy + c.xy
__device__ __forceinline__ unsigned long long q_ffma2(float a, unsigned long long b, unsigned long long c)
{
    unsigned long long aa, d;
    asm("mov.b64 %0, {%1, %1};" : "=l"(aa) : "f"(a));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(aa), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ unsigned long long q_fmul2(float a, unsigned long long b)
{
    unsigned long long aa, d;
    asm("mov.b64 %0, {%1, %1};" : "=l"(aa) : "f"(a));
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(aa), "l"(b));
    return d;
}
__device__ __forceinline__ float2 q_unpack(unsigned long long r)
{
    float2 v;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r));
    return v;
}
// exp2 of both lanes of an f32x2 pair on the FMA pipe (factorised exponents lie
// in [-2 coef^2 + cs_min, 2 coef^2], inside [-125, 60]: no clamping): split
// x = j + f by the 1.5 * 2^23 shifter, degree-5 polynomial for 2^f (rel. err
// 2.3e-7, the coefficients of k_blf.cu poly_ex2), 2^j by an exponent add
__device__ __forceinline__ float2 q_poly_ex2x2(unsigned long long x)
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
__device__ __forceinline__ int q_sw(int col)
{
    const int k = col >> 1;
    return ((k ^ ((k >> 3) & 1)) << 1) | (col & 1);
}
__device__ __forceinline__ void q_decode(const uint32_t* lohi, int b, float coef, float& s, float& range)
{
    const float lo = ordered_to_float(lohi[2 * b]);
    const float hi = ordered_to_float(lohi[2 * b + 1]);
    range = hi - lo;
    s = range > 0.f ? coef / range : coef;
}

constexpr float kP2rSentinel = 1.0e15f;  // difference form: a guide value whose weight is exactly 0

template <int R, bool XF = true>
struct P2rGeom {
    static constexpr int P = 4, TW = 64, TH = 32, NT = 256;
    static constexpr int ROWS = TH + 2 * R;
    static constexpr int OX = (R + 3) & ~3;          // staged tile origin left of the outputs (aligned quads)
    static constexpr int J0 = OX - R;
    static constexpr int VN = P + 2 * R;
    static constexpr int VN4 = (J0 + VN + 3) & ~3;
    static constexpr int COLS = TW - P + VN4;
    static constexpr int GP = XF ? COLS : 0, SP = COLS;  // difference form: b is the source's .x
    static constexpr int MINB = R <= 7 ? 4 : 3;
    static constexpr size_t smem_bytes()
    {
        return (size_t)ROWS * GP * sizeof(float) + (size_t)ROWS * SP * sizeof(float2);
    }
};

// the taps of one staged source row for the output rows in MASK (bit k: row k)
// XF: factorised exponent e = {2a_q, 2a_q+1} b + cs (sources {b B, B}); else the
// difference form d = a - b, e = -d d + cs (sources {b, 1}, b read from the source)
template <int R, int MASK, int POLYK, bool XF>
__device__ __forceinline__ void p2r_row(const BlfParams& p, const float* __restrict__ grow,
                                        const float2* __restrict__ sv, int tx,
                                        const unsigned long long (&gsp)[2][2], unsigned long long (&acc)[2][4])
{
    using Gm = P2rGeom<R, XF>;
    constexpr int P = Gm::P, VN = Gm::VN, VN4 = Gm::VN4;
    unsigned long long m1;
    asm("mov.b64 %0, {%1, %1};" : "=l"(m1) : "f"(-1.0f));
#pragma unroll
    for (int j4 = 0; j4 < VN4; j4 += 4) {
        float gt[4];
        if constexpr (XF) {
            const float4 g4 = *reinterpret_cast<const float4*>(grow + j4);
            gt[0] = g4.x;
            gt[1] = g4.y;
            gt[2] = g4.z;
            gt[3] = g4.w;
        }
        unsigned long long v1[4];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const float4 a = *reinterpret_cast<const float4*>(sv + q_sw(tx * P + j4 + 2 * h));
            asm("mov.b64 %0, {%1, %2};" : "=l"(v1[2 * h]) : "f"(a.x), "f"(a.y));
            asm("mov.b64 %0, {%1, %2};" : "=l"(v1[2 * h + 1]) : "f"(a.z), "f"(a.w));
            if constexpr (!XF) {
                gt[2 * h] = a.x;
                gt[2 * h + 1] = a.z;
            }
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
                    if constexpr (XF) {
                        asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(e) : "l"(gtt), "l"(gsp[k][h]), "l"(ce));
                    } else {
                        unsigned long long d, nd;
                        asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(gtt), "l"(m1), "l"(gsp[k][h]));
                        const float2 dd = q_unpack(d);
                        asm("mov.b64 %0, {%1, %2};" : "=l"(nd) : "f"(-dd.x), "f"(-dd.y));
                        asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(e) : "l"(nd), "l"(d), "l"(ce));
                    }
                    constexpr int PK = POLYK > 0 ? POLYK : 1;
                    const bool poly = POLYK > 0 && ok0 && ok1 && ((j * (P / 2) + h) * 2 + k) % PK == PK - 1;
                    float2 ww;
                    if (poly) {
                        if constexpr (!XF) {  // the polynomial's range: clamp (weights below 2^-125 are 0 to fp32 sums)
                            const float2 ee = q_unpack(e);
                            asm("mov.b64 %0, {%1, %2};" : "=l"(e) : "f"(fmaxf(ee.x, -125.0f)), "f"(fmaxf(ee.y, -125.0f)));
                        }
                        ww = q_poly_ex2x2(e);
                    } else {
                        const float2 ee = q_unpack(e);
                        ww.x = ok0 ? q_ex2(ee.x) : 0.f;
                        ww.y = ok1 ? q_ex2(ee.y) : 0.f;
                    }
                    if (ok0) acc[k][q0] = q_ffma2(ww.x, v1[u], acc[k][q0]);
                    if (ok1) acc[k][q0 + 1] = q_ffma2(ww.y, v1[u], acc[k][q0 + 1]);
                }
            }
        }
    }
}

}  // namespace

// blockIdx.y = tile row * 2 + axis, blockIdx.z = plane (image * C + channel)
template <int R, bool PEERS, int POLYK, bool XF = true>
__global__ void __launch_bounds__(256, P2rGeom<R, XF>::MINB) k_blf_p2r(const BlfParams p)
{
    using Gm = P2rGeom<R, XF>;
    constexpr int P = Gm::P, TW = Gm::TW, TH = Gm::TH, NT = Gm::NT, ROWS = Gm::ROWS, COLS = Gm::COLS;
    constexpr int GP = Gm::GP, SP = Gm::SP;
    extern __shared__ __align__(16) float smq[];
    float* G = smq;                                              // [ROWS][GP]  b (scaled gradient)
    float2* SV = reinterpret_cast<float2*>(smq + ROWS * GP);     // [ROWS][SP] {b B, B}, B = exp2(-b^2); !XF: {b, 1}

    const int H = p.H, W = p.W, C = p.C;
    const int pl = blockIdx.z, axis = blockIdx.y & 1;
    const int b = pl / C;
    const int tx0 = blockIdx.x * TW;
    const int ty0 = p.y0 + (blockIdx.y >> 1) * TH;
    const size_t plane = (size_t)H * W;
    float s, range;
    q_decode(p.lohi, b, p.range_coef, s, range);
    const float* fimg = p.f + (size_t)pl * plane;

    // ---- staging: this axis' circular gradient, scaled; cells outside the
    // image: b = 0 and a zero source (no weight reaches the sums)
    if ((W & 3) == 0 && (reinterpret_cast<uintptr_t>(fimg) & 15) == 0) {
        constexpr int QPR = COLS / 4;
        for (int t = threadIdx.x; t < ROWS * QPR; t += NT) {
            const int i = t / QPR, c = t - i * QPR;
            const int y = ty0 - R + i, x = tx0 - Gm::OX + 4 * c;
            float4 bq = make_float4(0.f, 0.f, 0.f, 0.f), sa = bq, sb = bq;
            if constexpr (!XF) sa = sb = make_float4(kP2rSentinel, 0.f, kP2rSentinel, 0.f);
            if (y >= 0 && y < H && x >= 0 && x < W) {
                const int r0 = y * W + x;
                const float4 a = __ldg(reinterpret_cast<const float4*>(fimg + r0));
                float4 n;
                if (axis == 0)
                    n = make_float4(a.y, a.z, a.w, __ldg(fimg + y * W + (x + 4 == W ? 0 : x + 4)));
                else
                    n = __ldg(reinterpret_cast<const float4*>(fimg + (y + 1 == H ? 0 : y + 1) * W + x));
                bq = make_float4((n.x - a.x) * s, (n.y - a.y) * s, (n.z - a.z) * s, (n.w - a.w) * s);
                if constexpr (XF) {
                    const float w0 = q_ex2(-bq.x * bq.x), w1 = q_ex2(-bq.y * bq.y);
                    const float w2 = q_ex2(-bq.z * bq.z), w3 = q_ex2(-bq.w * bq.w);
                    sa = make_float4(bq.x * w0, w0, bq.y * w1, w1);
                    sb = make_float4(bq.z * w2, w2, bq.w * w3, w3);
                } else {
                    sa = make_float4(bq.x, 1.0f, bq.y, 1.0f);
                    sb = make_float4(bq.z, 1.0f, bq.w, 1.0f);
                }
            }
            const int k0 = (2 * c) ^ ((c >> 2) & 1), k1 = k0 ^ 1;  // q_sw of chunks 2c, 2c + 1
            if constexpr (XF) *reinterpret_cast<float4*>(G + i * GP + 4 * c) = bq;
            *reinterpret_cast<float4*>(SV + i * SP + 2 * k0) = sa;
            *reinterpret_cast<float4*>(SV + i * SP + 2 * k1) = sb;
        }
    } else {
        const int lane = threadIdx.x & 31;
        for (int i = threadIdx.x >> 5; i < ROWS; i += NT / 32) {
            const int y = ty0 - R + i;
            const bool yin = y >= 0 && y < H;
            const int yn = axis == 0 ? y : (y + 1 == H ? 0 : y + 1);
            const float* f0 = fimg + (size_t)(yin ? y : 0) * W;
            const float* f1 = fimg + (size_t)(yin ? yn : 0) * W;
            for (int j = lane; j < COLS; j += 32) {
                const int x = tx0 - Gm::OX + j;
                float bb = XF ? 0.f : kP2rSentinel, bw = 0.f;
                if (yin && x >= 0 && x < W) {
                    const int x1 = axis == 0 ? (x + 1 == W ? 0 : x + 1) : x;
                    bb = (__ldg(f1 + x1) - __ldg(f0 + x)) * s;
                    bw = XF ? q_ex2(-bb * bb) : 1.0f;
                }
                if constexpr (XF) G[i * GP + j] = bb;
                SV[i * SP + q_sw(j)] = XF ? make_float2(bb * bw, bw) : make_float2(bb, bw);
            }
        }
    }
    __syncthreads();

    const int tx = threadIdx.x & 15, typ = threadIdx.x >> 4;
    unsigned long long gsp[2][2], acc[2][4];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        float ga[4];
#pragma unroll
        for (int q = 0; q < P; ++q)
            ga[q] = XF ? 2.0f * G[(2 * typ + k + R) * GP + tx * P + Gm::OX + q]
                       : SV[(2 * typ + k + R) * SP + q_sw(tx * P + Gm::OX + q)].x;
        asm("mov.b64 %0, {%1, %2};" : "=l"(gsp[k][0]) : "f"(ga[0]), "f"(ga[1]));
        asm("mov.b64 %0, {%1, %2};" : "=l"(gsp[k][1]) : "f"(ga[2]), "f"(ga[3]));
#pragma unroll
        for (int q = 0; q < P; ++q) acc[k][q] = 0ull;
    }
    // staged row 2 typ + i holds source row (output row 0) - R + i
    const float* grow = G + (2 * typ) * GP + tx * P;
    const float2* sv = SV + (2 * typ) * SP;
    p2r_row<R, 1, POLYK, XF>(p, grow, sv, tx, gsp, acc);
#pragma unroll 1
    for (int i = 1; i <= 2 * R; ++i) {
        grow += GP;
        sv += SP;
        const float f0 = p.rfold[i], f1 = p.rfold[i - 1];
#pragma unroll
        for (int q = 0; q < P; ++q) {
            acc[0][q] = q_fmul2(f0, acc[0][q]);
            acc[1][q] = q_fmul2(f1, acc[1][q]);
        }
        p2r_row<R, 3, POLYK, XF>(p, grow, sv, tx, gsp, acc);
    }
    {
        const float f1 = p.rfold[2 * R];
#pragma unroll
        for (int q = 0; q < P; ++q) acc[1][q] = q_fmul2(f1, acc[1][q]);
        p2r_row<R, 2, POLYK, XF>(p, grow + GP, sv + SP, tx, gsp, acc);
    }

    const int ox = tx0 + tx * P;
    const float oscale = p.normalized_out ? 1.f / p.range_coef : 1.f / s;
    float* dst = axis == 0 ? p.tx : p.ty;
    const size_t plo = (size_t)p.out_rows * W;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const int oy = ty0 + 2 * typ + k;
        if (oy >= p.y1) continue;
        float t[P];
#pragma unroll
        for (int q = 0; q < P; ++q) {
            const float2 nz = q_unpack(acc[k][q]);
            t[q] = nz.x / nz.y * oscale;
        }
        const size_t off = (size_t)pl * plo + (size_t)(oy - (p.out_rows == H ? 0 : p.y0)) * W + ox;
        if constexpr (PEERS) {
            const bool vec = ox + P <= W && (off & 3) == 0;  // 16-byte peer stores
            for (int n = 0; n < p.npeers; ++n) {
                float* d = (axis == 0 ? p.peer_tx[n] : p.peer_ty[n]) + off;
                if (vec)
                    *reinterpret_cast<float4*>(d) = make_float4(t[0], t[1], t[2], t[3]);
                else
                    for (int q = 0; q < P && ox + q < W; ++q) d[q] = t[q];
            }
        } else if (ox + P <= W && (off & 3) == 0) {
            *reinterpret_cast<float4*>(dst + off) = make_float4(t[0], t[1], t[2], t[3]);
        } else {
#pragma unroll
            for (int q = 0; q < P; ++q)
                if (ox + q < W) dst[off + q] = t[q];
        }
    }
}

template <int R, bool PEERS, int POLYK, bool XF = true>
static cudaError_t launch_p2r_t(const BlfParams& p, int nplanes, cudaStream_t st)
{
    using Gm = P2rGeom<R, XF>;
    constexpr size_t smem = Gm::smem_bytes();
    cudaError_t e =
        cudaFuncSetAttribute(k_blf_p2r<R, PEERS, POLYK, XF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int gy = (p.y1 - p.y0 + Gm::TH - 1) / Gm::TH;
    dim3 grid((p.W + Gm::TW - 1) / Gm::TW, 2 * gy, nplanes);
    k_blf_p2r<R, PEERS, POLYK, XF><<<grid, Gm::NT, smem, st>>>(p);
    return cudaGetLastError();
}

template <int R, int DEF, bool XF = true>
static cudaError_t launch_p2r(const BlfParams& p, int nplanes, cudaStream_t st)
{
    if (p.npeers > 0) return launch_p2r_t<R, true, DEF, XF>(p, nplanes, st);
#ifdef BLFLS_EXPERIMENTS
    switch (knob("BLFLS_P2R_POLY", DEF)) {
        case 0: return launch_p2r_t<R, false, 0, XF>(p, nplanes, st);
        case 3: return launch_p2r_t<R, false, 3, XF>(p, nplanes, st);
        case 4: return launch_p2r_t<R, false, 4, XF>(p, nplanes, st);
        case 5: return launch_p2r_t<R, false, 5, XF>(p, nplanes, st);
        case 6: return launch_p2r_t<R, false, 6, XF>(p, nplanes, st);
        case 8: return launch_p2r_t<R, false, 8, XF>(p, nplanes, st);
        case 12: return launch_p2r_t<R, false, 12, XF>(p, nplanes, st);
        default: break;
    }
#endif
    return launch_p2r_t<R, false, DEF, XF>(p, nplanes, st);
}

// Two-row self-guided filter where it applies: r = 7 or 15, factorised
// exponents cannot overflow (2 coef^2 <= 60), the folded row factors stay in
// range, and the grid fills the GPU (32-row tiles).  false: not covered.
bool launch_grad_blf_p2r(const BlfParams& p, int nplanes, int nsm, cudaStream_t st, cudaError_t* err)
{
    if (knob("BLFLS_P2R", 1) == 0) return false;
    if (-p.cs[p.radius] > 57.0f) return false;
    const long ctas = (long)((p.W + 63) / 64) * ((p.y1 - p.y0 + 31) / 32) * 2 * nplanes;
    if (ctas < 6L * 3 * nsm) return false;
    if (2.0f * p.range_coef * p.range_coef > 60.0f) {
        // difference form (sigma_r < 0.0775: c3): r = 5 only; every 8th exponent pair on the
        // FMA pipe (tools/ab_p2r_diff.sh, c3: k_blf_p2 0.901 | none 0.875, 12th 0.906, 8th
        // 0.947, 6th 0.937, 5th 0.919, 4th 0.894, 3rd 0.832 of the MUFU rate)
        if (p.radius != 5 || knob("BLFLS_P2R_DIFF", 1) == 0) return false;
        *err = launch_p2r<5, 8, false>(p, nplanes, st);
        return true;
    }
    if (p.radius != 7 && p.radius != 15) return false;
    // every 4th exponent pair of a window row on the FMA pipe (r02 B200, tools/ab_p2r.sh;
    // fraction of the MUFU rate, k_blf_p2 first: c2 1.001 | none 0.907, 12th 0.963, 8th
    // 1.001, 6th 1.012, 5th 1.025, 4th 1.059, 3rd 0.987; c4 1.104 | 0.970, 1.045, 1.086,
    // 1.115, 1.140, 1.144, 1.082)
    *err = p.radius == 7 ? launch_p2r<7, 4>(p, nplanes, st) : launch_p2r<15, 4>(p, nplanes, st);
    return true;
}

}  // namespace blfls
