// k_blf.cu -- fused circular-gradient + brute-force (joint) bilateral filter.
//
// Replaces, per smooth() iteration, forward_gradients (image.cpp:72-95),
// to_unit_range / from_unit_range_into (pipelines.cpp:17-31), the per-axis,
// per-channel loop of filter_gradients (pipelines.cpp:33-53) and the
// brute-force filter itself (bilateral.cpp:28-77, with an explicit radius in
// place of ceil(3 sigma_s) at bilateral.cpp:37).
//
// Algebra ("Fold"): the [0,1] remap halves gradient
// differences, and the image normalisation divides them by (hi - lo), so the
// reference's range weight exp(-d^2 / (2 sr^2)) on remapped normalised
// gradients equals exp2(-(s * dg)^2) on RAW gradient differences dg with
// s = sqrt(log2(e) / (8 sr^2)) / (hi - lo).  The spatial weight is
// exp2(cs[|dx|] + cs[|dy|]).  The window is clipped at the image border
// (bilateral.cpp:56-57) while the gradients wrap (image.cpp:82,88): halo
// cells outside the image carry a huge guide value so their weight is
// exactly 0, never a zero-filled sample.
//
// Tiling: a 256-thread CTA owns a TH x TW = 16 x (16*P) output tile; each
// thread owns P horizontally adjacent outputs of one row and slides a
// register window along the (2R+1)-tap row, so one shared-memory vector load
// feeds P outputs.  Per tap: FADD, FFMA (exponent with the spatial term as a
// constant-bank operand), MUFU.EX2, FADD, FFMA -- the SFU pipe (16 ex2 per
// clock per SM) is the roofline.
#include "blfls_internal.cuh"

namespace blfls {

constexpr float kSentinel = 1.0e15f;

__device__ __forceinline__ float fast_ex2(float x)
{
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// exp2 on the FMA/ALU pipes (FlashAttention-4-style SFU offload): round to
// nearest with the 1.5*2^23 magic constant, degree-5 near-minimax polynomial
// for 2^f on [-0.5, 0.5] (max relative error 2.3e-7 in fp32 Horner, on par
// with ex2.approx), exponent added in the integer domain.  Inputs below -125
// are clamped (weights < 2^-125 are zero for every practical purpose; the
// MUFU path flushes them to exactly 0).
__device__ __forceinline__ float poly_ex2(float x)
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

// one target value: the local band buffer, or (fused band exchange) the
// same offset of every peer's full-height buffer over NVLink
__device__ __forceinline__ void store_target(const BlfParams& p, int axis, size_t off, float v)
{
    if (p.npeers == 0) {
        (axis == 0 ? p.tx : p.ty)[off] = v;
        return;
    }
    for (int j = 0; j < p.npeers; ++j) (axis == 0 ? p.peer_tx[j] : p.peer_ty[j])[off] = v;
}

__device__ __forceinline__ void decode_range(const uint32_t* lohi, int b, float coef, float& s,
                                             float& range)
{
    const float lo = ordered_to_float(lohi[2 * b]);
    const float hi = ordered_to_float(lohi[2 * b + 1]);
    range = hi - lo;
    // constant image: every gradient is exactly 0 and any finite scale works
    s = range > 0.f ? coef / range : coef;
}

// MODE 0: self-guided (guide = the filtered gradient itself), one channel per CTA
// MODE 1: joint, guide channel == image channel (or C == GC == 1)
// MODE 2: joint, one grayscale guide shared by NC = 3 image channels: one
//         exponential per tap serves all three channels.
// POLY: every POLY-th tap of a row evaluates its exponential with poly_ex2
// on the FMA pipe instead of MUFU.EX2 (0 = never), balancing the two pipes.
// PEERS: the fused band exchange (multi-GPU row bands, p.npeers > 0) -- a
// separate instantiation so the single-GPU kernels carry no peer code.
template <int R, int P, int MODE, int POLY, int TH = 16, bool PEERS = false>
__global__ void __launch_bounds__(16 * TH) k_grad_blf(const BlfParams p)
{
    constexpr int TW = 16 * P;
    constexpr int NT = 16 * TH;  // threads: 16 per output row
    constexpr int NC = MODE == 2 ? 3 : 1;
    constexpr int ROWS = TH + 2 * R;
    constexpr int COLS = TW + 2 * R;
    constexpr int PITCH = (COLS + 3) & ~3;
    constexpr int VN = 2 * R + P;                 // register window per row
    constexpr int VEC = P % 4 == 0 ? 4 : 2;       // shared-memory vector width
    constexpr int NV = (VN + VEC - 1) / VEC;
    constexpr int NS = MODE == 0 ? 0 : NC;        // separate source arrays per axis

    extern __shared__ __align__(16) float sm[];
    float* G = sm;                                 // [2][ROWS][PITCH] guide (scaled)
    float* S = sm + 2 * ROWS * PITCH;              // [2][NS][ROWS][PITCH] raw gradients

    const int H = p.H, W = p.W, C = p.C;
    const int b = MODE == 2 ? blockIdx.z : blockIdx.z / C;
    const int c0 = MODE == 2 ? 0 : blockIdx.z % C;
    const int tx0 = blockIdx.x * TW;
    const int ty0 = p.y0 + blockIdx.y * TH;
    const size_t plane = (size_t)H * W;

    float s, range;
    decode_range(p.lohi, b, p.range_coef, s, range);
    float sg = s, grange = range;
    if (MODE != 0) decode_range(p.glohi, b, p.range_coef, sg, grange);

    // ---- prologue: circular gradients of the tile + R halo into shared memory
    const float* fimg = p.f + ((size_t)b * C + c0) * plane;
    const float* gimg = nullptr;
    if (MODE == 1) gimg = p.guide + ((size_t)b * p.GC + (p.GC == 1 ? 0 : c0)) * plane;
    if (MODE == 2) gimg = p.guide + (size_t)b * p.GC * plane;
    for (int idx = threadIdx.x; idx < ROWS * COLS; idx += NT) {
        const int i = idx / COLS, j = idx - (idx / COLS) * COLS;
        const int y = ty0 - R + i, x = tx0 - R + j;
        const bool in = y >= 0 && y < H && x >= 0 && x < W;
        const int o = i * PITCH + j;
        if (in) {
            const int xn = x + 1 == W ? 0 : x + 1;
            const int yn = y + 1 == H ? 0 : y + 1;
            const size_t r0 = (size_t)y * W, r1 = (size_t)yn * W;
            if (MODE == 0) {
                const float v = __ldg(fimg + r0 + x);
                G[o] = (__ldg(fimg + r0 + xn) - v) * s;
                G[ROWS * PITCH + o] = (__ldg(fimg + r1 + x) - v) * s;
            } else {
                const float gv = __ldg(gimg + r0 + x);
                G[o] = (__ldg(gimg + r0 + xn) - gv) * sg;
                G[ROWS * PITCH + o] = (__ldg(gimg + r1 + x) - gv) * sg;
#pragma unroll
                for (int c = 0; c < NS; ++c) {
                    const float* fc = fimg + (size_t)c * plane;
                    const float v = __ldg(fc + r0 + x);
                    S[(0 * NS + c) * ROWS * PITCH + o] = __ldg(fc + r0 + xn) - v;
                    S[(1 * NS + c) * ROWS * PITCH + o] = __ldg(fc + r1 + x) - v;
                }
            }
        } else {
            G[o] = kSentinel;
            G[ROWS * PITCH + o] = kSentinel;
#pragma unroll
            for (int c = 0; c < NS; ++c) {
                S[(0 * NS + c) * ROWS * PITCH + o] = 0.f;
                S[(1 * NS + c) * ROWS * PITCH + o] = 0.f;
            }
        }
    }
    __syncthreads();

    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int oy = ty0 + ty;
    const int ox = tx0 + tx * P;

    // output scale: MODE 0 accumulates scaled gradients (s * g)
    float oscale;
    if (MODE == 0)
        oscale = p.normalized_out ? 1.f / p.range_coef : 1.f / s;
    else
        oscale = (p.normalized_out && range > 0.f) ? 1.f / range : 1.f;

#pragma unroll 1
    for (int axis = 0; axis < 2; ++axis) {
        const float* Ga = G + axis * ROWS * PITCH;
        const float* Sa = S + axis * NS * ROWS * PITCH;
        float gs[P], z[P], num[NC][P];
#pragma unroll
        for (int q = 0; q < P; ++q) {
            gs[q] = Ga[(ty + R) * PITCH + tx * P + q + R];
            z[q] = 0.f;
#pragma unroll
            for (int c = 0; c < NC; ++c) num[c][q] = 0.f;
        }
#pragma unroll 1
        for (int dy = -R; dy <= R; ++dy) {
            const int row = (ty + R + dy) * PITCH + tx * P;
            float gv[NV * VEC];
            float sv[NS == 0 ? 1 : NS][NV * VEC];
#pragma unroll
            for (int k = 0; k < NV; ++k) {
                if (VEC == 4) {
                    const float4 t = *reinterpret_cast<const float4*>(Ga + row + 4 * k);
                    gv[4 * k] = t.x; gv[4 * k + 1] = t.y; gv[4 * k + 2] = t.z; gv[4 * k + 3] = t.w;
                } else {
                    const float2 t = *reinterpret_cast<const float2*>(Ga + row + 2 * k);
                    gv[2 * k] = t.x; gv[2 * k + 1] = t.y;
                }
#pragma unroll
                for (int c = 0; c < NS; ++c) {
                    const float* Sc = Sa + c * ROWS * PITCH;
                    if (VEC == 4) {
                        const float4 t = *reinterpret_cast<const float4*>(Sc + row + 4 * k);
                        sv[c][4 * k] = t.x; sv[c][4 * k + 1] = t.y; sv[c][4 * k + 2] = t.z; sv[c][4 * k + 3] = t.w;
                    } else {
                        const float2 t = *reinterpret_cast<const float2*>(Sc + row + 2 * k);
                        sv[c][2 * k] = t.x; sv[c][2 * k + 1] = t.y;
                    }
                }
            }
            float zr[P], nr[NC][P];
#pragma unroll
            for (int q = 0; q < P; ++q) {
                zr[q] = 0.f;
#pragma unroll
                for (int c = 0; c < NC; ++c) nr[c][q] = 0.f;
            }
#pragma unroll
            for (int dx = -R; dx <= R; ++dx) {
                const float cx = p.cs[dx < 0 ? -dx : dx];
#pragma unroll
                for (int q = 0; q < P; ++q) {
                    const float v = gv[q + dx + R];
                    const float d = gs[q] - v;
                    const float e = fmaf(-d, d, cx);
                    const int tap = (dx + R) * P + q;
                    const float w = (POLY > 0 && tap % POLY == POLY - 1) ? poly_ex2(e) : fast_ex2(e);
                    zr[q] += w;
#pragma unroll
                    for (int c = 0; c < NC; ++c)
                        nr[c][q] = fmaf(w, MODE == 0 ? v : sv[c][q + dx + R], nr[c][q]);
                }
            }
            const float wy = p.wrow[dy < 0 ? -dy : dy];
#pragma unroll
            for (int q = 0; q < P; ++q) {
                z[q] = fmaf(zr[q], wy, z[q]);
#pragma unroll
                for (int c = 0; c < NC; ++c) num[c][q] = fmaf(nr[c][q], wy, num[c][q]);
            }
        }
        // ---- epilogue
        if (oy < p.y1) {
            const size_t orow = (size_t)(oy - (p.out_rows == H ? 0 : p.y0)) * W;
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                const size_t o = ((size_t)b * C + c0 + c) * ((size_t)p.out_rows * W) + orow + ox;
#pragma unroll
                for (int q = 0; q < P; ++q) {
                    if (ox + q >= W) continue;
                    const float v = num[c][q] / z[q] * oscale;
                    if constexpr (PEERS)
                        store_target(p, axis, o + q, v);
                    else
                        (axis == 0 ? p.tx : p.ty)[o + q] = v;
                }
            }
        }
    }
}

// MODE 2 with packed accumulation: one grayscale guide shared by three image
// channels.  Channels are interleaved in shared memory as {g0, g1} and
// {g2, 1}, so each tap's weight updates all four sums (three numerators and
// the normaliser) with two FFMA2 (sm_100 packed f32x2) instead of four FP32
// instructions: per tap FADD, FFMA, MUFU.EX2, 2x FFMA2.
__device__ __forceinline__ unsigned long long pk2(float a, float b)
{
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ float2 upk2(unsigned long long r)
{
    float2 v;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r));
    return v;
}
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b,
                                                    unsigned long long c)
{
    unsigned long long d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}

template <int R, int QR, int P, int MINB>
__global__ void __launch_bounds__(256, MINB) k_grad_blf_joint3(const BlfParams p)
{
    // 256 threads = 16 x 16; a thread owns QR rows x P = 2 columns of outputs,
    // so every shared-memory window row it loads feeds QR output rows (fewer
    // MIO ops per MUFU.EX2).  One gradient axis is staged at a time.
    constexpr int TW = 16 * P, TH = 16 * QR;
    constexpr int ROWS = TH + 2 * R;
    constexpr int COLS = TW + 2 * R;
    constexpr int PITCH = (COLS + 3) & ~1;        // float2 elements (+ room for vector tails)
    constexpr int VN = 2 * R + P;
    constexpr int GP = (COLS + 3) & ~3;           // guide pitch (floats)
    extern __shared__ __align__(16) float sm[];
    float* G = sm;                                          // [ROWS][GP]
    float2* S01 = reinterpret_cast<float2*>(sm + ROWS * GP); // [ROWS][PITCH] {g0, g1}
    float2* S2 = S01 + ROWS * PITCH;                        // [ROWS][PITCH] {g2, 1}

    const int H = p.H, W = p.W;
    const int b = blockIdx.z;
    const int tx0 = blockIdx.x * TW;
    const int ty0 = p.y0 + blockIdx.y * TH;
    const size_t plane = (size_t)H * W;
    float s, range, sg, grange;
    decode_range(p.lohi, b, p.range_coef, s, range);
    decode_range(p.glohi, b, p.range_coef, sg, grange);
    const float* fimg = p.f + (size_t)b * 3 * plane;
    const float* gimg = p.guide + (size_t)b * p.GC * plane;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int ox = tx0 + tx * P;
    const float oscale = (p.normalized_out && range > 0.f) ? 1.f / range : 1.f;

#pragma unroll 1
    for (int axis = 0; axis < 2; ++axis) {
        if (axis) __syncthreads();
        for (int idx = threadIdx.x; idx < ROWS * COLS; idx += 256) {
            const int i = idx / COLS, j = idx - (idx / COLS) * COLS;
            const int y = ty0 - R + i, x = tx0 - R + j;
            const bool in = y >= 0 && y < H && x >= 0 && x < W;
            const int og = i * GP + j, o = i * PITCH + j;
            if (in) {
                const int x1 = axis == 0 ? (x + 1 == W ? 0 : x + 1) : x;
                const int y1 = axis == 0 ? y : (y + 1 == H ? 0 : y + 1);
                const size_t r0 = (size_t)y * W + x, r1 = (size_t)y1 * W + x1;
                G[og] = (__ldg(gimg + r1) - __ldg(gimg + r0)) * sg;
                float g[3];
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const float* fc = fimg + (size_t)c * plane;
                    g[c] = __ldg(fc + r1) - __ldg(fc + r0);
                }
                S01[o] = make_float2(g[0], g[1]);
                S2[o] = make_float2(g[2], 1.0f);
            } else {
                G[og] = kSentinel;
                S01[o] = make_float2(0.f, 0.f);
                S2[o] = make_float2(0.f, 0.f);
            }
        }
        __syncthreads();

        const unsigned long long* A01 = reinterpret_cast<const unsigned long long*>(S01);
        const unsigned long long* A2 = reinterpret_cast<const unsigned long long*>(S2);
        float gs[QR][P];
        unsigned long long acc01[QR][P], acc2z[QR][P];
#pragma unroll
        for (int i = 0; i < QR; ++i)
#pragma unroll
            for (int q = 0; q < P; ++q) {
                gs[i][q] = G[(ty * QR + i + R) * GP + tx * P + q + R];
                acc01[i][q] = 0ull;
                acc2z[i][q] = 0ull;
            }
        // source rows ty*QR + sr, sr in [0, QR + 2R): output row i sees dy = sr - i - R
#pragma unroll 1
        for (int sr = 0; sr < QR + 2 * R; ++sr) {
            const int rowg = (ty * QR + sr) * GP + tx * P;
            const int rows = (ty * QR + sr) * PITCH + tx * P;
            float gv[VN];
#pragma unroll
            for (int k = 0; k < VN / 2; ++k) {
                const float2 t = *reinterpret_cast<const float2*>(G + rowg + 2 * k);
                gv[2 * k] = t.x;
                gv[2 * k + 1] = t.y;
            }
            unsigned long long a01[VN], a2[VN];
#pragma unroll
            for (int k = 0; k < VN; ++k) {
                a01[k] = A01[rows + k];
                a2[k] = A2[rows + k];
            }
#pragma unroll
            for (int i = 0; i < QR; ++i) {
                const int dy = sr - i - R;
                if (dy < -R || dy > R) continue;  // warp-uniform
                unsigned long long r01[P], r2z[P];
#pragma unroll
                for (int q = 0; q < P; ++q) {
                    r01[q] = 0ull;
                    r2z[q] = 0ull;
                }
#pragma unroll
                for (int dx = -R; dx <= R; ++dx) {
                    const float cx = p.cs[dx < 0 ? -dx : dx];
#pragma unroll
                    for (int q = 0; q < P; ++q) {
                        const int k = q + dx + R;
                        const float d = gs[i][q] - gv[k];
                        const float w = fast_ex2(fmaf(-d, d, cx));
                        const unsigned long long ww = pk2(w, w);
                        r01[q] = ffma2(ww, a01[k], r01[q]);
                        r2z[q] = ffma2(ww, a2[k], r2z[q]);
                    }
                }
                const float wy = p.wrow[dy < 0 ? -dy : dy];
                const unsigned long long wyy = pk2(wy, wy);
#pragma unroll
                for (int q = 0; q < P; ++q) {
                    acc01[i][q] = ffma2(r01[q], wyy, acc01[i][q]);
                    acc2z[i][q] = ffma2(r2z[q], wyy, acc2z[i][q]);
                }
            }
        }
        float* dst = axis == 0 ? p.tx : p.ty;
        const size_t pl = (size_t)p.out_rows * W;
#pragma unroll
        for (int i = 0; i < QR; ++i) {
            const int oy = ty0 + ty * QR + i;
            if (oy >= p.y1) continue;
            const size_t orow = (size_t)(oy - (p.out_rows == H ? 0 : p.y0)) * W;
#pragma unroll
            for (int q = 0; q < P; ++q) {
                if (ox + q >= W) continue;
                const float2 n01 = upk2(acc01[i][q]);
                const float2 n2z = upk2(acc2z[i][q]);
                const float inv = oscale / n2z.y;
                const size_t o = orow + ox + q;
                dst[((size_t)b * 3 + 0) * pl + o] = n01.x * inv;
                dst[((size_t)b * 3 + 1) * pl + o] = n01.y * inv;
                dst[((size_t)b * 3 + 2) * pl + o] = n2z.x * inv;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Packed self-guided kernel (MODE 0): pairs of adjacent outputs (q, q+1)
// share every instruction through sm_100 f32x2 math:
//   d = {gs_q, gs_q+1} - {v_k, v_k+1}        FADD2
//   e = -d*d + {c_dx, c_dx}                  FFMA2
//   w = {ex2(e.x), ex2(e.y)}                 2x MUFU.EX2 (or the FMA-pipe poly)
//   {z_q, z_q+1} += w ; {n_q, n_q+1} += w*v  FADD2 + FFMA2
// so a tap costs 2 issue slots + 1 MUFU instead of 4 + 1.  {v_k, v_k+1} must be
// an aligned register pair; the window is kept twice (from the gradient array
// and from a copy shifted by one column) so both parities of k are aligned.
// POLY: every POLY-th pair-tap evaluates both exponentials with poly_ex2 on
// the FMA pipe, balancing the FMA and SFU pipes.
typedef unsigned long long f2x;
__device__ __forceinline__ f2x f2(float a, float b)
{
    f2x r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ float2 f2u(f2x r)
{
    float2 v;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r));
    return v;
}
__device__ __forceinline__ f2x add2(f2x a, f2x b)
{
    f2x d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ f2x sub2(f2x a, f2x b)
{
    f2x d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ f2x fma2(f2x a, f2x b, f2x c)
{
    f2x d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ f2x neg2(f2x a) { return a ^ 0x8000000080000000ull; }

__device__ __forceinline__ f2x poly_ex2x2(f2x e)
{
    float2 x = f2u(e);
    x.x = fmaxf(x.x, -125.0f);
    x.y = fmaxf(x.y, -125.0f);
    const f2x xx = f2(x.x, x.y);
    const f2x magic = f2(12582912.0f, 12582912.0f);
    const f2x t = add2(xx, magic);
    const f2x f = sub2(xx, sub2(t, magic));
    f2x p = fma2(f2(0.001327647129073739f, 0.001327647129073739f), f,
                 f2(0.009675541892647743f, 0.009675541892647743f));
    p = fma2(p, f, f2(0.05550713092088699f, 0.05550713092088699f));
    p = fma2(p, f, f2(0.24022120237350464f, 0.24022120237350464f));
    p = fma2(p, f, f2(0.6931469440460205f, 0.6931469440460205f));
    p = fma2(p, f, f2(1.0000001192092896f, 1.0000001192092896f));
    const float2 pp = f2u(p), tt = f2u(t);
    return f2(__int_as_float(__float_as_int(pp.x) + (__float_as_int(tt.x) << 23)),
              __int_as_float(__float_as_int(pp.y) + (__float_as_int(tt.y) << 23)));
}

template <int R, int POLY>
__global__ void __launch_bounds__(256) k_grad_blf_x2(const BlfParams p)
{
    constexpr int P = 4, TW = 64, TH = 16;
    constexpr int ROWS = TH + 2 * R;
    constexpr int COLS = TW + 2 * R;
    constexpr int PITCH = ((COLS + 3) & ~3) + 4;  // room for the +1-shifted copy's tail
    constexpr int VN = ((2 * R + P + 1) + 3) & ~3; // window floats (multiple of 4)
    constexpr int NV = VN / 4;
    extern __shared__ __align__(16) float sm[];
    float* G0 = sm;                 // [ROWS][PITCH] scaled gradients of this axis
    float* G1 = sm + ROWS * PITCH;  // G1[i][j] = G0[i][j + 1]

    const int H = p.H, W = p.W, C = p.C;
    const int b = blockIdx.z / C;
    const int c0 = blockIdx.z % C;
    const int tx0 = blockIdx.x * TW;
    const int ty0 = p.y0 + blockIdx.y * TH;
    const size_t plane = (size_t)H * W;
    float s, range;
    decode_range(p.lohi, b, p.range_coef, s, range);
    const float* fimg = p.f + ((size_t)b * C + c0) * plane;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int oy = ty0 + ty;
    const int ox = tx0 + tx * P;
    const float oscale = p.normalized_out ? 1.f / p.range_coef : 1.f / s;

#pragma unroll 1
    for (int axis = 0; axis < 2; ++axis) {
        if (axis) __syncthreads();
        for (int idx = threadIdx.x; idx < ROWS * (COLS + 1); idx += 256) {
            const int i = idx / (COLS + 1), j = idx - (idx / (COLS + 1)) * (COLS + 1);
            const int y = ty0 - R + i, x = tx0 - R + j;
            float g = kSentinel;
            if (y >= 0 && y < H && x >= 0 && x < W) {
                const int x1 = axis == 0 ? (x + 1 == W ? 0 : x + 1) : x;
                const int y1 = axis == 0 ? y : (y + 1 == H ? 0 : y + 1);
                g = (__ldg(fimg + (size_t)y1 * W + x1) - __ldg(fimg + (size_t)y * W + x)) * s;
            }
            if (j < COLS) G0[i * PITCH + j] = g;
            if (j > 0) G1[i * PITCH + j - 1] = g;
        }
        __syncthreads();

        f2x gs01, gs23, z01 = 0ull, z23 = 0ull, n01 = 0ull, n23 = 0ull;
        {
            const float* c = G0 + (ty + R) * PITCH + tx * P + R;
            gs01 = f2(c[0], c[1]);
            gs23 = f2(c[2], c[3]);
        }
#pragma unroll 1
        for (int dy = -R; dy <= R; ++dy) {
            const int row = (ty + R + dy) * PITCH + tx * P;
            // wa[m] = {v_2m, v_2m+1}, wb[m] = {v_2m+1, v_2m+2}
            f2x wa[VN / 2], wb[VN / 2];
#pragma unroll
            for (int k = 0; k < NV; ++k) {
                const float4 a = *reinterpret_cast<const float4*>(G0 + row + 4 * k);
                const float4 c = *reinterpret_cast<const float4*>(G1 + row + 4 * k);
                wa[2 * k] = f2(a.x, a.y);
                wa[2 * k + 1] = f2(a.z, a.w);
                wb[2 * k] = f2(c.x, c.y);
                wb[2 * k + 1] = f2(c.z, c.w);
            }
            f2x zr01 = 0ull, zr23 = 0ull, nr01 = 0ull, nr23 = 0ull;
#pragma unroll
            for (int dx = -R; dx <= R; ++dx) {
                const float cxs = p.cs[dx < 0 ? -dx : dx];
                const f2x cx = f2(cxs, cxs);
#pragma unroll
                for (int h = 0; h < 2; ++h) {       // output pair (0,1) or (2,3)
                    const int k = 2 * h + dx + R;   // window index of output 2h's tap
                    const f2x v = (k & 1) ? wb[k >> 1] : wa[k >> 1];
                    const f2x d = sub2(h ? gs23 : gs01, v);
                    const f2x e = fma2(neg2(d), d, cx);
                    f2x w;
                    if (POLY > 0 && ((dx + R) * 2 + h) % POLY == POLY - 1) {
                        w = poly_ex2x2(e);
                    } else {
                        const float2 ee = f2u(e);
                        w = f2(fast_ex2(ee.x), fast_ex2(ee.y));
                    }
                    if (h) {
                        zr23 = add2(zr23, w);
                        nr23 = fma2(w, v, nr23);
                    } else {
                        zr01 = add2(zr01, w);
                        nr01 = fma2(w, v, nr01);
                    }
                }
            }
            const float wys = p.wrow[dy < 0 ? -dy : dy];
            const f2x wy = f2(wys, wys);
            z01 = fma2(zr01, wy, z01);
            z23 = fma2(zr23, wy, z23);
            n01 = fma2(nr01, wy, n01);
            n23 = fma2(nr23, wy, n23);
        }
        if (oy < p.y1) {
            float* dst = axis == 0 ? p.tx : p.ty;
            float* o = dst + ((size_t)b * C + c0) * ((size_t)p.out_rows * W) +
                       (size_t)(oy - (p.out_rows == H ? 0 : p.y0)) * W;
            const float2 za = f2u(z01), zb = f2u(z23), na = f2u(n01), nb = f2u(n23);
            const float r[4] = {na.x / za.x * oscale, na.y / za.y * oscale, nb.x / zb.x * oscale,
                                nb.y / zb.y * oscale};
#pragma unroll
            for (int q = 0; q < P; ++q)
                if (ox + q < W) o[ox + q] = r[q];
        }
    }
}

// Generic-radius variant (any R up to kMaxRadius): same tiling, window loops
// not unrolled, taps read straight from shared memory.
template <int MODE>
__global__ void __launch_bounds__(256) k_grad_blf_any(const BlfParams p)
{
    constexpr int P = 4, TW = 64, TH = 16;
    constexpr int NC = MODE == 2 ? 3 : 1;
    constexpr int NS = MODE == 0 ? 0 : NC;
    const int R = p.radius;
    const int ROWS = TH + 2 * R, COLS = TW + 2 * R, PITCH = (COLS + 3) & ~3;
    extern __shared__ __align__(16) float sm[];
    float* G = sm;
    float* S = sm + 2 * ROWS * PITCH;
    const int H = p.H, W = p.W, C = p.C;
    const int b = MODE == 2 ? blockIdx.z : blockIdx.z / C;
    const int c0 = MODE == 2 ? 0 : blockIdx.z % C;
    const int tx0 = blockIdx.x * TW;
    const int ty0 = p.y0 + blockIdx.y * TH;
    const size_t plane = (size_t)H * W;
    float s, range;
    decode_range(p.lohi, b, p.range_coef, s, range);
    float sg = s, grange = range;
    if (MODE != 0) decode_range(p.glohi, b, p.range_coef, sg, grange);
    const float* fimg = p.f + ((size_t)b * C + c0) * plane;
    const float* gimg = nullptr;
    if (MODE == 1) gimg = p.guide + ((size_t)b * p.GC + (p.GC == 1 ? 0 : c0)) * plane;
    if (MODE == 2) gimg = p.guide + (size_t)b * p.GC * plane;
    for (int idx = threadIdx.x; idx < ROWS * COLS; idx += 256) {
        const int i = idx / COLS, j = idx % COLS;
        const int y = ty0 - R + i, x = tx0 - R + j;
        const bool in = y >= 0 && y < H && x >= 0 && x < W;
        const int o = i * PITCH + j;
        if (in) {
            const int xn = x + 1 == W ? 0 : x + 1;
            const int yn = y + 1 == H ? 0 : y + 1;
            const size_t r0 = (size_t)y * W, r1 = (size_t)yn * W;
            if (MODE == 0) {
                const float v = fimg[r0 + x];
                G[o] = (fimg[r0 + xn] - v) * s;
                G[ROWS * PITCH + o] = (fimg[r1 + x] - v) * s;
            } else {
                const float gv = gimg[r0 + x];
                G[o] = (gimg[r0 + xn] - gv) * sg;
                G[ROWS * PITCH + o] = (gimg[r1 + x] - gv) * sg;
                for (int c = 0; c < NS; ++c) {
                    const float* fc = fimg + (size_t)c * plane;
                    const float v = fc[r0 + x];
                    S[(0 * NS + c) * ROWS * PITCH + o] = fc[r0 + xn] - v;
                    S[(1 * NS + c) * ROWS * PITCH + o] = fc[r1 + x] - v;
                }
            }
        } else {
            G[o] = kSentinel;
            G[ROWS * PITCH + o] = kSentinel;
            for (int c = 0; c < NS; ++c) {
                S[(0 * NS + c) * ROWS * PITCH + o] = 0.f;
                S[(1 * NS + c) * ROWS * PITCH + o] = 0.f;
            }
        }
    }
    __syncthreads();
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int oy = ty0 + ty, ox = tx0 + tx * P;
    float oscale;
    if (MODE == 0)
        oscale = p.normalized_out ? 1.f / p.range_coef : 1.f / s;
    else
        oscale = (p.normalized_out && range > 0.f) ? 1.f / range : 1.f;
    for (int axis = 0; axis < 2; ++axis) {
        const float* Ga = G + axis * ROWS * PITCH;
        const float* Sa = S + axis * NS * ROWS * PITCH;
        float z[P], num[NC][P], gs[P];
        for (int q = 0; q < P; ++q) {
            gs[q] = Ga[(ty + R) * PITCH + tx * P + q + R];
            z[q] = 0.f;
            for (int c = 0; c < NC; ++c) num[c][q] = 0.f;
        }
        for (int dy = -R; dy <= R; ++dy) {
            const int row = (ty + R + dy) * PITCH + tx * P;
            const float wy = p.wrow[dy < 0 ? -dy : dy];
            for (int dx = -R; dx <= R; ++dx) {
                const float cx = p.cs[dx < 0 ? -dx : dx];
#pragma unroll
                for (int q = 0; q < P; ++q) {
                    const float v = Ga[row + q + dx + R];
                    const float d = gs[q] - v;
                    const float w = fast_ex2(fmaf(-d, d, cx)) * wy;
                    z[q] += w;
#pragma unroll
                    for (int c = 0; c < NC; ++c)
                        num[c][q] = fmaf(w, MODE == 0 ? v : Sa[c * ROWS * PITCH + row + q + dx + R], num[c][q]);
                }
            }
        }
        if (oy < p.y1) {
            const size_t orow = (size_t)(oy - (p.out_rows == H ? 0 : p.y0)) * W;
            for (int c = 0; c < NC; ++c) {
                const size_t o = ((size_t)b * C + c0 + c) * ((size_t)p.out_rows * W) + orow + ox;
                for (int q = 0; q < P; ++q)
                    if (ox + q < W) store_target(p, axis, o + q, num[c][q] / z[q] * oscale);
            }
        }
    }
}

// ------------------------------------------------------------- dispatch --

template <int R, int P, int MODE, int POLY, int TH, bool PEERS = false>
static cudaError_t launch_fixed_th(const BlfParams& p, int nz, cudaStream_t st)
{
    constexpr int TW = 16 * P;
    constexpr int ROWS = TH + 2 * R, COLS = TW + 2 * R, PITCH = (COLS + 3) & ~3;
    constexpr int NARR = MODE == 0 ? 2 : (MODE == 1 ? 4 : 8);
    const size_t smem = (size_t)NARR * ROWS * PITCH * sizeof(float);
    // not a stream operation: legal while the stream is being captured
    cudaError_t e = cudaFuncSetAttribute(k_grad_blf<R, P, MODE, POLY, TH, PEERS>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dim3 grid((p.W + TW - 1) / TW, (p.y1 - p.y0 + TH - 1) / TH, nz);
    k_grad_blf<R, P, MODE, POLY, TH, PEERS><<<grid, 16 * TH, smem, st>>>(p);
    return cudaGetLastError();
}

// Tile height: 16 rows (256 threads) normally; 8 rows (128 threads) when the
// 16-row grid would fill fewer than ~8 waves of resident CTAs, so the last
// partial wave idles a smaller fraction of the SMs (r01: c2 = 3.5 waves).
template <int R, int P, int MODE, int POLY>
static cudaError_t launch_fixed(const BlfParams& p, int nz, cudaStream_t st)
{
    const long tiles16 = (long)((p.W + 16 * P - 1) / (16 * P)) * ((p.y1 - p.y0 + 15) / 16) * nz;
    const int th = p.tile_rows > 0 ? p.tile_rows : (tiles16 < 8L * 148 * 6 ? 8 : 16);
    if (th == 8) return launch_fixed_th<R, P, MODE, POLY, 8>(p, nz, st);
    return launch_fixed_th<R, P, MODE, POLY, 16>(p, nz, st);
}

template <int MODE>
static cudaError_t launch_any(const BlfParams& p, int nz, cudaStream_t st)
{
    const int R = p.radius;
    const int ROWS = 16 + 2 * R, COLS = 64 + 2 * R, PITCH = (COLS + 3) & ~3;
    const int NARR = MODE == 0 ? 2 : (MODE == 1 ? 4 : 8);
    const size_t smem = (size_t)NARR * ROWS * PITCH * sizeof(float);
    cudaError_t e = cudaFuncSetAttribute(k_grad_blf_any<MODE>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dim3 grid((p.W + 63) / 64, (p.y1 - p.y0 + 15) / 16, nz);
    k_grad_blf_any<MODE><<<grid, 256, smem, st>>>(p);
    return cudaGetLastError();
}

// default SFU-offload period per mode: self / per-channel joint spend 4 FP32
// ops per tap next to the MUFU op, the shared-guide mode 6 (3 channels)
template <int MODE>
constexpr int kPolyDefault = 0;  // r01 sweep (tools/poly_sweep.py): offload does not pay yet

#ifdef BLFLS_EXPERIMENTS
template <int R, int QR, int P, int MINB>
static cudaError_t launch_joint3_q(const BlfParams& p, int nz, cudaStream_t st)
{
    constexpr int TW = 16 * P, TH = 16 * QR, ROWS = TH + 2 * R, COLS = TW + 2 * R;
    constexpr int PITCH = (COLS + 3) & ~1, GP = (COLS + 3) & ~3;
    const size_t smem = (size_t)ROWS * GP * sizeof(float) + (size_t)2 * ROWS * PITCH * sizeof(float2);
    cudaError_t e = cudaFuncSetAttribute(k_grad_blf_joint3<R, QR, P, MINB>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dim3 grid((p.W + TW - 1) / TW, (p.y1 - p.y0 + TH - 1) / TH, nz);
    k_grad_blf_joint3<R, QR, P, MINB><<<grid, 256, smem, st>>>(p);
    return cudaGetLastError();
}

template <int R>
static cudaError_t launch_joint3(const BlfParams& p, int nz, cudaStream_t st)
{
    // rows per thread: experiment override via BLFLS_J3_ROWS, default 2
    switch (p.joint3_rows) {
        case 2: return launch_joint3_q<R, 2, 2, 1>(p, nz, st);
        case 4: return launch_joint3_q<R, 1, 4, 1>(p, nz, st);   // 4 columns per thread
        case 5: return launch_joint3_q<R, 1, 4, 2>(p, nz, st);   // 4 columns, <= 128 regs
        case 6: return launch_joint3_q<R, 1, 2, 3>(p, nz, st);   // 2 columns, <= 80 regs
        default: return launch_joint3_q<R, 1, 2, 1>(p, nz, st);
    }
}

template <int R, int POLY>
static cudaError_t launch_x2(const BlfParams& p, int nz, cudaStream_t st)
{
    constexpr int TW = 64, TH = 16, ROWS = TH + 2 * R, COLS = TW + 2 * R;
    constexpr int PITCH = ((COLS + 3) & ~3) + 4;
    const size_t smem = (size_t)2 * ROWS * PITCH * sizeof(float);
    cudaError_t e = cudaFuncSetAttribute(k_grad_blf_x2<R, POLY>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dim3 grid((p.W + TW - 1) / TW, (p.y1 - p.y0 + TH - 1) / TH, nz);
    k_grad_blf_x2<R, POLY><<<grid, 256, smem, st>>>(p);
    return cudaGetLastError();
}

template <int R>
static cudaError_t launch_x2_poly(const BlfParams& p, int nz, cudaStream_t st)
{
    switch (p.x2_poly) {
        case 0: return launch_x2<R, 0>(p, nz, st);
        case 3: return launch_x2<R, 3>(p, nz, st);
        case 5: return launch_x2<R, 5>(p, nz, st);
        case 6: return launch_x2<R, 6>(p, nz, st);
        case 8: return launch_x2<R, 8>(p, nz, st);
        default: return launch_x2<R, 4>(p, nz, st);
    }
}

#endif  // BLFLS_EXPERIMENTS

template <int R, int P, int MODE>
static cudaError_t launch_poly(const BlfParams& p, int nz, cudaStream_t st)
{
#ifndef BLFLS_EXPERIMENTS
    return launch_fixed<R, P, MODE, kPolyDefault<MODE>>(p, nz, st);
#else
    if (p.cols_per_thread == 8) return launch_fixed<R, 8, MODE, 0>(p, nz, st);  // experiment
    // p.poly_period < 0: the per-mode default; otherwise an experiment override
    switch (p.poly_period < 0 ? kPolyDefault<MODE> : p.poly_period) {
        case 0: return launch_fixed<R, P, MODE, 0>(p, nz, st);
        case 4: return launch_fixed<R, P, MODE, 4>(p, nz, st);
        case 5: return launch_fixed<R, P, MODE, 5>(p, nz, st);
        case 8: return launch_fixed<R, P, MODE, 8>(p, nz, st);
        case 12: return launch_fixed<R, P, MODE, 12>(p, nz, st);
        default: return launch_fixed<R, P, MODE, 6>(p, nz, st);
    }
#endif
}

template <int MODE>
static cudaError_t dispatch_mode(const BlfParams& p, int nz, cudaStream_t st)
{
    constexpr int P = 4;
    constexpr int D = kPolyDefault<MODE>;
    if (p.npeers > 0) {
        // fused band exchange: peer-storing instantiations at the BASELINE radii
        // (16-row tiles: a band is a fraction of a large image), any other radius
        // through the generic-radius kernel
        switch (p.radius) {
            case 3: return launch_fixed_th<3, P, MODE, 0, 16, true>(p, nz, st);
            case 5: return launch_fixed_th<5, P, MODE, 0, 16, true>(p, nz, st);
            case 7: return launch_fixed_th<7, P, MODE, 0, 16, true>(p, nz, st);
            case 15: return launch_fixed_th<15, P, MODE, 0, 16, true>(p, nz, st);
            default: return launch_any<MODE>(p, nz, st);
        }
    }
#ifdef BLFLS_EXPERIMENTS
    if constexpr (MODE == 0) {
        if (p.x2_poly >= 0) {
            switch (p.radius) {
                case 3: return launch_x2_poly<3>(p, nz, st);
                case 4: return launch_x2_poly<4>(p, nz, st);
                case 5: return launch_x2_poly<5>(p, nz, st);
                case 6: return launch_x2_poly<6>(p, nz, st);
                case 7: return launch_x2_poly<7>(p, nz, st);
                case 15: return launch_x2_poly<15>(p, nz, st);
                default: break;
            }
        }
    }
    if constexpr (MODE == 2) {
        // experiment only (BLFLS_PACKED_JOINT3=1): FFMA2-packed accumulation.
        // r01 sweep (tools/variant_sweep.py, c5): the unpacked 4-column kernel
        // is faster (0.70 vs 0.64-0.66 of MUFU peak), so it is the default.
        if (p.legacy_joint3 < 0) {
            switch (p.radius) {
                case 3: return launch_joint3<3>(p, nz, st);
                case 5: return launch_joint3<5>(p, nz, st);
                case 7: return launch_joint3<7>(p, nz, st);
                case 11: return launch_joint3<11>(p, nz, st);
                case 15: return launch_joint3<15>(p, nz, st);
                default: break;
            }
        }
    }
#endif
    switch (p.radius) {
        case 1: return launch_fixed<1, P, MODE, D>(p, nz, st);
        case 2: return launch_fixed<2, P, MODE, D>(p, nz, st);
        case 3: return launch_fixed<3, P, MODE, D>(p, nz, st);
        case 4: return launch_fixed<4, P, MODE, D>(p, nz, st);
        case 5: return launch_poly<5, P, MODE>(p, nz, st);
        case 6: return launch_fixed<6, P, MODE, D>(p, nz, st);
        case 7: return launch_poly<7, P, MODE>(p, nz, st);
        case 8: return launch_fixed<8, P, MODE, D>(p, nz, st);
        case 10: return launch_fixed<10, P, MODE, D>(p, nz, st);
        case 12: return launch_fixed<12, P, MODE, D>(p, nz, st);
        case 15: return launch_poly<15, P, MODE>(p, nz, st);
        default: return launch_any<MODE>(p, nz, st);
    }
}

// mode: 0 self, 1 joint per-channel / single-channel, 2 joint shared gray guide (C == 3)
cudaError_t launch_grad_blf(const BlfParams& p, int mode, int batch, cudaStream_t st)
{
    cudaError_t e = cudaSuccess;
    if (mode == 2 && launch_grad_blf_j3r(p, batch, st, &e)) return e;
    if (mode == 2 && launch_grad_blf_j8(p, batch, st, &e)) return e;
    if (mode == 2 && launch_grad_blf_j3(p, batch, st, &e)) return e;
    if (mode != 2 && launch_grad_blf_p2(p, mode, batch, st, &e)) return e;
    switch (mode) {
        case 0: return dispatch_mode<0>(p, batch * p.C, st);
        case 1: return dispatch_mode<1>(p, batch * p.C, st);
        default: return dispatch_mode<2>(p, batch, st);
    }
}

}  // namespace blfls
