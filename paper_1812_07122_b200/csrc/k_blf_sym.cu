// k_blf_sym.cu -- brute-force (joint) bilateral filter of the gradient fields
// with each pair weight evaluated ONCE (bilateral.cpp:28-77 semantics).
//
// The weight of bilateral.cpp:58-66 is symmetric,
//   w(s, t) = exp(-|t - s|^2 / (2 sigma_s^2)) exp(-(g_s - g_t)^2 / (8 sigma_r^2)) = w(t, s),
// so the (2r+1)^2 - 1 off-centre taps of every output split into pairs that
// the brute-force kernel (k_blf.cu) evaluates twice, once from each end.  Here
// every unordered pair {s, t} is evaluated once, by its upper (or left) end s,
// and feeds both sums:
//   Z_s += w, N_s += w v_t      (s side, registers of the thread owning s)
//   Z_t += w, N_t += w v_s      (t side, a register strip per window row,
//                                reduced across lanes with shuffles, then
//                                added into a shared ring of row accumulators)
// The exponent is (cs[|dy|] + cs[|dx|]) - (s g_s - s g_t)^2 (k_blf.cu instead
// multiplies each window row's sums by exp2(cs[|dy|])): the same weights up
// to fp32 rounding, and identical for the two ends of a pair.
//
// Tiling: a CTA of NW = 8 warps owns a tile of TWo = 32 P - 2R output columns
// and TH = NG NW - R output rows of one (plane, axis).  Lane l of a warp
// holds P adjacent "source" columns; the warp's 32 P source columns extend R
// beyond the tile on both sides, and the source rows start R above it, so
// every pair with an output end is evaluated inside the CTA (pairs whose
// other end lies in a neighbouring tile are evaluated by both tiles, each
// keeping its own side).  Rows are processed in NG groups of NW (one row per
// warp); inside a group the window rows dy = 0..R are visited in lockstep,
// with a barrier between them so the NW warps' ring updates never overlap.
// Out-of-image samples carry the guide sentinel, as in k_blf.cu: their
// weights with in-image samples are exactly 0.
#include <cstdlib>
#include <type_traits>

#include "blfls_internal.cuh"

namespace blfls {

namespace {

constexpr float kSymSentinel = 1.0e15f;

__device__ __forceinline__ float sym_ex2(float x)
{
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ void sym_decode_range(const uint32_t* lohi, int b, float coef, float& s,
                                                 float& range)
{
    const float lo = ordered_to_float(lohi[2 * b]);
    const float hi = ordered_to_float(lohi[2 * b + 1]);
    range = hi - lo;
    s = range > 0.f ? coef / range : coef;
}

}  // namespace

// MODE 0: self-guided (source = guide = the scaled gradient)
// MODE 1: joint, one source channel, guide channel = image channel (or gray)
template <int R, int P, int NG, int MODE>
struct SymGeom {
    static constexpr int NW = 8;                       // warps (one source row each)
    static constexpr int NT = 32 * NW;
    static constexpr int TWO = 32 * P - 2 * R;         // output columns per tile
    static constexpr int TH = NG * NW - R;             // output rows per tile
    static constexpr int ROWS = TH + 2 * R;            // staged rows: y0 - R .. y0 + TH + R
    static constexpr int COLS = 32 * P + 2 * R;        // staged cols: x0 - 2R .. x0 + TWO + 2R
    static constexpr int PITCH = (COLS + 3) & ~3;
    static constexpr int NA = MODE == 0 ? 1 : 2;       // guide (+ source)
    static constexpr int RING = NW + R;                // live accumulator rows
    static constexpr int SW = P + 2 * R;               // t-side strip width
    static constexpr int KMIN = -((R + P - 1) / P);    // strip chunks relative to the lane
    static constexpr int KMAX = (P + R - 1) / P;
    static constexpr size_t smem_bytes()
    {
        return (size_t)NA * ROWS * PITCH * sizeof(float) + (size_t)2 * RING * 32 * P * sizeof(float);
    }
};

template <int R, int P, int NG, int MODE>
__global__ void __launch_bounds__(256) k_blf_sym(const BlfParams p)
{
    using Gm = SymGeom<R, P, NG, MODE>;
    constexpr int NW = Gm::NW, NT = Gm::NT, TWO = Gm::TWO, TH = Gm::TH, ROWS = Gm::ROWS;
    constexpr int COLS = Gm::COLS, PITCH = Gm::PITCH, RING = Gm::RING, SW = Gm::SW;
    extern __shared__ __align__(16) float sms[];
    float* G = sms;                                   // [ROWS][PITCH] scaled guide gradient
    float* S = sms + ROWS * PITCH;                    // [ROWS][PITCH] raw source gradient (MODE 1)
    float* RZ = sms + Gm::NA * ROWS * PITCH;          // [RING][32 P] t-side sums of w
    float* RN = RZ + RING * 32 * P;                   // [RING][32 P] t-side sums of w v

    const int H = p.H, W = p.W, C = p.C;
    const int axis = blockIdx.z & 1;
    const int pl = blockIdx.z >> 1;                   // plane = b * C + c
    const int b = pl / C, c0 = pl - (pl / C) * C;
    const int x0 = blockIdx.x * TWO;
    const int y0 = p.y0 + blockIdx.y * TH;
    const size_t plane = (size_t)H * W;

    float s, range;
    sym_decode_range(p.lohi, b, p.range_coef, s, range);
    float sg = s, grange = range;
    if (MODE != 0) sym_decode_range(p.glohi, b, p.range_coef, sg, grange);

    // ---- prologue: this axis' circular gradients of the staged window
    const float* fimg = p.f + ((size_t)b * C + c0) * plane;
    const float* gimg = MODE == 0 ? fimg : p.guide + ((size_t)b * p.GC + (p.GC == 1 ? 0 : c0)) * plane;
    for (int idx = threadIdx.x; idx < ROWS * COLS; idx += NT) {
        const int i = idx / COLS, j = idx - (idx / COLS) * COLS;
        const int y = y0 - R + i, x = x0 - 2 * R + j;
        const int o = i * PITCH + j;
        if (y >= 0 && y < H && x >= 0 && x < W) {
            const size_t r0 = (size_t)y * W;
            const size_t n1 = axis == 0 ? r0 + (x + 1 == W ? 0 : x + 1) : (size_t)(y + 1 == H ? 0 : y + 1) * W + x;
            const size_t n0 = r0 + x;
            G[o] = (__ldg(gimg + n1) - __ldg(gimg + n0)) * (MODE == 0 ? s : sg);
            if (MODE == 1) S[o] = __ldg(fimg + n1) - __ldg(fimg + n0);
        } else {
            G[o] = kSymSentinel;
            if (MODE == 1) S[o] = 0.f;
        }
    }
    for (int idx = threadIdx.x; idx < 2 * RING * 32 * P; idx += NT) RZ[idx] = 0.f;
    __syncthreads();

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float oscale;
    if (MODE == 0)
        oscale = p.normalized_out ? 1.f / p.range_coef : 1.f / s;
    else
        oscale = (p.normalized_out && range > 0.f) ? 1.f / range : 1.f;
    float* outp = (axis == 0 ? p.tx : p.ty) + ((size_t)b * C + c0) * ((size_t)p.out_rows * W);
    const int yrow0 = p.out_rows == H ? 0 : p.y0;

#pragma unroll 1
    for (int grp = 0; grp < NG; ++grp) {
        const int rs = grp * NW + warp;               // staged source row (0 .. TH + R - 1)
        const float* Gs = G + rs * PITCH + R + P * lane;
        float gs[P], vs[P], Z[P], N[P];
#pragma unroll
        for (int q = 0; q < P; ++q) {
            gs[q] = Gs[q];
            vs[q] = MODE == 0 ? gs[q] : S[rs * PITCH + R + P * lane + q];
            Z[q] = 1.f;                               // centre tap: weight exp2(0) = 1
            N[q] = vs[q];
        }
        // one window row: pairs (s, t = s + (dy, dx)); dy = 0 takes dx > 0 only
        auto window_row = [&](auto first, int dy) {
            constexpr bool DY0 = decltype(first)::value;
            const int rt = rs + dy;                   // row of the partners t
            const float* Gt = G + rt * PITCH + P * lane;
            const float* St = S + rt * PITCH + P * lane;
            const float cy = p.cs[dy];
            float ce[R + 1];                          // log2 spatial weight of (dy, |dx|)
#pragma unroll
            for (int k = 0; k <= R; ++k) ce[k] = cy + p.cs[k];
            float sz[SW], sn[SW];
#pragma unroll
            for (int j = 0; j < SW; ++j) {
                sz[j] = 0.f;
                sn[j] = 0.f;
            }
#pragma unroll
            for (int j4 = 0; j4 < SW; j4 += 4) {
                if (DY0 && j4 + 3 < R + 1) continue;  // no partner in this float4
                const float4 g4 = *reinterpret_cast<const float4*>(Gt + j4);
                float4 v4 = g4;
                if (MODE == 1) v4 = *reinterpret_cast<const float4*>(St + j4);
                const float gt[4] = {g4.x, g4.y, g4.z, g4.w};
                const float vt[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int j = j4 + u;
                    if (j >= SW) break;
#pragma unroll
                    for (int q = 0; q < P; ++q) {
                        const int dx = j - q - R;
                        if (dx < -R || dx > R) continue;
                        if (DY0 && dx <= 0) continue;
                        const float d = gs[q] - gt[u];
                        const float w = sym_ex2(fmaf(-d, d, ce[dx < 0 ? -dx : dx]));
                        Z[q] += w;
                        N[q] = fmaf(w, vt[u], N[q]);
                        sz[j] += w;
                        sn[j] = fmaf(w, vs[q], sn[j]);
                    }
                }
            }
            // strip column j <-> source column P lane + j - R: chunk k = floor((j - R) / P)
            // belongs to lane + k; lane l collects chunk k of lane l - k
            float oz[P], on[P];
#pragma unroll
            for (int q = 0; q < P; ++q) {
                oz[q] = sz[R + q];
                on[q] = sn[R + q];
            }
#pragma unroll
            for (int k = Gm::KMIN; k <= Gm::KMAX; ++k) {
                if (k == 0) continue;
#pragma unroll
                for (int q = 0; q < P; ++q) {
                    const int j = R + P * k + q;
                    if (j < 0 || j >= SW) continue;
                    if (DY0 && j < R + 1) continue;   // never written for dy = 0
                    float az, an;
                    if (k > 0) {
                        az = __shfl_up_sync(0xffffffffu, sz[j], k);
                        an = __shfl_up_sync(0xffffffffu, sn[j], k);
                    } else {
                        az = __shfl_down_sync(0xffffffffu, sz[j], -k);
                        an = __shfl_down_sync(0xffffffffu, sn[j], -k);
                    }
                    const bool ok = k > 0 ? lane >= k : lane < 32 + k;
                    oz[q] += ok ? az : 0.f;
                    on[q] += ok ? an : 0.f;
                }
            }
            float* rz = RZ + (rt % RING) * 32 * P + P * lane;
            float* rn = RN + (rt % RING) * 32 * P + P * lane;
            if constexpr (P == 4) {
                float4 a = *reinterpret_cast<float4*>(rz), c = *reinterpret_cast<float4*>(rn);
                a.x += oz[0]; a.y += oz[1]; a.z += oz[2]; a.w += oz[3];
                c.x += on[0]; c.y += on[1]; c.z += on[2]; c.w += on[3];
                *reinterpret_cast<float4*>(rz) = a;
                *reinterpret_cast<float4*>(rn) = c;
            } else {
#pragma unroll
                for (int q = 0; q < P; ++q) {
                    rz[q] += oz[q];
                    rn[q] += on[q];
                }
            }
            __syncthreads();  // the next dy's ring rows belong to this dy's neighbour warps
        };
        window_row(std::true_type{}, 0);
#pragma unroll 1
        for (int dy = 1; dy <= R; ++dy) window_row(std::false_type{}, dy);
        // ---- row rs complete (its partners above were delivered by earlier rows)
        float* rz = RZ + (rs % RING) * 32 * P + P * lane;
        float* rn = RN + (rs % RING) * 32 * P + P * lane;
        const int y = y0 - R + rs;
        if (rs >= R && y < p.y1 && y < y0 + TH) {
#pragma unroll
            for (int q = 0; q < P; ++q) {
                const int xc = P * lane + q - R;      // output column within the tile
                const int x = x0 + xc;
                if (xc >= 0 && xc < TWO && x < W)
                    outp[(size_t)(y - yrow0) * W + x] = (N[q] + rn[q]) / (Z[q] + rz[q]) * oscale;
            }
        }
#pragma unroll
        for (int q = 0; q < P; ++q) {
            rz[q] = 0.f;
            rn[q] = 0.f;
        }
        __syncthreads();
    }
}

template <int R, int P, int NG, int MODE>
static cudaError_t launch_sym(const BlfParams& p, int nplanes, cudaStream_t st)
{
    using Gm = SymGeom<R, P, NG, MODE>;
    constexpr size_t smem = Gm::smem_bytes();
    cudaError_t e = cudaFuncSetAttribute(k_blf_sym<R, P, NG, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    dim3 grid((p.W + Gm::TWO - 1) / Gm::TWO, (p.y1 - p.y0 + Gm::TH - 1) / Gm::TH, 2 * nplanes);
    k_blf_sym<R, P, NG, MODE><<<grid, Gm::NT, smem, st>>>(p);
    return cudaGetLastError();
}

// groups per tile: NG = 8 (taller tiles, less halo work) when the grid still
// fills ~2 waves of 4 CTAs per SM, else NG = 4
template <int R, int MODE>
static cudaError_t launch_sym_ng(const BlfParams& p, int nplanes, cudaStream_t st)
{
    static const int forced = [] {
        const char* e = std::getenv("BLFLS_SYM_NG");
        return e ? std::atoi(e) : 0;
    }();
    constexpr int NGL = R >= 12 ? 16 : 8, NGS = R >= 12 ? 8 : 4;
    using GL = SymGeom<R, 4, NGL, MODE>;
    const long ctas = (long)((p.W + GL::TWO - 1) / GL::TWO) * ((p.y1 - p.y0 + GL::TH - 1) / GL::TH) * 2 * nplanes;
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const bool large = forced ? forced == NGL : ctas >= 8L * nsm;
    if (large) return launch_sym<R, 4, NGL, MODE>(p, nplanes, st);
    return launch_sym<R, 4, NGS, MODE>(p, nplanes, st);
}

template <int MODE>
static bool dispatch_sym(const BlfParams& p, int nplanes, cudaStream_t st, cudaError_t* err)
{
    switch (p.radius) {
        case 3: *err = launch_sym_ng<3, MODE>(p, nplanes, st); return true;
        case 5: *err = launch_sym_ng<5, MODE>(p, nplanes, st); return true;
        case 7: *err = launch_sym_ng<7, MODE>(p, nplanes, st); return true;
        case 15: *err = launch_sym_ng<15, MODE>(p, nplanes, st); return true;
        default: return false;
    }
}

// Pair-symmetric brute-force filter for modes 0 (self) and 1 (per-channel
// joint); false when no instantiation covers the request (the caller then
// runs k_blf.cu).  Experiment, enabled by BLFLS_BLF_SYM=1: measured on B200
// (r01) it halves the MUFU work but is issue-bound at ~9 instructions per
// pair (t-side strip, shuffle reduction, per-window-row barriers) and the
// halo tiles add 25-45% pairs, so it ties with k_blf.cu (c2 -1..+3%, c3 -3%,
// c4 -2%).
bool launch_grad_blf_sym(const BlfParams& p, int mode, int batch, cudaStream_t st, cudaError_t* err)
{
    static const bool enabled = [] {
        const char* e = std::getenv("BLFLS_BLF_SYM");  // experiment: off by default (r01)
        return e != nullptr && std::atoi(e) != 0;
    }();
    // row bands keep the brute-force kernel: its per-output summation order
    // does not depend on the tiling, so bands reproduce the full image bit for bit
    if (!enabled || p.npeers > 0 || mode == 2 || p.y0 != 0 || p.y1 != p.H) return false;
    if (mode == 0) return dispatch_sym<0>(p, batch * p.C, st, err);
    return dispatch_sym<1>(p, batch * p.C, st, err);
}

}  // namespace blfls
