// k_bilateral.cu -- the standalone brute-force (joint) bilateral filter of
// arbitrary planes, blf_brute (bilateral.cpp:28-77), for callers of the
// reference's public filter API (bilateral.hpp:26) rather than the fused
// gradient path of k_blf.cu.
//
// out_c(s) = sum_t w(s,t) src_c(t) / sum_t w(s,t) over the clipped window
// |t - s|_inf <= r, w = exp(-|s-t|^2 / (2 ss^2)) * exp(-|g(s) - g(t)|^2 / (2 sr^2))
// with |.| the Euclidean norm over the CG guide channels (1, or CS).  In fp32
// on the exp2 pipe: the guide is staged pre-multiplied by
// sqrt(log2(e) / (2 sr^2)) and the spatial term is -dx^2 / (2 ss^2) log2(e), so
// w = ex2(cs[|dx|] - sum_c d_c^2) * wrow[|dy|].  Out-of-image halo cells carry a
// guide sentinel (weight exactly 0: the window is clipped, bilateral.cpp:56-57).
//
// Tiling: 256 threads = 16 rows x 16 threads, P = 4 adjacent outputs each; for
// every window row a thread walks the source columns its outputs need
// (P + 2R of them, one shared-memory read per guide / source channel) and
// updates each output whose window contains the column.  Any radius (runtime
// R); shared memory holds (CG + CS) planes of (16 + 2R) x (64 + 2R) floats.
#include <algorithm>
#include <cmath>

#include "blfls_internal.cuh"

namespace blfls {

namespace {

constexpr float kPlainSentinel = 1.0e15f;
constexpr int kPlainP = 4;
constexpr int kPlainTH = 16;
constexpr int kPlainTW = 16 * kPlainP;

__device__ __forceinline__ float ex2_approx(float x)
{
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

struct PlainParams {
    const float* src;    // batch x CS x H x W
    const float* guide;  // batch x CG x H x W (may alias src)
    float* out;          // batch x CS x H x W
    int H, W, R;
    float gscale;        // sqrt(log2(e) / (2 sr^2))
    const float* cs;     // [R + 1] -d^2 log2(e) / (2 ss^2)
    const float* wrow;   // [R + 1] exp2(cs[d])
};

template <int CG, int CS>
__global__ void __launch_bounds__(256) k_blf_plain(PlainParams p)
{
    extern __shared__ float sm[];
    const int R = p.R;
    const int ROWS = kPlainTH + 2 * R, COLS = kPlainTW + 2 * R;
    const int PITCH = COLS;
    float* G = sm;                          // [CG][ROWS][PITCH] scaled guide
    float* S = sm + CG * ROWS * PITCH;      // [CS][ROWS][PITCH] source
    float* tab = S + CS * ROWS * PITCH;     // [R + 1] cs, [R + 1] wrow
    const int H = p.H, W = p.W;
    const int b = blockIdx.z;
    const int tx0 = blockIdx.x * kPlainTW, ty0 = blockIdx.y * kPlainTH;
    const size_t plane = (size_t)H * W;
    const float* gimg = p.guide + (size_t)b * CG * plane;
    const float* simg = p.src + (size_t)b * CS * plane;
    for (int d = threadIdx.x; d <= R; d += blockDim.x) {
        tab[d] = p.cs[d];
        tab[R + 1 + d] = p.wrow[d];
    }
    for (int idx = threadIdx.x; idx < ROWS * COLS; idx += blockDim.x) {
        const int i = idx / COLS, j = idx - i * COLS;
        const int y = ty0 - R + i, x = tx0 - R + j;
        const bool in = y >= 0 && y < H && x >= 0 && x < W;
        const size_t o = (size_t)y * W + x;
#pragma unroll
        for (int c = 0; c < CG; ++c)
            G[(c * ROWS + i) * PITCH + j] = in ? __ldg(gimg + c * plane + o) * p.gscale : kPlainSentinel;
#pragma unroll
        for (int c = 0; c < CS; ++c) S[(c * ROWS + i) * PITCH + j] = in ? __ldg(simg + c * plane + o) : 0.f;
    }
    __syncthreads();

    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int oy = ty0 + ty, ox = tx0 + tx * kPlainP;
    float gs[CG][kPlainP], z[kPlainP], num[CS][kPlainP];
#pragma unroll
    for (int q = 0; q < kPlainP; ++q) {
#pragma unroll
        for (int c = 0; c < CG; ++c) gs[c][q] = G[(c * ROWS + ty + R) * PITCH + tx * kPlainP + q + R];
        z[q] = 0.f;
#pragma unroll
        for (int c = 0; c < CS; ++c) num[c][q] = 0.f;
    }
    for (int dy = -R; dy <= R; ++dy) {
        const int row = ty + R + dy;
        const float wy = tab[R + 1 + (dy < 0 ? -dy : dy)];
        float zr[kPlainP], nr[CS][kPlainP];
#pragma unroll
        for (int q = 0; q < kPlainP; ++q) {
            zr[q] = 0.f;
#pragma unroll
            for (int c = 0; c < CS; ++c) nr[c][q] = 0.f;
        }
        // source column k (relative to the thread's first output) feeds output q at dx = k - R - q
        for (int k = 0; k < kPlainP + 2 * R; ++k) {
            const int col = tx * kPlainP + k;
            float gv[CG], sv[CS];
#pragma unroll
            for (int c = 0; c < CG; ++c) gv[c] = G[(c * ROWS + row) * PITCH + col];
#pragma unroll
            for (int c = 0; c < CS; ++c) sv[c] = S[(c * ROWS + row) * PITCH + col];
#pragma unroll
            for (int q = 0; q < kPlainP; ++q) {
                const int dx = k - R - q;
                if (dx < -R || dx > R) continue;
                float e = tab[dx < 0 ? -dx : dx];
#pragma unroll
                for (int c = 0; c < CG; ++c) {
                    const float d = gs[c][q] - gv[c];
                    e = fmaf(-d, d, e);
                }
                const float w = ex2_approx(e);
                zr[q] += w;
#pragma unroll
                for (int c = 0; c < CS; ++c) nr[c][q] = fmaf(w, sv[c], nr[c][q]);
            }
        }
#pragma unroll
        for (int q = 0; q < kPlainP; ++q) {
            z[q] = fmaf(zr[q], wy, z[q]);
#pragma unroll
            for (int c = 0; c < CS; ++c) num[c][q] = fmaf(nr[c][q], wy, num[c][q]);
        }
    }
    if (oy < H) {
#pragma unroll
        for (int c = 0; c < CS; ++c) {
            float* o = p.out + ((size_t)b * CS + c) * plane + (size_t)oy * W;
#pragma unroll
            for (int q = 0; q < kPlainP; ++q)
                if (ox + q < W) o[ox + q] = num[c][q] / z[q];
        }
    }
}

// forward_gradients (image.cpp:72-95): circular forward differences per plane
__global__ void k_forward_gradients(const float* img, float* gx, float* gy, int H, int W, size_t n)
{
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) {
        const size_t plane = (size_t)H * W;
        const size_t pl = i / plane, r = i - pl * plane;
        const int y = (int)(r / W), x = (int)(r - (size_t)y * W);
        const float* base = img + pl * plane;
        const float v = base[r];
        gx[i] = base[(size_t)y * W + (x + 1 == W ? 0 : x + 1)] - v;
        gy[i] = base[(size_t)(y + 1 == H ? 0 : y + 1) * W + x] - v;
    }
}

}  // namespace

cudaError_t launch_forward_gradients(const float* img, float* gx, float* gy, int planes, int H, int W,
                                     int nsm, cudaStream_t st)
{
    const size_t n = (size_t)planes * H * W;
    const unsigned blocks = (unsigned)std::min<size_t>((n + 255) / 256, (size_t)nsm * 8);
    k_forward_gradients<<<blocks, 256, 0, st>>>(img, gx, gy, H, W, n);
    return cudaGetLastError();
}

size_t blf_plain_smem(int cg, int cs, int R)
{
    return sizeof(float) * ((size_t)(cg + cs) * (kPlainTH + 2 * R) * (kPlainTW + 2 * R) + 2 * (R + 1));
}

cudaError_t launch_blf_plain(const float* src, int cs, const float* guide, int cg, float* out, int batch,
                             int H, int W, int R, double sigma_s, double sigma_r, const float* tables,
                             cudaStream_t st)
{
    PlainParams p;
    p.src = src;
    p.guide = guide;
    p.out = out;
    p.H = H;
    p.W = W;
    p.R = R;
    p.gscale = (float)std::sqrt(1.4426950408889634 / (2.0 * sigma_r * sigma_r));
    p.cs = tables;
    p.wrow = tables + (R + 1);
    const size_t smem = blf_plain_smem(cg, cs, R);
    const dim3 grid((unsigned)((W + kPlainTW - 1) / kPlainTW), (unsigned)((H + kPlainTH - 1) / kPlainTH),
                    (unsigned)batch);
#define BLFLS_PLAIN(CG, CS)                                                                         \
    if (cg == CG && cs == CS) {                                                                    \
        if (smem > 48 * 1024)                                                                      \
            cudaFuncSetAttribute(k_blf_plain<CG, CS>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                 (int)smem);                                                       \
        k_blf_plain<CG, CS><<<grid, 256, smem, st>>>(p);                                           \
        return cudaGetLastError();                                                                 \
    }
    BLFLS_PLAIN(1, 1)
    BLFLS_PLAIN(1, 3)
    BLFLS_PLAIN(3, 3)
#undef BLFLS_PLAIN
    return cudaErrorInvalidValue;
}

}  // namespace blfls
