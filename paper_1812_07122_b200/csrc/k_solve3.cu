// k_solve3.cu -- persistent, bulk-copy-pipelined row passes of the periodic
// least-squares solve (solver.cpp:88-124).
//
// The row passes of k_solve.cu load a row block, transform it and store it
// with nothing in flight in between; one wave of such CTAs alternates the
// whole GPU between "all loading" and "all computing" and reaches ~45% of
// HBM.  Here a persistent CTA walks row blocks with a ring of STG shared
// staging slots: one elected thread issues `cp.async.bulk` (TMA bulk copies,
// completion counted on an mbarrier) for the rows of block i + STG - 1 while
// all threads fold / transform / store block i.
//
//   r2c : staging = rows of f, Tx, Ty and Ty[y-1] (the divergence fold r =
//         f + lambda (Dx^T Tx + Dy^T Ty)); then the W/2-point complex FFT and
//         the even/odd split into the half spectrum (as k_row_r2c)
//   c2r : staging = half-spectrum rows; then the split's inverse, the
//         inverse FFT and the pixel stores with crop and min/max (as
//         k_row_c2r)
//
// Same arithmetic as k_solve.cu, so results are bit-identical to it.
#include <cstdlib>

#include "blfls_internal.cuh"
#include "fft.cuh"

namespace blfls {

namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p)
{
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init()
{
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity)
{
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra DONE;\n\t"
        "bra WAIT;\n\t"
        "DONE:\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// global -> shared bulk copy (16-byte aligned, size a multiple of 16)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void block_minmax_atomic3(float lo, float hi, uint32_t* slot)
{
    __shared__ float slo[32], shi[32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
        slo[warp] = lo;
        shi[warp] = hi;
    }
    __syncthreads();
    if (warp == 0) {
        const int nw = (blockDim.x + 31) >> 5;
        lo = lane < nw ? slo[lane] : INFINITY;
        hi = lane < nw ? shi[lane] : -INFINITY;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        }
        if (lane == 0) {
            atomicMin(slot, float_to_ordered(lo));
            atomicMax(slot + 1, float_to_ordered(hi));
        }
    }
    __syncthreads();  // slo / shi are reused by the next block
}

}  // namespace

// bytes of a CtFft row strip (ct_pad: one pad slot per 8 elements), 16-aligned
template <class F>
__host__ __device__ constexpr size_t strip_bytes()
{
    return ((size_t)(F::V * F::N - 1 + ((F::V * F::N - 1) >> 3) + 1) * sizeof(float2) + 15) & ~(size_t)15;
}

// Row-block bookkeeping shared by both passes: block b -> (plane, first row).
struct RowBlocks {
    int nrb;     // row blocks per plane
    int total;   // planes * nrb
};

// ---------------------------------------------------------------- r2c --
// smem: [STG][NA][V][W] floats staging (NA = 4 with targets, else 1), then
// the FFT strip (F::smem_bytes(false)), then STG mbarriers.
template <class F, int STG>
__global__ void __launch_bounds__(F::THREADS) k3_row_r2c(const SolveParams p, const F fft, const RowBlocks rb)
{
    extern __shared__ __align__(128) float sm3[];
    constexpr int V = F::V, n = F::N, NT = F::THREADS;
    const int W = p.W, H = p.H;
    const bool fold = p.tx != nullptr;
    const int NA = fold ? 4 : 1;
    const size_t slot_floats = (size_t)NA * V * W;
    float* stage = sm3;
    float2* buf = reinterpret_cast<float2*>(sm3 + STG * (size_t)4 * V * W);
    uint64_t* bar = reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(buf) +
                                                strip_bytes<F>());
    if (threadIdx.x == 0) {
        for (int s = 0; s < STG; ++s) mbar_init(&bar[s], 1);
        mbar_fence_init();
    }
    __syncthreads();

    auto issue = [&](int blk, int s) {  // one thread
        const int plane = blk / rb.nrb, y0 = (blk - plane * rb.nrb) * V;
        const int rows = min(V, H - y0);
        const size_t poff = (size_t)plane * H * W;
        const uint32_t row_bytes = (uint32_t)W * 4u;
        mbar_expect_tx(&bar[s], (uint32_t)(NA * rows) * row_bytes);
        float* dst = stage + (size_t)s * slot_floats;
        for (int v = 0; v < rows; ++v) {
            const int y = y0 + v;
            bulk_g2s(dst + (size_t)v * W, p.f + poff + (size_t)y * W, row_bytes, &bar[s]);
            if (fold) {
                const int ym = y == 0 ? H - 1 : y - 1;
                bulk_g2s(dst + (size_t)(V + v) * W, p.tx + poff + (size_t)y * W, row_bytes, &bar[s]);
                bulk_g2s(dst + (size_t)(2 * V + v) * W, p.ty + poff + (size_t)y * W, row_bytes, &bar[s]);
                bulk_g2s(dst + (size_t)(3 * V + v) * W, p.ty + poff + (size_t)ym * W, row_bytes, &bar[s]);
            }
        }
    };

    const int first = blockIdx.x, step = gridDim.x;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STG - 1; ++s) {
            const int blk = first + s * step;
            if (blk < rb.total) issue(blk, s);
        }
    }
    const float L = p.lambda;
    const int wc = p.wc;
    int it = 0;
    for (int blk = first; blk < rb.total; blk += step, ++it) {
        const int s = it % STG;
        // refill the slot consumed in the previous iteration (freed by its barrier)
        if (threadIdx.x == 0) {
            const int nb = blk + (STG - 1) * step;
            if (nb < rb.total) issue(nb, (it + STG - 1) % STG);
        }
        const int plane = blk / rb.nrb, y0 = (blk - plane * rb.nrb) * V;
        mbar_wait(&bar[s], (uint32_t)((it / STG) & 1));
        const float* sf = stage + (size_t)s * slot_floats;
        // fold from the staged rows into the FFT strip (2 pixels per complex)
        for (int e = threadIdx.x; e < V * n; e += NT) {
            const int v = e / n, j = e - v * n;
            float2 r = make_float2(0.f, 0.f);
            if (y0 + v < H) {
                r = *reinterpret_cast<const float2*>(sf + (size_t)v * W + 2 * j);
                if (fold) {
                    const float* tx = sf + (size_t)(V + v) * W;
                    const float2 a = *reinterpret_cast<const float2*>(tx + 2 * j);
                    const float2 b = *reinterpret_cast<const float2*>(sf + (size_t)(2 * V + v) * W + 2 * j);
                    const float2 c = *reinterpret_cast<const float2*>(sf + (size_t)(3 * V + v) * W + 2 * j);
                    const float am = tx[j == 0 ? W - 1 : 2 * j - 1];
                    r.x = fmaf(L, (am - a.x) + (c.x - b.x), r.x);
                    r.y = fmaf(L, (a.x - a.y) + (c.y - b.y), r.y);
                }
            }
            buf[fft.template pad<false>(e)] = r;
        }
        __syncthreads();  // staging slot s free; strip complete
        fft.template run<false>(buf, false);
        for (int idx = threadIdx.x; idx < V * wc; idx += NT) {
            const int v = idx / wc, k = idx - v * wc;
            const int y = y0 + v;
            if (y >= H) continue;
            const float2 zk = buf[fft.template pad<false>(v * n + (k == n ? 0 : k))];
            const float2 zn = cconj(buf[fft.template pad<false>(v * n + (k == 0 ? 0 : n - k))]);
            const float2 e = cscale(cadd(zk, zn), 0.5f);
            const float2 o = cscale(cmuli(csub(zk, zn), -1.0f), 0.5f);
            p.spec[((size_t)plane * H + y) * p.spitch + k] = cadd(e, cmul(__ldg(&p.post[k]), o));
        }
        __syncthreads();  // strip reads done before the next fold writes it
    }
}

// ---------------------------------------------------------------- c2r --
// smem: [STG][V][SP] float2 staging of spectrum rows (SP = n + 2 complex,
// a multiple of 16 bytes), the FFT strip, STG mbarriers.
template <class F, int STG>
__global__ void __launch_bounds__(F::THREADS) k3_row_c2r(const SolveParams p, const F fft, const RowBlocks rb)
{
    extern __shared__ __align__(128) float sm3[];
    constexpr int V = F::V, n = F::N, NT = F::THREADS;
    constexpr int SP = n + 2;
    const int H = p.H;
    float2* stage = reinterpret_cast<float2*>(sm3);
    float2* buf = stage + (size_t)STG * V * SP;
    uint64_t* bar = reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(buf) +
                                                strip_bytes<F>());
    if (threadIdx.x == 0) {
        for (int s = 0; s < STG; ++s) mbar_init(&bar[s], 1);
        mbar_fence_init();
    }
    __syncthreads();

    auto issue = [&](int blk, int s) {
        const int plane = blk / rb.nrb, y0 = (blk - plane * rb.nrb) * V;
        const int rows = min(V, H - y0);
        const uint32_t row_bytes = (uint32_t)SP * 8u;
        mbar_expect_tx(&bar[s], (uint32_t)rows * row_bytes);
        for (int v = 0; v < rows; ++v)
            bulk_g2s(stage + ((size_t)s * V + v) * SP, p.spec + ((size_t)plane * H + y0 + v) * p.spitch,
                     row_bytes, &bar[s]);
    };

    const int first = blockIdx.x, step = gridDim.x;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STG - 1; ++s) {
            const int blk = first + s * step;
            if (blk < rb.total) issue(blk, s);
        }
    }
    int it = 0;
    for (int blk = first; blk < rb.total; blk += step, ++it) {
        const int s = it % STG;
        if (threadIdx.x == 0) {
            const int nb = blk + (STG - 1) * step;
            if (nb < rb.total) issue(nb, (it + STG - 1) % STG);
        }
        const int plane = blk / rb.nrb, y0 = (blk - plane * rb.nrb) * V;
        mbar_wait(&bar[s], (uint32_t)((it / STG) & 1));
        const float2* ss = stage + (size_t)s * V * SP;
        for (int e = threadIdx.x; e < V * n; e += NT) {
            const int v = e / n, k = e - v * n;
            float2 Z = make_float2(0.f, 0.f);
            if (y0 + v < H) {
                const float2* srow = ss + (size_t)v * SP;
                float2 xk = srow[k];
                float2 xn = srow[n - k];
                if (k == 0) {  // c2r ignores Im of DC and Nyquist
                    xk.y = 0.f;
                    xn.y = 0.f;
                }
                const float2 xnc = cconj(xn);
                const float2 a = cadd(xk, xnc);
                const float2 bb = cmul(csub(xk, xnc), cconj(__ldg(&p.post[k])));
                Z = cadd(a, cmuli(bb, 1.0f));
            }
            buf[fft.template pad<false>(e)] = Z;
        }
        __syncthreads();
        fft.template run<false>(buf, true);
        float lo = INFINITY, hi = -INFINITY;
        float* out = p.out + (size_t)plane * p.oH * p.oW;
        for (int e = threadIdx.x; e < V * n; e += NT) {
            const int v = e / n, j = e - v * n;
            const int y = y0 + v;
            const int yo = y - p.opad;
            if (y >= H || yo < 0 || yo >= p.oH) continue;
            const float2 z = buf[fft.template pad<false>(e)];
            float* orow = out + (size_t)yo * p.oW;
            if (p.opad == 0) {
                *reinterpret_cast<float2*>(orow + 2 * j) = z;
                lo = fminf(lo, fminf(z.x, z.y));
                hi = fmaxf(hi, fmaxf(z.x, z.y));
            } else {
                const int x0 = 2 * j - p.opad;
                if (x0 >= 0 && x0 < p.oW) {
                    orow[x0] = z.x;
                    lo = fminf(lo, z.x);
                    hi = fmaxf(hi, z.x);
                }
                if (x0 + 1 >= 0 && x0 + 1 < p.oW) {
                    orow[x0 + 1] = z.y;
                    lo = fminf(lo, z.y);
                    hi = fmaxf(hi, z.y);
                }
            }
        }
        // block_minmax_atomic3 ends with a barrier: the strip is free again
        if (p.lohi_out != nullptr)
            block_minmax_atomic3(lo, hi, p.lohi_out + 2 * ((p.plane0 + plane) / p.C));
        else
            __syncthreads();
    }
}

// ------------------------------------------------------------ launchers --

// (n = W/2, V rows per block, TV threads per row, STG staging slots)
#define BLFLS_V3_ROWS(X) X(256, 4, 32, 3) X(512, 2, 64, 3) X(960, 1, 128, 3) X(1024, 1, 128, 3) \
    X(2048, 1, 256, 2)

template <class F, int STG>
static cudaError_t launch3(int which, const SolveParams& p, const float2* tw, int planes, int nsm,
                           cudaStream_t st)
{
    F fft{tw};
    RowBlocks rb;
    rb.nrb = (p.H + F::V - 1) / F::V;
    rb.total = rb.nrb * planes;
    const size_t fft_bytes = strip_bytes<F>();
    size_t smem;
    int occ = 0;
    if (which == 0) {
        smem = (size_t)STG * 4 * F::V * p.W * sizeof(float) + fft_bytes + STG * sizeof(uint64_t);
        cudaFuncSetAttribute(k3_row_r2c<F, STG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k3_row_r2c<F, STG>, F::THREADS, smem);
    } else {
        smem = (size_t)STG * F::V * (F::N + 2) * sizeof(float2) + fft_bytes + STG * sizeof(uint64_t);
        cudaFuncSetAttribute(k3_row_c2r<F, STG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k3_row_c2r<F, STG>, F::THREADS, smem);
    }
    if (occ < 1) return cudaErrorInvalidConfiguration;
    const int grid = std::min(rb.total, occ * nsm);
    if (which == 0)
        k3_row_r2c<F, STG><<<grid, F::THREADS, smem, st>>>(p, fft, rb);
    else
        k3_row_c2r<F, STG><<<grid, F::THREADS, smem, st>>>(p, fft, rb);
    return cudaGetLastError();
}

// Row pass `which` (0 r2c, 2 c2r) on the persistent pipelined kernels when a
// geometry exists for n = W/2 (even W, W % 4 == 0); false otherwise.
bool launch_v3_row_pass(int which, const SolveParams& p, int n, const float2* tw, int planes, int nsm,
                        cudaStream_t st, cudaError_t* err)
{
    static const bool enabled = [] {
        const char* e = std::getenv("BLFLS_SOLVE_V3");  // experiment: off by default
        return e != nullptr && std::atoi(e) != 0;
    }();
    if (!enabled || (p.W & 3) != 0 || 2 * n != p.W) return false;
    // bulk copies need 16-byte aligned sources (plane offsets keep the
    // alignment of the base pointers)
    auto al = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
    if (!al(p.f) || (p.tx && (!al(p.tx) || !al(p.ty))) || !al(p.spec)) return false;
#define BLFLS_V3_GO(N, VV, TV, STG)                                                     \
    if (n == N) {                                                                       \
        *err = launch3<CtFft<N, VV, TV>, STG>(which, p, tw, planes, nsm, st);           \
        return true;                                                                    \
    }
    BLFLS_V3_ROWS(BLFLS_V3_GO)
#undef BLFLS_V3_GO
    return false;
}

}  // namespace blfls
