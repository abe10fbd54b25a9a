// k_solve2.cu -- the periodic least-squares solve (solver.cpp:88-124) on the
// high-radix engine of fft2.cuh.  Same three passes and the same arithmetic
// contract as k_solve.cu (divergence fold, 1/(H W den) with a correctly
// rounded reciprocal, min/max epilogue), but each pass touches shared memory
// only between its FFT stages:
//
//   row r2c : stage 0 reads the fold r = f + lambda (Dx^T Tx + Dy^T Ty)
//             straight from global; the even/odd split reads the last stage
//             from shared memory and writes the half spectrum
//   column  : forward stage 0 reads the spectrum column strip from global;
//             the inverse's stage 0 applies 1 / (H W den) to its inputs; the
//             inverse's last stage writes the strip back to global
//   row c2r : stage 0 builds the half-length complex row from the spectrum
//             (global); the last stage writes the pixels (crop for padded
//             grids) and reduces the next iteration's min/max
//
// Geometries exist for the even-width BASELINE sizes; every other size (and
// the stage entry points' forward-only / inverse-only column modes) runs the
// kernels of k_solve.cu.
#include "blfls_internal.cuh"
#include <algorithm>
#include <cstdlib>

#include "fft2.cuh"

namespace blfls {

__device__ __forceinline__ void block_minmax_atomic2(float lo, float hi, uint32_t* slot)
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
}

// grid (ceil(H / V), planes); n = W / 2 complex points per row
template <class G>
__global__ void __launch_bounds__(G::THREADS) k2_row_r2c(const SolveParams p, const float2* __restrict__ tw)
{
    extern __shared__ __align__(16) float2 buf[];
    constexpr int n = G::N;
    const int v = threadIdx.x / G::TV, t = threadIdx.x - v * G::TV;
    const int plane = blockIdx.y;
    const int y = blockIdx.x * G::V + v;
    const bool live = y < p.H;
    const int W = p.W;
    const size_t poff = (size_t)plane * p.H * W;
    const size_t roff = poff + (size_t)(live ? y : 0) * W;
    const size_t rprev = poff + (size_t)(live ? (y == 0 ? p.H - 1 : y - 1) : 0) * W;
    const float L = p.lambda;
    const bool fold = p.tx != nullptr;
    auto ld = [&](int j) -> float2 {
        if (!live) return make_float2(0.f, 0.f);
        float2 r = __ldg(reinterpret_cast<const float2*>(p.f + roff) + j);
        if (fold) {
            const float2 a = __ldg(reinterpret_cast<const float2*>(p.tx + roff) + j);
            const float2 b = __ldg(reinterpret_cast<const float2*>(p.ty + roff) + j);
            const float2 c = __ldg(reinterpret_cast<const float2*>(p.ty + rprev) + j);
            const float am = __ldg(p.tx + roff + (j == 0 ? W - 1 : 2 * j - 1));
            r.x = fmaf(L, (am - a.x) + (c.x - b.x), r.x);
            r.y = fmaf(L, (a.x - a.y) + (c.y - b.y), r.y);
        }
        return r;
    };
    auto st = [&](int j, float2 z) { buf[G::ra(v, j)] = z; };
    s2_stage<G, false, 0, false>(t, tw, ld, st);
    __syncthreads();
    s2_smem_stages<G, false, false, 1, G::NST>(buf, v, t, tw);
    // even/odd split: X_k = (Z_k + conj Z_{n-k}) / 2 + e^{-2 pi i k / W} (Z_k - conj Z_{n-k}) / (2i)
    const int wc = p.wc;
    for (int idx = threadIdx.x; idx < G::V * wc; idx += G::THREADS) {
        const int vv = idx / wc, k = idx - vv * wc;
        const int yy = blockIdx.x * G::V + vv;
        if (yy >= p.H) continue;
        const float2 zk = buf[G::ra(vv, k == n ? 0 : k)];
        const float2 zn = cconj(buf[G::ra(vv, k == 0 ? 0 : n - k)]);
        const float2 e = cscale(cadd(zk, zn), 0.5f);
        const float2 o = cscale(cmuli(csub(zk, zn), -1.0f), 0.5f);
        p.spec[((size_t)plane * p.H + yy) * p.spitch + k] = cadd(e, cmul(__ldg(&p.post[k]), o));
    }
}

// The column FFT pair (forward, 1 / den, inverse) of r01 / early r02.  The
// production solve runs the column pass as a cyclic tridiagonal solve
// (k_col_tri.cu, launch_col in k_solve.cu); these kernels remain in the
// experiments build for A/B runs (BLFLS_COL_TRI=0).
#ifdef BLFLS_EXPERIMENTS
// grid (ceil(wc / V), planes): V adjacent spectrum columns, forward FFT,
// 1 / (H W (1 + lambda (4 sin^2(pi u/H) + 4 sin^2(pi v/W)))), inverse FFT
template <class G>
__global__ void __launch_bounds__(G::THREADS, G::THREADS <= 512 ? 65536 / (64 * G::THREADS) : 1) k2_col(const SolveParams p, const float2* __restrict__ tw)
{
    extern __shared__ __align__(16) float2 buf[];
    const int v = threadIdx.x % G::V, t = threadIdx.x / G::V;
    const int plane = blockIdx.y;
    const int vc = blockIdx.x * G::V + v;
    const bool live = vc < p.wc;
    float2* spec = p.spec + (size_t)plane * G::N * p.spitch + (live ? vc : 0);
    const size_t sp = p.spitch;
    auto ldg = [&](int u) -> float2 { return live ? __ldcg(spec + (size_t)u * sp) : make_float2(0.f, 0.f); };
    auto sts = [&](int u, float2 z) { buf[G::ca(v, u)] = z; };
    auto lds = [&](int u) { return buf[G::ca(v, u)]; };
    s2_stage<G, false, 0, false>(t, tw, ldg, sts);
    __syncthreads();
    const float gx = live ? __ldg(&p.gain_x[vc]) : 0.f;
    const float L = p.lambda, ihw = p.inv_hw;
    auto stg = [&](int u, float2 z) {
        if (live) spec[(size_t)u * sp] = z;
    };
    if constexpr (G::NST == 1) {
        s2_smem_stages<G, true, false, 1, G::NST>(buf, v, t, tw);
        auto lds_scaled = [&](int u) {
            const float sc = ihw * __frcp_rn(fmaf(L, __ldg(&p.gain_y[u]) + gx, 1.0f));
            return cscale(buf[G::ca(v, u)], sc);
        };
        s2_stage<G, true, 0, false>(t, tw, lds_scaled, stg);
    } else {
        // forward stages 1 .. NST-2 in shared memory, then the forward's last
        // stage and the inverse's first (reversed radix order) in registers
        // with 1 / (H W den) in between (fft2.cuh s2_fwd_last_inv_first)
        using R = typename G::Rev;
        s2_smem_stages<G, true, false, 1, G::NST - 1>(buf, v, t, tw);
        auto scale = [&](int u) { return ihw * __frcp_rn(fmaf(L, __ldg(&p.gain_y[u]) + gx, 1.0f)); };
        s2_fwd_last_inv_first<G>(t, tw, lds, scale, sts);
        __syncthreads();
        s2_smem_stages<R, true, true, 1, R::NST - 1>(buf, v, t, tw);
        s2_stage<R, true, R::NST - 1, false>(t, tw, lds, stg);
    }
}

// Pipelined column pass: persistent CTAs stride over the column strips
// (plane-major) with two shared buffers; the next strip is copied in by
// 16-byte cp.async while the current one is transformed, so the global loads
// never stall the transform (k2_col's stage 0 reads global memory directly
// and every CTA alternates load / transform / store phases).  Same
// arithmetic as k2_col (stage 0 runs from shared memory), bit-identical
// spectra.  Strips past wc read the spectrum's pad columns (spitch is a
// multiple of 16 >= roundup(wc, V)); their results are not stored.
template <class G>
constexpr int col_pipe_minb()
{
    return (int)((227u * 1024u) / (2 * G::smem_bytes() + 1024)) > 0
               ? (int)((227u * 1024u) / (2 * G::smem_bytes() + 1024))
               : 1;
}

template <class G>
__global__ void __launch_bounds__(G::THREADS, col_pipe_minb<G>())
    k2_col_pipe(const SolveParams p, const float2* __restrict__ tw, int nsp, int total)
{
    extern __shared__ __align__(16) float2 buf2[];
    constexpr int N = G::N, V = G::V, BUF = G::PADN * G::V;
    static_assert(V % 2 == 0, "16-byte chunks of two columns");
    const int v = threadIdx.x % V, t = threadIdx.x / V;
    const size_t sp = p.spitch;
    auto issue = [&](int s, float2* dst) {
        const int plane = s / nsp, c0 = (s - plane * nsp) * V;
        const float2* src = p.spec + (size_t)plane * N * sp + c0;
        for (int c = threadIdx.x; c < N * V / 2; c += G::THREADS) {
            const int u = c / (V / 2), h = c - u * (V / 2);
            const unsigned d = (unsigned)__cvta_generic_to_shared(dst + G::ca(2 * h, u));
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src + (size_t)u * sp + 2 * h)
                         : "memory");
        }
    };
    int s = blockIdx.x;
    if (s >= total) return;
    issue(s, buf2);
    asm volatile("cp.async.commit_group;" ::: "memory");
    for (int k = 0; s < total; s += gridDim.x, ++k) {
        float2* buf = buf2 + (k & 1) * BUF;
        const int sn = s + gridDim.x;
        if (sn < total) issue(sn, buf2 + ((k + 1) & 1) * BUF);
        asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group 1;" ::: "memory");
        __syncthreads();  // strip s landed
        const int plane = s / nsp;
        const int vc = (s - plane * nsp) * V + v;
        const bool live = vc < p.wc;
        float2* spec = p.spec + (size_t)plane * N * sp + (live ? vc : 0);
        auto lds = [&](int u) { return buf[G::ca(v, u)]; };
        auto sts = [&](int u, float2 z) { buf[G::ca(v, u)] = z; };
        const float gx = live ? __ldg(&p.gain_x[vc]) : 0.f;
        const float L = p.lambda, ihw = p.inv_hw;
        auto stg = [&](int u, float2 z) {
            if (live) spec[(size_t)u * sp] = z;
        };
        if constexpr (G::NST == 1) {
            s2_smem_stages<G, true, false, 0, G::NST>(buf, v, t, tw);
            auto lds_scaled = [&](int u) {
                const float sc = ihw * __frcp_rn(fmaf(L, __ldg(&p.gain_y[u]) + gx, 1.0f));
                return cscale(buf[G::ca(v, u)], sc);
            };
            s2_stage<G, true, 0, true>(t, tw, lds_scaled, stg);
        } else {
            using R = typename G::Rev;
            s2_smem_stages<G, true, false, 0, G::NST - 1>(buf, v, t, tw);
            auto scale = [&](int u) { return ihw * __frcp_rn(fmaf(L, __ldg(&p.gain_y[u]) + gx, 1.0f)); };
            s2_fwd_last_inv_first<G>(t, tw, lds, scale, sts);
            __syncthreads();
            s2_smem_stages<R, true, true, 1, R::NST - 1>(buf, v, t, tw);
            s2_stage<R, true, R::NST - 1, false>(t, tw, lds, stg);
        }
        __syncthreads();  // buf free for the copies of strip s + 2 gridDim.x
    }
}

#endif  // BLFLS_EXPERIMENTS

// grid (ceil(H / V), planes)
template <class G>
__global__ void __launch_bounds__(G::THREADS) k2_row_c2r(const SolveParams p, const float2* __restrict__ tw)
{
    extern __shared__ __align__(16) float2 buf[];
    constexpr int n = G::N;
    const int v = threadIdx.x / G::TV, t = threadIdx.x - v * G::TV;
    const int plane = blockIdx.y;
    const int y = blockIdx.x * G::V + v;
    const bool live = y < p.H;
    const float2* srow = p.spec + ((size_t)plane * p.H + (live ? y : 0)) * p.spitch;
    // Z_k = (X_k + conj X_{n-k}) + i e^{+2 pi i k / W} (X_k - conj X_{n-k}); c2r
    // ignores Im of DC and Nyquist
    auto ldg = [&](int k) -> float2 {
        if (!live) return make_float2(0.f, 0.f);
        float2 xk = __ldcg(srow + k);
        float2 xn = __ldcg(srow + (n - k));
        if (k == 0) {
            xk.y = 0.f;
            xn.y = 0.f;
        }
        const float2 xnc = cconj(xn);
        const float2 a = cadd(xk, xnc);
        const float2 bb = cmul(csub(xk, xnc), cconj(__ldg(&p.post[k])));
        return cadd(a, cmuli(bb, 1.0f));
    };
    auto sts = [&](int j, float2 z) { buf[G::ra(v, j)] = z; };
    auto lds = [&](int j) { return buf[G::ra(v, j)]; };
    float lo = INFINITY, hi = -INFINITY;
    const int yo = y - p.opad;
    const bool out_row = live && yo >= 0 && yo < p.oH;
    float* orow = p.out + (size_t)plane * p.oH * p.oW + (size_t)(out_row ? yo : 0) * p.oW;
    auto sto = [&](int j, float2 z) {
        if (!out_row) return;
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
    };
    if constexpr (G::NST == 1) {
        s2_stage<G, true, 0, false>(t, tw, ldg, sto);
    } else {
        s2_stage<G, true, 0, false>(t, tw, ldg, sts);
        __syncthreads();
        s2_smem_stages<G, false, true, 1, G::NST - 1>(buf, v, t, tw);
        s2_stage<G, true, G::NST - 1, false>(t, tw, lds, sto);
    }
    if (p.lohi_out != nullptr) block_minmax_atomic2(lo, hi, p.lohi_out + 2 * ((p.plane0 + plane) / p.C));
}

// ---------------------------------------------------- TMA bulk-copy c2r --
// Persistent row c2r: CTAs stride over tiles of V spectrum rows (plane-major).
// The V padded rows of a tile are contiguous in the half spectrum (pitch
// spitch), so ONE bulk copy (cp.async.bulk, the TMA engine: SASS UBLKCP)
// moves them into a shared landing buffer, completing on an mbarrier; two
// landing buffers, so tile k + 1's copy is in flight while tile k is
// transformed.  Stage 0 then builds the half-length complex rows from shared
// memory instead of two dependent global loads per element (k2_row_c2r's top
// stall, 39-47% long-scoreboard at c5).  Same arithmetic and output order as
// k2_row_c2r: bit-identical images and min/max.
__device__ __forceinline__ void tma_mbar_init(uint64_t* bar, unsigned count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)),
                 "r"(count)
                 : "memory");
}
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar)
{
    const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     (unsigned)__cvta_generic_to_shared(dst)),
                 "l"(src), "r"(bytes), "r"(b)
                 : "memory");
}
__device__ __forceinline__ void tma_mbar_wait(uint64_t* bar, unsigned parity)
{
    const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
    unsigned done = 0;
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
            : "=r"(done)
            : "r"(b), "r"(parity)
            : "memory");
    }
}

template <class G>
__global__ void __launch_bounds__(G::THREADS, 2) k2_row_c2r_tma(const SolveParams p, const float2* __restrict__ tw,
                                                            int tiles_per_plane, int total)
{
    extern __shared__ __align__(128) float2 smc[];
    constexpr int n = G::N, V = G::V;
    const int sp = p.spitch;
    float2* buf = smc;                                                     // FFT work buffer
    float2* land = smc + ((G::smem_bytes() / sizeof(float2) + 15) & ~(size_t)15);  // [2][V][spitch]
    __shared__ __align__(8) uint64_t bar[2];
    const int v = threadIdx.x / G::TV, t = threadIdx.x - v * G::TV;
    auto tile_src = [&](int tile, int& plane, int& y0, int& rows) {
        plane = tile / tiles_per_plane;
        y0 = (tile - plane * tiles_per_plane) * V;
        rows = min(V, p.H - y0);
    };
    auto issue = [&](int tile, int s) {
        int plane, y0, rows;
        tile_src(tile, plane, y0, rows);
        tma_bulk_g2s(land + (size_t)s * V * sp, p.spec + ((size_t)plane * p.H + y0) * sp,
                     (unsigned)(rows * sp * sizeof(float2)), &bar[s]);
    };
    if (threadIdx.x == 0) {
        tma_mbar_init(&bar[0], 1);
        tma_mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    int tile = blockIdx.x;
    if (threadIdx.x == 0) {
        if (tile < total) issue(tile, 0);
        if (tile + (int)gridDim.x < total) issue(tile + gridDim.x, 1);
    }
    for (int k = 0; tile < total; ++k, tile += gridDim.x) {
        const int s = k & 1;
        int plane, y0, rows;
        tile_src(tile, plane, y0, rows);
        const int y = y0 + v;
        const bool live = v < rows;
        const float2* srow = land + ((size_t)s * V + v) * sp;
        auto ld = [&](int kk) -> float2 {
            if (!live) return make_float2(0.f, 0.f);
            float2 xk = srow[kk];
            float2 xn = srow[n - kk];
            if (kk == 0) {
                xk.y = 0.f;
                xn.y = 0.f;
            }
            const float2 xnc = cconj(xn);
            const float2 a = cadd(xk, xnc);
            const float2 bb = cmul(csub(xk, xnc), cconj(__ldg(&p.post[kk])));
            return cadd(a, cmuli(bb, 1.0f));
        };
        auto sts = [&](int j, float2 z) { buf[G::ra(v, j)] = z; };
        auto lds = [&](int j) { return buf[G::ra(v, j)]; };
        float lo = INFINITY, hi = -INFINITY;
        const int yo = y - p.opad;
        const bool out_row = live && yo >= 0 && yo < p.oH;
        float* orow = p.out + (size_t)plane * p.oH * p.oW + (size_t)(out_row ? yo : 0) * p.oW;
        auto sto = [&](int j, float2 z) {
            if (!out_row) return;
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
        };
        tma_mbar_wait(&bar[s], (k >> 1) & 1);
        s2_stage<G, true, 0, false>(t, tw, ld, sts);
        __syncthreads();  // landing[s] consumed, buffer written
        if (threadIdx.x == 0 && tile + 2 * (int)gridDim.x < total) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(tile + 2 * gridDim.x, s);
        }
        s2_smem_stages<G, false, true, 1, G::NST - 1>(buf, v, t, tw);
        s2_stage<G, true, G::NST - 1, false>(t, tw, lds, sto);
        if (p.lohi_out != nullptr) block_minmax_atomic2(lo, hi, p.lohi_out + 2 * ((p.plane0 + plane) / p.C));
        __syncthreads();  // buf reads of the last stage done before the next tile's stage 0
    }
}

// ------------------------------------------------------------ launchers --

// Row geometries (N = W/2, V rows, TV threads per row, PMAX) and column
// geometries (N = H, V columns, TV threads per column, PMAX).  No radix-16
// row geometry for n = 960 (c3): its 15 x 16 x 4 c2r measured slower than
// the radix-8 engine's (31 vs 27 us per iteration); no radix-16 column
// geometry for H = 512 (c1: 15.9 vs 12.1 us).
// Radix-32 geometries (PMAX 32) are experiment-only (BLFLS_V2_PMAX_*=32):
// too many registers (94-201), slower than radix 16 everywhere (r01).
#define BLFLS_V2_ROWS16(X) X(256, 8, 16, 16) X(512, 8, 32, 16) X(512, 2, 32, 16) \
    X(1024, 4, 64, 16) X(1024, 1, 64, 16) X(2048, 2, 128, 16) X(2048, 1, 128, 16)
#define BLFLS_V2_COLS16(X) X(1024, 4, 64, 16) X(1024, 2, 64, 16) X(1080, 4, 72, 16) \
    X(2048, 4, 128, 16) X(2048, 2, 128, 16) X(4096, 2, 256, 16) X(4096, 4, 256, 16)
#ifdef BLFLS_EXPERIMENTS
#define BLFLS_V2_ROWS(X) BLFLS_V2_ROWS16(X) X(256, 16, 8, 32) X(256, 4, 8, 32) X(512, 8, 16, 32) \
    X(512, 2, 16, 32) X(960, 8, 32, 32) X(960, 2, 32, 32) X(1024, 8, 32, 32) X(1024, 2, 32, 32) \
    X(2048, 4, 64, 32) X(2048, 1, 64, 32)
#define BLFLS_V2_COLS(X) BLFLS_V2_COLS16(X) X(512, 8, 16, 32) X(512, 2, 16, 32) X(1024, 4, 32, 32) \
    X(1024, 2, 32, 32) X(1080, 8, 36, 32) X(1080, 4, 40, 32) X(2048, 4, 64, 32) X(2048, 2, 64, 32) \
    X(4096, 4, 128, 32) X(4096, 2, 128, 32)
#else
#define BLFLS_V2_ROWS(X) BLFLS_V2_ROWS16(X)
#define BLFLS_V2_COLS(X) BLFLS_V2_COLS16(X)
#endif

template <class K>
static void set_smem2(K kernel, size_t smem)
{
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

template <class G>
static void launch2(int which, const SolveParams& p, const float2* tw, int planes, cudaStream_t st)
{
    constexpr size_t smem = G::smem_bytes();
    if (which == 1) {
#ifdef BLFLS_EXPERIMENTS
        // BLFLS_COL_PIPE: 1 pipelined column pass, 0 plain; unset = pipelined
        // for power-of-two columns up to 1024 whose spectra stay L2-resident
        // (c2 column 62 -> 57 us per step; c3's 1080, the HBM-streaming c5 and
        // L2-resident 2048-point groups of c5 measured slower,
        // profiles/r01_solve_knobs_c23.txt)
        static const int pipe_env = knob("BLFLS_COL_PIPE", -1);
        const size_t spec_bytes = (size_t)planes * G::N * p.spitch * sizeof(float2);
        const bool pipe = pipe_env >= 0 ? pipe_env != 0
                                        : ((G::N & (G::N - 1)) == 0 && G::N <= 1024 && spec_bytes <= ((size_t)48 << 20));
        if constexpr (G::V % 2 == 0) {
            if (pipe) {
                const int nsp = (p.wc + G::V - 1) / G::V;
                const int total = nsp * planes;
                // two strip buffers must fit the opt-in shared memory (4096-point
                // columns at V = 4 need 278,592 B > 227 KB: the plain pass runs)
                int occ = 0, dev = 0, nsm = 148, optin = 0;
                cudaGetDevice(&dev);
                cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
                cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
                if (2 * smem <= (size_t)optin &&
                    cudaFuncSetAttribute(k2_col_pipe<G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)(2 * smem)) == cudaSuccess &&
                    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k2_col_pipe<G>, G::THREADS, 2 * smem) ==
                        cudaSuccess &&
                    occ > 0) {
                    const int grid = std::min(total, occ * nsm);
                    k2_col_pipe<G><<<grid, G::THREADS, 2 * smem, st>>>(p, tw, nsp, total);
                    return;
                }
                (void)cudaGetLastError();  // a failed opt-in leaves no sticky error
            }
        }
        dim3 grid((p.wc + G::V - 1) / G::V, planes);
        set_smem2(k2_col<G>, smem);
        k2_col<G><<<grid, G::THREADS, smem, st>>>(p, tw);
#endif
    } else if (which == 0) {
        dim3 grid((p.H + G::V - 1) / G::V, planes);
        set_smem2(k2_row_r2c<G>, smem);
        k2_row_r2c<G><<<grid, G::THREADS, smem, st>>>(p, tw);
    } else {
        // the TMA-fed persistent c2r for streaming workloads (spectra beyond
        // L2, power-of-two rows of a multi-stage geometry): BLFLS_C2R_TMA
        static const int tma = knob("BLFLS_C2R_TMA", 1);
        const size_t spec_bytes = (size_t)planes * p.H * p.spitch * sizeof(float2);
        if constexpr (G::NST > 1) {
            if (tma && spec_bytes > ((size_t)64 << 20)) {
                const size_t land = (size_t)2 * G::V * p.spitch * sizeof(float2);
                const size_t sm2 = ((smem + 127) & ~(size_t)127) + land;
                int occ = 0, dev = 0, nsm = 148, optin = 0;
                cudaGetDevice(&dev);
                cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
                cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
                if (sm2 <= (size_t)optin &&
                    cudaFuncSetAttribute(k2_row_c2r_tma<G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)sm2) == cudaSuccess &&
                    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k2_row_c2r_tma<G>, G::THREADS, sm2) ==
                        cudaSuccess &&
                    occ > 0) {
                    const int tpp = (p.H + G::V - 1) / G::V;
                    const long total = (long)tpp * planes;
                    const int grid = (int)std::min<long>(total, (long)occ * nsm);
                    k2_row_c2r_tma<G><<<grid, G::THREADS, sm2, st>>>(p, tw, tpp, (int)total);
                    return;
                }
                (void)cudaGetLastError();
            }
        }
        dim3 grid((p.H + G::V - 1) / G::V, planes);
        set_smem2(k2_row_c2r<G>, smem);
        k2_row_c2r<G><<<grid, G::THREADS, smem, st>>>(p, tw);
    }
}

// Runs pass `which` (0 row r2c, 1 column, 2 row c2r) on the high-radix
// engine when a geometry exists for length n; returns false otherwise.  The
// widest geometry that still launches >= 2 CTAs per SM is chosen.
bool launch_v2_pass(int which, const SolveParams& p, int n, const float2* tw, int planes, int nsm,
                    cudaStream_t st)
{
    static const bool disabled = (knob("BLFLS_FFT_V1", 0) != 0);
    if (disabled) return false;
    if (which == 1 && p.mode != 3) return false;
#ifndef BLFLS_EXPERIMENTS
    if (which == 1) return false;  // mode 3 is k_col_tri; modes 1 / 2 run k_col (k_solve.cu)
#endif
    // passes routed here (bit 0 row r2c, bit 1 column, bit 2 row c2r)
    static const int passes = knob("BLFLS_V2_PASSES", 6);  // column + row c2r (streaming ncu, r01)
    if (!((passes >> which) & 1)) return false;
    // radix cap of the row / column engines (experiment knob; default 32)
    static const int pmax_rows = knob("BLFLS_V2_PMAX_ROWS", 16);
    static const int pmax_cols = knob("BLFLS_V2_PMAX_COLS", 16);
    const int pmax = which == 1 ? pmax_cols : pmax_rows;
    const int nvec = which == 1 ? p.wc : p.H;
    int bestV = 0, narrowV = 1 << 30;
    auto consider = [&](int N, int V, int PM) {
        if (N != n || PM != pmax) return;
        const long ctas = (long)planes * ((nvec + V - 1) / V);
        if (ctas >= 2L * nsm && V > bestV) bestV = V;
        if (V < narrowV) narrowV = V;
    };
#define BLFLS_V2_CONSIDER(N, V, TV, PM) consider(N, V, PM);
    if (which == 1) {
        BLFLS_V2_COLS(BLFLS_V2_CONSIDER)
    } else {
        BLFLS_V2_ROWS(BLFLS_V2_CONSIDER)
    }
#undef BLFLS_V2_CONSIDER
    int V = bestV ? bestV : narrowV;
    if (V == 1 << 30) return false;
    // experiment knob: force the vectors per CTA of the column / row passes
    static const int forceV[2] = {knob("BLFLS_V2_ROWV", 0),
                                  knob("BLFLS_V2_COLV", 0)};
    if (const int fv = forceV[which == 1 ? 1 : 0]) {
        bool have = false;
#define BLFLS_V2_HAVE(N, VV, TV, PM) have = have || (N == n && VV == fv && PM == pmax);
        if (which == 1) {
            BLFLS_V2_COLS(BLFLS_V2_HAVE)
        } else {
            BLFLS_V2_ROWS(BLFLS_V2_HAVE)
        }
#undef BLFLS_V2_HAVE
        if (have) V = fv;
    }
#define BLFLS_V2_GO(N, VV, TV, PM)                                  \
    if (n == N && V == VV && pmax == PM) {                          \
        launch2<Fft2<N, VV, TV, PM>>(which, p, tw, planes, st);     \
        return true;                                                \
    }
    if (which == 1) {
        BLFLS_V2_COLS(BLFLS_V2_GO)
    } else {
        BLFLS_V2_ROWS(BLFLS_V2_GO)
    }
#undef BLFLS_V2_GO
    return false;
}

}  // namespace blfls
