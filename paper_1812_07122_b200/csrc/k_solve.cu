// k_solve.cu -- periodic least-squares solve (solver.cpp:88-124) as three
// kernels over one half spectrum per plane:
//
//   row r2c  : r = f + lambda (Dx^T Tx + Dy^T Ty)   (divergence fold, exact:
//              conj(otf) F(T) = F(D^T T); Dx^T t[x] = t[x-1] - t[x], circular)
//              then the W-point real FFT of each row as a W/2-point complex
//              Stockham FFT plus the even/odd split (post-twiddle exp(-2 pi i v/W))
//   column   : H-point FFT of V adjacent spectrum columns, divide by
//              H W (1 + lambda (4 sin^2(pi u/H) + 4 sin^2(pi v/W))), inverse FFT
//              (solver.cpp:117-118 with the 1/(hw) of fft2d.cpp:49-51 folded in)
//   row c2r  : inverse real FFT of each row, written as the next image; the
//              epilogue reduces min/max for the next iteration's normalisation
//              (image.cpp:46-60) with ordered-integer atomics.
//
// Spectrum layout: plane-major, H rows of `spitch` complex64 (W/2+1 used).
#include "blfls_internal.cuh"
#include "fft.cuh"

namespace blfls {

__device__ __forceinline__ float fold_value(const SolveParams& p, const float* f, const float* tx,
                                            const float* ty, int y, int x)
{
    float v = f[(size_t)y * p.W + x];
    if (tx != nullptr) {
        const int xm = x == 0 ? p.W - 1 : x - 1;
        const int ym = y == 0 ? p.H - 1 : y - 1;
        const float dx = tx[(size_t)y * p.W + xm] - tx[(size_t)y * p.W + x];
        const float dy = ty[(size_t)ym * p.W + x] - ty[(size_t)y * p.W + x];
        v = fmaf(p.lambda, dx + dy, v);
    }
    return v;
}

// grid: (ceil(H / V), planes); V rows per CTA; n = W/2 (even W) or W (odd W)
template <bool ODD, class F>
__global__ void __launch_bounds__(F::kMaxThreads, F::kRowMinBlocks) k_row_r2c(const SolveParams p, const F fft)
{
    extern __shared__ __align__(16) float2 buf[];
    const int n = fft.n(), V = fft.vecs();
    const int plane = blockIdx.y;
    const int row0 = blockIdx.x * V;
    const size_t poff = (size_t)plane * p.H * p.W;
    const float* f = p.f + poff;
    const float* tx = p.tx ? p.tx + poff : nullptr;
    const float* ty = p.ty ? p.ty + poff : nullptr;
    if (!ODD && (p.W & 3) == 0) {
        // 4 pixels (2 complex) per thread: float4 loads of f, Tx, Ty and the
        // previous Ty row; Tx[x-1] is one scalar load (fold r = f + lambda D^T T)
        const int w4 = fft.n() >> 1;  // = W / 4, compile-time for the CT engine
#pragma unroll
        for (int e = threadIdx.x; e < V * w4; e += fft.threads()) {
            const int v = e / w4, x4 = e - v * w4;
            const int y = row0 + v;
            float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
            if (y < p.H) {
                const size_t o = (size_t)y * p.W + 4 * x4;
                r = __ldg(reinterpret_cast<const float4*>(f + o));
                if (tx != nullptr) {
                    const int ym = y == 0 ? p.H - 1 : y - 1;
                    const float4 a = __ldg(reinterpret_cast<const float4*>(tx + o));
                    const float4 b = __ldg(reinterpret_cast<const float4*>(ty + o));
                    const float4 c = __ldg(reinterpret_cast<const float4*>(ty + (size_t)ym * p.W + 4 * x4));
                    const float am = __ldg(tx + (size_t)y * p.W + (x4 == 0 ? p.W - 1 : 4 * x4 - 1));
                    const float L = p.lambda;
                    r.x = fmaf(L, (am - a.x) + (c.x - b.x), r.x);
                    r.y = fmaf(L, (a.x - a.y) + (c.y - b.y), r.y);
                    r.z = fmaf(L, (a.y - a.z) + (c.z - b.z), r.z);
                    r.w = fmaf(L, (a.z - a.w) + (c.w - b.w), r.w);
                }
            }
            const int j = v * n + 2 * x4;
            buf[fft.template pad<false>(j)] = make_float2(r.x, r.y);
            buf[fft.template pad<false>(j + 1)] = make_float2(r.z, r.w);
        }
    } else {
        for (int idx = threadIdx.x; idx < V * n; idx += blockDim.x) {
            const int v = idx / n, j = idx - (idx / n) * n;
            const int y = row0 + v;
            float2 z = make_float2(0.f, 0.f);
            if (y < p.H) {
                if (!ODD) {
                    z.x = fold_value(p, f, tx, ty, y, 2 * j);
                    z.y = fold_value(p, f, tx, ty, y, 2 * j + 1);
                } else {
                    z.x = fold_value(p, f, tx, ty, y, j);
                }
            }
            buf[fft.template pad<false>(idx)] = z;
        }
    }
    __syncthreads();
    fft.template run<false>(buf, false);
    const int wc = p.wc;
    for (int idx = threadIdx.x; idx < V * wc; idx += fft.threads()) {
        const int v = idx / wc, k = idx - (idx / wc) * wc;
        const int y = row0 + v;
        if (y >= p.H) continue;
        float2 X;
        if (!ODD) {
            const float2 zk = buf[fft.template pad<false>(v * n + (k == n ? 0 : k))];
            const float2 zn = cconj(buf[fft.template pad<false>(v * n + (k == 0 ? 0 : n - k))]);
            const float2 e = cscale(cadd(zk, zn), 0.5f);
            const float2 o = cscale(cmuli(csub(zk, zn), -1.0f), 0.5f);  // (zk - zn) / (2i)
            X = cadd(e, cmul(__ldg(&p.post[k]), o));
        } else {
            X = buf[fft.template pad<false>(v * n + k)];
        }
        p.spec[((size_t)plane * p.H + y) * p.spitch + k] = X;
    }
}

// ------------------------------------------------ TMA bulk-copy row r2c --
// Persistent row r2c (even W, W % 4 == 0, targets present) for streaming
// solves: a tile is V rows of one plane.  Its inputs are contiguous rows --
// f and Tx rows [y0, y0 + V), Ty rows [y0 - 1, y0 + V) (row H - 1 for the
// circular Ty[y - 1] of row 0) -- so three or four bulk copies (the TMA
// engine, SASS UBLKCP) land them in shared memory, completing on an mbarrier.
// One landing buffer: the next tile's copies are issued as soon as this
// tile's fold has read it, so they fly during the FFT and the spectrum
// stores.  The fold reads shared memory instead of four dependent float4
// global loads per 4 pixels (k_row_r2c's top stall, 27% long-scoreboard at
// c5).  Same arithmetic and order as k_row_r2c: bit-identical spectra.
__device__ __forceinline__ void r2c_mbar_init(uint64_t* bar)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)) : "memory");
}
__device__ __forceinline__ void r2c_bulk(void* dst, const void* src, unsigned bytes, uint64_t* bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     (unsigned)__cvta_generic_to_shared(dst)),
                 "l"(src), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(bar))
                 : "memory");
}
__device__ __forceinline__ void r2c_expect(uint64_t* bar, unsigned bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                     (unsigned)__cvta_generic_to_shared(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void r2c_wait(uint64_t* bar, unsigned parity)
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

template <class F>
__global__ void __launch_bounds__(1024) k_row_r2c_tma(const SolveParams p, const F fft, int tiles_per_plane,
                                                      int total)
{
    extern __shared__ __align__(128) float2 buf[];
    constexpr int n = F::N, V = F::V, W = 2 * F::N;
    // landing rows after the FFT buffer: f [V][W], tx [V][W], ty [V + 1][W]
    float* land = reinterpret_cast<float*>(buf) + ((F::smem_bytes(false) / sizeof(float) + 31) & ~(size_t)31);
    float* lf = land;
    float* ltx = land + V * W;
    float* lty = land + 2 * V * W;  // row 0 = Ty[y0 - 1]
    __shared__ __align__(8) uint64_t bar;
    auto tile_of = [&](int tile, int& plane, int& y0, int& rows) {
        plane = tile / tiles_per_plane;
        y0 = (tile - plane * tiles_per_plane) * V;
        rows = min(V, p.H - y0);
    };
    auto issue = [&](int tile) {  // one thread
        int plane, y0, rows;
        tile_of(tile, plane, y0, rows);
        const size_t po = (size_t)plane * p.H * W;
        const unsigned rb = (unsigned)(rows * W * sizeof(float)), wb = (unsigned)(W * sizeof(float));
        r2c_expect(&bar, 3 * rb + wb);
        r2c_bulk(lf, p.f + po + (size_t)y0 * W, rb, &bar);
        r2c_bulk(ltx, p.tx + po + (size_t)y0 * W, rb, &bar);
        if (y0 > 0) {
            r2c_bulk(lty, p.ty + po + (size_t)(y0 - 1) * W, rb + wb, &bar);
        } else {
            r2c_bulk(lty, p.ty + po + (size_t)(p.H - 1) * W, wb, &bar);
            r2c_bulk(lty + W, p.ty + po, rb, &bar);
        }
    };
    if (threadIdx.x == 0) {
        r2c_mbar_init(&bar);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    int tile = blockIdx.x;
    if (threadIdx.x == 0 && tile < total) issue(tile);
    for (int k = 0; tile < total; ++k, tile += gridDim.x) {
        int plane, y0, rows;
        tile_of(tile, plane, y0, rows);
        r2c_wait(&bar, k & 1);
        // fold r = f + lambda (Dx^T Tx + Dy^T Ty), 4 pixels (2 complex) per thread
        constexpr int w4 = W / 4;
        const float L = p.lambda;
#pragma unroll
        for (int e = threadIdx.x; e < V * w4; e += F::THREADS) {
            const int v = e / w4, x4 = e - v * w4;
            float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
            if (v < rows) {
                const int o = v * W + 4 * x4;
                r = *reinterpret_cast<const float4*>(lf + o);
                const float4 a = *reinterpret_cast<const float4*>(ltx + o);
                const float4 b = *reinterpret_cast<const float4*>(lty + W + o);
                const float4 c = *reinterpret_cast<const float4*>(lty + o);
                const float am = ltx[v * W + (x4 == 0 ? W - 1 : 4 * x4 - 1)];
                r.x = fmaf(L, (am - a.x) + (c.x - b.x), r.x);
                r.y = fmaf(L, (a.x - a.y) + (c.y - b.y), r.y);
                r.z = fmaf(L, (a.y - a.z) + (c.z - b.z), r.z);
                r.w = fmaf(L, (a.z - a.w) + (c.w - b.w), r.w);
            }
            const int j = v * n + 2 * x4;
            buf[fft.template pad<false>(j)] = make_float2(r.x, r.y);
            buf[fft.template pad<false>(j + 1)] = make_float2(r.z, r.w);
        }
        __syncthreads();  // landing consumed: the next tile's copies may land now
        if (threadIdx.x == 0 && tile + (int)gridDim.x < total) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(tile + gridDim.x);
        }
        fft.template run<false>(buf, false);
        const int wc = p.wc;
        for (int idx = threadIdx.x; idx < V * wc; idx += F::THREADS) {
            const int v = idx / wc, kk = idx - (idx / wc) * wc;
            const int y = y0 + v;
            if (v >= rows) continue;
            const float2 zk = buf[fft.template pad<false>(v * n + (kk == n ? 0 : kk))];
            const float2 zn = cconj(buf[fft.template pad<false>(v * n + (kk == 0 ? 0 : n - kk))]);
            const float2 e = cscale(cadd(zk, zn), 0.5f);
            const float2 o = cscale(cmuli(csub(zk, zn), -1.0f), 0.5f);
            p.spec[((size_t)plane * p.H + y) * p.spitch + kk] = cadd(e, cmul(__ldg(&p.post[kk]), o));
        }
        __syncthreads();  // buf reads done before the next fold writes it
    }
}

// grid: (ceil(wc / V), planes); V adjacent columns per CTA, layout buf[u*V + c]
template <class F>
__global__ void __launch_bounds__(1024) k_col(const SolveParams p, const F fft)
{
    extern __shared__ __align__(16) float2 buf[];
    const int H = fft.n(), V = fft.vecs();  // compile-time for the CT engine
    const int plane = blockIdx.y;
    const int v0 = blockIdx.x * V;
    float2* spec = p.spec + (size_t)plane * H * p.spitch;
    // cp.async (LDGSTS) straight into the padded strip: every copy of the
    // thread is in flight at once instead of one load per loop trip
    for (int idx = threadIdx.x; idx < V * H; idx += fft.threads()) {
        const int u = idx / V, c = idx - (idx / V) * V;
        const int v = v0 + c;
        float2* dst = buf + fft.template pad<true>(idx);
        if (v < p.wc) {
            const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa),
                         "l"(spec + (size_t)u * p.spitch + v));
        } else {
            *dst = make_float2(0.f, 0.f);
        }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    if (p.mode & 1) fft.template run<true>(buf, false);
    if (p.mode & 2) {
        for (int idx = threadIdx.x; idx < V * H; idx += fft.threads()) {
            const int u = idx / V, c = idx - (idx / V) * V;
            const int v = v0 + c;
            float sc = p.inv_hw;
            if (p.mode == 3 && v < p.wc)
                sc = p.inv_hw * __frcp_rn(fmaf(p.lambda, __ldg(&p.gain_y[u]) + __ldg(&p.gain_x[v]), 1.0f));
            const int pi = fft.template pad<true>(idx);
            buf[pi] = cscale(buf[pi], sc);
        }
        __syncthreads();
        fft.template run<true>(buf, true);
    }
    for (int idx = threadIdx.x; idx < V * H; idx += fft.threads()) {
        const int u = idx / V, c = idx - (idx / V) * V;
        const int v = v0 + c;
        if (v < p.wc) spec[(size_t)u * p.spitch + v] = buf[fft.template pad<true>(idx)];
    }
}

__device__ __forceinline__ void block_minmax_atomic(float lo, float hi, uint32_t* slot)
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

// grid: (ceil(H / V), planes)
template <bool ODD, class F>
__global__ void __launch_bounds__(1024) k_row_c2r(const SolveParams p, const F fft)
{
    extern __shared__ __align__(16) float2 buf[];
    const int n = fft.n(), V = fft.vecs();
    const int plane = blockIdx.y;
    const int row0 = blockIdx.x * V;
    const int W = p.W;
#pragma unroll 8
    for (int idx = threadIdx.x; idx < V * n; idx += fft.threads()) {
        const int v = idx / n, k = idx - (idx / n) * n;
        const int y = row0 + v;
        float2 Z = make_float2(0.f, 0.f);
        if (y < p.H) {
            const float2* srow = p.spec + ((size_t)plane * p.H + y) * p.spitch;
            if (!ODD) {
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
            } else {
                if (k <= (W - 1) / 2) {
                    Z = srow[k];
                    if (k == 0) Z.y = 0.f;
                } else {
                    Z = cconj(srow[W - k]);
                }
            }
        }
        buf[fft.template pad<false>(idx)] = Z;
    }
    __syncthreads();
    fft.template run<false>(buf, true);
    float lo = INFINITY, hi = -INFINITY;
    // crop (reflect-padded grids): only rows/cols [opad, opad + oH/oW) are written
    float* out = p.out + (size_t)plane * p.oH * p.oW;
    for (int idx = threadIdx.x; idx < V * n; idx += fft.threads()) {
        const int v = idx / n, j = idx - (idx / n) * n;
        const int y = row0 + v;
        const int yo = y - p.opad;
        if (y >= p.H || yo < 0 || yo >= p.oH) continue;
        const float2 z = buf[fft.template pad<false>(idx)];
        float* orow = out + (size_t)yo * p.oW;
        if (!ODD && p.opad == 0) {
            *reinterpret_cast<float2*>(orow + 2 * j) = z;
            lo = fminf(lo, fminf(z.x, z.y));
            hi = fmaxf(hi, fmaxf(z.x, z.y));
        } else if (!ODD) {
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
        } else {
            const int xo = j - p.opad;
            if (xo >= 0 && xo < p.oW) {
                orow[xo] = z.x;
                lo = fminf(lo, z.x);
                hi = fmaxf(hi, z.x);
            }
        }
    }
    if (p.lohi_out != nullptr) block_minmax_atomic(lo, hi, p.lohi_out + 2 * ((p.plane0 + plane) / p.C));
}

// ---------------------------------------------------------------- misc --

// per-image min/max over all channels; grid (blocks, batch)
__global__ void k_minmax(const float* __restrict__ x, size_t per_image, uint32_t* lohi)
{
    const float* xi = x + (size_t)blockIdx.y * per_image;
    float lo = INFINITY, hi = -INFINITY;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if ((per_image & 3) == 0 && (reinterpret_cast<uintptr_t>(xi) & 15) == 0) {
        const float4* x4 = reinterpret_cast<const float4*>(xi);
        for (size_t k = i; k < per_image / 4; k += stride) {
            const float4 t = __ldg(x4 + k);
            lo = fminf(lo, fminf(fminf(t.x, t.y), fminf(t.z, t.w)));
            hi = fmaxf(hi, fmaxf(fmaxf(t.x, t.y), fmaxf(t.z, t.w)));
        }
    } else {
        for (size_t k = i; k < per_image; k += stride) {
            const float t = __ldg(xi + k);
            lo = fminf(lo, t);
            hi = fmaxf(hi, t);
        }
    }
    block_minmax_atomic(lo, hi, lohi + 2 * blockIdx.y);
}

__global__ void k_reset_lohi(uint32_t* lohi, int n)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        lohi[2 * i] = 0xffffffffu;
        lohi[2 * i + 1] = 0u;
    }
}

// counts non-finite samples (require_finite, image.cpp:21-27)
__global__ void k_count_nonfinite(const float* __restrict__ x, size_t n, unsigned* count)
{
    unsigned local = 0;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x)
        local += !isfinite(__ldg(x + i));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
    if ((threadIdx.x & 31) == 0 && local) atomicAdd(count, local);
}

// reflect padding without edge repeat (image.cpp:185-212): dst (H+2pad) x
// (W+2pad) per plane from src H x W; grid-stride over all planes
__device__ __forceinline__ int reflect_index(int q, int n)
{
    if (n == 1) return 0;
    const int period = 2 * (n - 1);
    q = abs(q) % period;
    return q < n ? q : period - q;
}

__global__ void k_reflect_pad(const float* __restrict__ src, float* __restrict__ dst, int H, int W,
                              int pad, size_t planes)
{
    const int Hp = H + 2 * pad, Wp = W + 2 * pad;
    const size_t per = (size_t)Hp * Wp, total = per * planes;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (size_t)gridDim.x * blockDim.x) {
        const size_t pl = i / per, r = i - pl * per;
        const int y = (int)(r / Wp), x = (int)(r - (size_t)y * Wp);
        const int sy = reflect_index(y - pad, H), sx = reflect_index(x - pad, W);
        dst[i] = __ldg(src + pl * H * W + (size_t)sy * W + sx);
    }
}

cudaError_t launch_reflect_pad(const float* src, float* dst, int H, int W, int pad, size_t planes,
                               int nsm, cudaStream_t st)
{
    size_t total = (size_t)(H + 2 * pad) * (W + 2 * pad) * planes;
    size_t blocks = (total + 255) / 256;
    if (blocks > (size_t)nsm * 16) blocks = (size_t)nsm * 16;
    k_reflect_pad<<<(unsigned)blocks, 256, 0, st>>>(src, dst, H, W, pad, planes);
    return cudaGetLastError();
}

// targets in normalised units -> raw: t * (hi - lo) (stage entry helper)
__global__ void k_scale_by_range(float* x, size_t per_image, const uint32_t* lohi, int to_raw)
{
    const float lo = ordered_to_float(lohi[2 * blockIdx.y]);
    const float hi = ordered_to_float(lohi[2 * blockIdx.y + 1]);
    const float r = hi - lo;
    const float sc = r > 0.f ? (to_raw ? r : 1.f / r) : (to_raw ? 0.f : 1.f);
    float* xi = x + (size_t)blockIdx.y * per_image;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < per_image;
         i += (size_t)gridDim.x * blockDim.x)
        xi[i] *= sc;
}

// SplitMix64 draw j of the stream `seed` (testimage.cpp:11-21: state += gamma, mix)
__device__ __forceinline__ uint64_t splitmix_at(uint64_t seed, uint64_t j)
{
    uint64_t z = seed + (j + 1) * 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
__device__ __forceinline__ double uniform_at(uint64_t seed, uint64_t j)
{
    return (double)(splitmix_at(seed, j) >> 11) * 0x1.0p-53;
}

// BASELINE synthetic generator; grid (ceil(H*W/256), planes).  Draw
// layout (the test checker restates it): sites at draws 3s..3s+2,
// pixel i at 3K + 3i + {0, 1, 2}.
__global__ void k_generate(int H, int W, const uint64_t* seeds, int K, double noise_sigma, double p_sp,
                           float* out)
{
    extern __shared__ double site[];  // 3K doubles
    const uint64_t seed = seeds[blockIdx.y];
    for (int s = threadIdx.x; s < K; s += blockDim.x) {
        site[3 * s] = uniform_at(seed, 3 * (uint64_t)s) * W;
        site[3 * s + 1] = uniform_at(seed, 3 * (uint64_t)s + 1) * H;
        site[3 * s + 2] = uniform_at(seed, 3 * (uint64_t)s + 2);
    }
    __syncthreads();
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (size_t)H * W) return;
    const int y = (int)(i / W), x = (int)(i % W);
    int best = 0;
    double bd = 1e300;
    for (int s = 0; s < K; ++s) {
        const double dx = x - site[3 * s], dy = y - site[3 * s + 1];
        const double dd = dx * dx + dy * dy;
        if (dd < bd) {
            bd = dd;
            best = s;
        }
    }
    const double rx = W > 1 ? 1.0 / (W - 1) : 0.0;
    const double ry = H > 1 ? 1.0 / (H - 1) : 0.0;
    double v = site[3 * best + 2] + 0.2 * ((x * rx + y * ry) * 0.5 - 0.5);
    const uint64_t base = 3 * (uint64_t)K;
    const double u1 = uniform_at(seed, base + 3 * i);
    const double u2 = uniform_at(seed, base + 3 * i + 1);
    v += noise_sigma * sqrt(-2.0 * log(1.0 - u1)) * cos(2.0 * 3.14159265358979323846 * u2);
    if (p_sp > 0.0) {
        const double u3 = uniform_at(seed, base + 3 * i + 2);
        if (u3 < 0.5 * p_sp)
            v = 0.0;
        else if (u3 < p_sp)
            v = 1.0;
    }
    v = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
    out[(size_t)blockIdx.y * H * W + i] = (float)v;
}

// -------------------------------------------------------------- launchers --

template <class K>
static void set_smem(K kernel, size_t smem)
{
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

// which = 0 row r2c, 1 column, 2 row c2r
template <class F>
static void launch_pass(int which, const SolveParams& p, const F& f, int V, int n, int threads,
                        int planes, bool odd, cudaStream_t st)
{
    const size_t smem = f.smem_bytes(which == 1);
    if (which == 1) {
        dim3 grid((p.wc + V - 1) / V, planes);
        set_smem(k_col<F>, smem);
        k_col<F><<<grid, threads, smem, st>>>(p, f);
        return;
    }
    dim3 grid((p.H + V - 1) / V, planes);
#ifdef BLFLS_EXPERIMENTS
    if constexpr (F::kCompileTime) {
        // the TMA-fed persistent r2c (experiments build, BLFLS_R2C_TMA=1):
        // measured slower than k_row_r2c (r02 B200: c5 9.22 vs 8.83 ms per
        // step, c4 175 vs 164 us) -- the 56 KB landing rows leave 3 CTAs per
        // SM where k_row_r2c runs 6, and its global loads were not the limit
        // (issue 70% active)
        static const int tma = knob("BLFLS_R2C_TMA", 0);
        const size_t in_bytes = (size_t)planes * p.H * p.W * 3 * sizeof(float);
        if (which == 0 && !odd && tma && p.tx != nullptr && (p.W % 4) == 0 && in_bytes > ((size_t)128 << 20)) {
            const size_t sm2 = ((smem + 127) & ~(size_t)127) + (size_t)(3 * F::V + 1) * p.W * sizeof(float);
            int occ = 0, dev = 0, nsm = 148, optin = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
            cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
            if (sm2 <= (size_t)optin &&
                cudaFuncSetAttribute(k_row_r2c_tma<F>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2) ==
                    cudaSuccess &&
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_row_r2c_tma<F>, threads, sm2) == cudaSuccess &&
                occ > 0) {
                const int tpp = (p.H + V - 1) / V;
                const long total = (long)tpp * planes;
                const int g = (int)std::min<long>(total, (long)occ * nsm);
                k_row_r2c_tma<F><<<g, threads, sm2, st>>>(p, f, tpp, (int)total);
                return;
            }
            (void)cudaGetLastError();
        }
    }
#endif
    if (which == 0) {
        if (odd) { set_smem(k_row_r2c<true, F>, smem); k_row_r2c<true, F><<<grid, threads, smem, st>>>(p, f); }
        else { set_smem(k_row_r2c<false, F>, smem); k_row_r2c<false, F><<<grid, threads, smem, st>>>(p, f); }
    } else {
        if (odd) { set_smem(k_row_c2r<true, F>, smem); k_row_c2r<true, F><<<grid, threads, smem, st>>>(p, f); }
        else { set_smem(k_row_c2r<false, F>, smem); k_row_c2r<false, F><<<grid, threads, smem, st>>>(p, f); }
    }
}

// Compile-time geometries of the BASELINE sizes (N, V vectors per CTA, TV
// threads per vector).  Rows: ~256 threads, one radix-8 butterfly per thread
// per stage, n = W/2 for W in {512, 1024, 1920, 2048, 4096}.  Columns: 512
// threads and <= 64 KB so two CTAs share an SM (4096 needs 1024 threads),
// V*8 >= 32-byte row segments (V = 4: whole 32-byte sectors per row, measured
// -13% on the c2 column pass against V = 2), H in {512, 1024, 1080, 2048, 4096}.  Narrow
// variants (small V) keep small images from running a handful of CTAs.
#define BLFLS_CT_ROWS(X) X(256, 8, 32) X(256, 2, 32) X(512, 4, 64) X(512, 1, 64) X(960, 2, 128) \
    X(1024, 2, 128) X(2048, 1, 256) BLFLS_CT_ROWS_PAD16(X)
#define BLFLS_CT_COLS(X) X(512, 16, 32) X(512, 2, 64) X(1024, 8, 64) X(1024, 4, 128) X(1024, 2, 128) \
    X(1080, 4, 128) X(2048, 4, 128) X(4096, 4, 256) BLFLS_CT_COLS_PAD16(X)
// the reference's default reflect padding (pad 16) of the power-of-two
// BASELINE sizes: 544 = 2^5 17, 1056 = 2^5 3 11, 2080 = 2^5 5 13 (rows: half)
#define BLFLS_CT_ROWS_PAD16(X) X(272, 8, 32) X(272, 2, 32) X(528, 4, 64) X(528, 1, 64) \
    X(1040, 2, 128) X(1040, 1, 128)
#define BLFLS_CT_COLS_PAD16(X) X(544, 16, 32) X(544, 2, 64) X(1056, 8, 64) X(1056, 4, 128) X(1056, 2, 128) \
    X(2080, 4, 128)

// Largest-V geometry that still launches >= 2 CTAs per SM for `planes`
// planes; otherwise the narrowest one.
// nvec: vectors per plane (spectrum columns W/2+1, or image rows H)
bool ct_geometry(bool cols, int n, int nvec, int planes, int nsm, int* V, int* threads)
{
    int bestV = 0, bestT = 0, narrowV = 1 << 30, narrowT = 0;
    auto consider = [&](int N, int VV, int TV) {
        if (n != N) return;
        const long ctas = (long)planes * ((nvec + VV - 1) / VV);
        if (ctas >= 2L * nsm && VV > bestV) {
            bestV = VV;
            bestT = VV * TV;
        }
        if (VV < narrowV) {
            narrowV = VV;
            narrowT = VV * TV;
        }
    };
#define BLFLS_GEOM(N, VV, TV) consider(N, VV, TV);
    if (cols) {
        BLFLS_CT_COLS(BLFLS_GEOM)
    } else {
        BLFLS_CT_ROWS(BLFLS_GEOM)
    }
#undef BLFLS_GEOM
    if (bestV) {
        *V = bestV;
        *threads = bestT;
        return true;
    }
    if (narrowT) {
        *V = narrowV;
        *threads = narrowT;
        return true;
    }
    return false;
}

static cudaError_t launch_fft_pass(int which, const SolveParams& p, const FftGeom& g, int planes,
                                   bool odd, cudaStream_t st)
{
    const int n = g.desc.n;
    if (!odd && !g.bluestein) {  // high-radix engine (k_solve2.cu) where a geometry exists
        int dev = 0, nsm = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        if (launch_v2_pass(which, p, n, g.desc.tw, planes, nsm, st)) return cudaGetLastError();
    }
    if (g.ct && !odd) {
#define BLFLS_CT_LAUNCH(N, VV, TV)                                                          \
    if (n == N && g.V == VV) {                                                             \
        launch_pass(which, p, CtFft<N, VV, TV>{g.desc.tw}, VV, N, VV * TV, planes, odd, st); \
        return cudaGetLastError();                                                         \
    }
        if (which == 1) {
            BLFLS_CT_COLS(BLFLS_CT_LAUNCH)
        } else {
            BLFLS_CT_ROWS(BLFLS_CT_LAUNCH)
        }
#undef BLFLS_CT_LAUNCH
    }
    if (g.E == 16) {
        if (g.generic)
            launch_pass(which, p, RtFft<16, true>{g.desc, g.V, g.log2V, g.direct, g.pmax, g.bluestein, g.blue}, g.V, n, g.threads, planes, odd, st);
        else
            launch_pass(which, p, RtFft<16, false>{g.desc, g.V, g.log2V, false, 0, g.bluestein, g.blue}, g.V, n, g.threads, planes, odd, st);
    } else {
        if (g.generic)
            launch_pass(which, p, RtFft<8, true>{g.desc, g.V, g.log2V, g.direct, g.pmax, g.bluestein, g.blue}, g.V, n, g.threads, planes, odd, st);
        else
            launch_pass(which, p, RtFft<8, false>{g.desc, g.V, g.log2V, false, 0, g.bluestein, g.blue}, g.V, n, g.threads, planes, odd, st);
    }
    return cudaGetLastError();
}

cudaError_t launch_row_r2c(const SolveParams& p, const FftGeom& g, int planes, bool odd,
                           cudaStream_t st)
{
    return launch_fft_pass(0, p, g, planes, odd, st);
}

cudaError_t launch_col(const SolveParams& p, const FftGeom& g, int planes, cudaStream_t st)
{
    // forward + 1 / den + inverse of a column = a cyclic tridiagonal solve
    if (p.mode == 3 && p.tri != nullptr) {
        int dev = 0, nsm = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        return launch_col_tri(p, planes, nsm, st);
    }
    return launch_fft_pass(1, p, g, planes, false, st);
}

cudaError_t launch_row_c2r(const SolveParams& p, const FftGeom& g, int planes, bool odd,
                           cudaStream_t st)
{
    return launch_fft_pass(2, p, g, planes, odd, st);
}

cudaError_t launch_minmax(const float* x, size_t per_image, int batch, uint32_t* lohi, int nsm,
                          cudaStream_t st)
{
    k_reset_lohi<<<(batch + 127) / 128, 128, 0, st>>>(lohi, batch);
    size_t blocks = (per_image / 4 + 255) / 256;
    const size_t cap = (size_t)nsm * 4;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    dim3 grid((unsigned)blocks, batch);
    k_minmax<<<grid, 256, 0, st>>>(x, per_image, lohi);
    return cudaGetLastError();
}

cudaError_t launch_reset_lohi(uint32_t* lohi, int n, cudaStream_t st)
{
    k_reset_lohi<<<(n + 127) / 128, 128, 0, st>>>(lohi, n);
    return cudaGetLastError();
}

cudaError_t launch_count_nonfinite(const float* x, size_t n, unsigned* count, int nsm, cudaStream_t st)
{
    size_t blocks = (n + 255) / 256;
    if (blocks > (size_t)nsm * 8) blocks = (size_t)nsm * 8;
    if (blocks < 1) blocks = 1;
    k_count_nonfinite<<<(unsigned)blocks, 256, 0, st>>>(x, n, count);
    return cudaGetLastError();
}

cudaError_t launch_scale_by_range(float* x, size_t per_image, int batch, const uint32_t* lohi,
                                  int to_raw, cudaStream_t st)
{
    dim3 grid(256, batch);
    k_scale_by_range<<<grid, 256, 0, st>>>(x, per_image, lohi, to_raw);
    return cudaGetLastError();
}

cudaError_t launch_generate(int H, int W, int planes, const uint64_t* seeds, int K, double sigma,
                            double p_sp, float* out, cudaStream_t st)
{
    dim3 grid((unsigned)(((size_t)H * W + 255) / 256), planes);
    k_generate<<<grid, 256, sizeof(double) * 3 * K, st>>>(H, W, seeds, K, sigma, p_sp, out);
    return cudaGetLastError();
}



// ------------------------------------------------------ SFU peak probe --
// 8 independent ex2 chains per thread: throughput-bound MUFU.EX2 loop.  Block
// 0 thread 0 samples clock64/globaltimer to report the SM clock under load.
__global__ void k_mufu_probe(int iters, float* sink, unsigned long long* clk)
{
    float y[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) y[k] = 0.1f * (k + 1) + 1e-7f * threadIdx.x;
    unsigned long long c0 = 0, t0 = 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        c0 = clock64();
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y[k]) : "f"(-y[k]));
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += y[k];
    if (s == 12345.f) sink[threadIdx.x] = s;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        unsigned long long c1 = clock64(), t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        clk[0] = c1 - c0;
        clk[1] = t1 - t0;
    }
}

cudaError_t measure_mufu(int device, double* ex2_per_s, double* clock_hz)
{
    cudaDeviceProp prop{};
    cudaGetDeviceProperties(&prop, device);
    const int blocks = prop.multiProcessorCount * 8, threads = 256, iters = 4096;
    float* sink = nullptr;
    unsigned long long* clk = nullptr;
    cudaError_t e;
    if ((e = cudaMalloc(&sink, 1024 * sizeof(float))) != cudaSuccess) return e;
    if ((e = cudaMalloc(&clk, 2 * sizeof(unsigned long long))) != cudaSuccess) return e;
    // the rate is a property of the device: other work still in flight on the
    // library's non-blocking streams (or a clock ramp) can only lower a sample,
    // so the device is drained first and the fastest of five launches counts
    cudaDeviceSynchronize();
    cudaEvent_t ev[6];
    for (auto& x : ev) cudaEventCreate(&x);
    k_mufu_probe<<<blocks, threads>>>(iters, sink, clk);  // warm-up
    cudaEventRecord(ev[0]);
    for (int r = 0; r < 5; ++r) {
        k_mufu_probe<<<blocks, threads>>>(iters, sink, clk);
        cudaEventRecord(ev[r + 1]);
    }
    e = cudaEventSynchronize(ev[5]);
    float ms = 0.f;
    for (int r = 0; r < 5; ++r) {
        float t = 0.f;
        cudaEventElapsedTime(&t, ev[r], ev[r + 1]);
        if (t > 0.f && (ms == 0.f || t < ms)) ms = t;
    }
    unsigned long long hc[2] = {0, 0};
    cudaMemcpy(hc, clk, sizeof(hc), cudaMemcpyDeviceToHost);
    *ex2_per_s = ms > 0.f ? (double)blocks * threads * iters * 8 / (ms * 1e-3) : 0.0;
    *clock_hz = hc[1] ? (double)hc[0] / ((double)hc[1] * 1e-9) : 0.0;
    for (auto& x : ev) cudaEventDestroy(x);
    cudaFree(sink);
    cudaFree(clk);
    return e == cudaSuccess ? cudaGetLastError() : e;
}

}  // namespace blfls
