// k_col_tri.cu -- the column pass of the periodic least-squares solve
// (solver.cpp:107-120: X / (1 + lambda (|o_x|^2 + |o_y|^2)) between the
// forward and inverse 2-D transforms) WITHOUT a column FFT.
//
// After the row r2c the buffer holds X~(y, v): row-transformed, still spatial
// in y.  For one spectrum column v the division by
//   den(u, v) = c_v + lambda (2 - 2 cos(2 pi u / H)),  c_v = 1 + lambda 4 sin^2(pi v / W)
// over the column frequency u IS the cyclic tridiagonal system
//   -lambda z[y-1] + (c_v + 2 lambda) z[y] - lambda z[y+1] = x[y]      (y mod H)
// whose operator factors as (lambda / rho) (1 - rho S^-1)(1 - rho S) with
//   rho = 2 lambda / (b + sqrt(c_v (c_v + 4 lambda))),  b = c_v + 2 lambda,  0 <= rho < 1,
// so z = (rho / lambda) * anticausal(causal(x)), two first-order cyclic
// recursions y[n] = x[n] + rho y[n -/+ 1] with real rho (Re and Im are
// independent real columns).  The forward FFT, the 1 / den scaling and the
// inverse FFT of the column collapse into ~5 FP32 operations per value.
//
// One CTA holds a strip of VF adjacent floats (VF / 2 complex columns) x H
// rows entirely in REGISTERS: thread (s, ct) owns rows [s RPT, (s + 1) RPT)
// of TC floats.  All RPT loads of a thread are independent (issued before
// the first use), so the pass is a streaming read -> registers -> write with
// no shared-memory traffic except the segment carries:
//   1. local recursion from a zero state -> segment aggregate T_s
//   2. one warp per real column scans the (a_s, T_s) pairs (state' = T + a state,
//      a_s = rho^{len_s}; Kogge-Stone over lanes, K segments per lane); the
//      cyclic wrap-around state is total / (1 - rho^H)
//   3. the recursion is re-run from the true entering state (same rounding
//      as a sequential sweep of the whole column)
// and the same three steps bottom-up for the anticausal factor, which scales
// by rho / (lambda W) (the 1 / W of the unnormalised row transform pair) and
// stores in place.  rho, rho^RPT, rho^{len_last}, 1 / (1 - rho^H) and the
// scale come from double-precision host tables (tri_tables).
#include <algorithm>
#include <cmath>

#include "blfls_internal.cuh"

#ifndef BLFLS_TRI_REGS64
#define BLFLS_TRI_REGS64 128  // register budget of the 64-value strips (experiments: -DBLFLS_TRI_REGS64=80)
#endif

namespace blfls {

namespace {

template <int TC>
struct TriVec;
template <>
struct TriVec<1> {
    static __device__ __forceinline__ void ld(const float* q, float (&d)[1]) { d[0] = __ldcg(q); }
    static __device__ __forceinline__ void st(float* q, const float (&d)[1]) { *q = d[0]; }
};
template <>
struct TriVec<2> {
    static __device__ __forceinline__ void ld(const float* q, float (&d)[2])
    {
        const float2 v = __ldcg(reinterpret_cast<const float2*>(q));
        d[0] = v.x;
        d[1] = v.y;
    }
    static __device__ __forceinline__ void st(float* q, const float (&d)[2])
    {
        *reinterpret_cast<float2*>(q) = make_float2(d[0], d[1]);
    }
};

// segment q of a column is stored at (q % K) * 32 + q / K: the scanning lane
// q / K reads its K consecutive segments conflict-free
__device__ __forceinline__ int tri_pos(int q, int K) { return (q % K) * 32 + q / K; }

// One recursion step S' = m S + t.  TriPlain: the state is one float.  TriComp
// (the low-frequency strips, below): the state is an unevaluated float pair
// h + l and the multiplier a hi + lo pair.  The rounding error of
// y = fl(m.hi h + t) is recovered as fl(m.hi h - y) + t -- that FMA result has
// the magnitude of t, (1 - rho) of the state's, so its own rounding is a few
// percent of the error it measures -- and carried in l, so the recursion does
// not accumulate the systematic rounding of a float state.  5 FP32 operations
// per step instead of 1; an exact two-sum version (11) measured no better, a
// double state 8x slower per CTA.
struct TriPlain {
    float h;
    __device__ __forceinline__ void zero() { h = 0.f; }
    __device__ __forceinline__ void set(float v) { h = v; }
    __device__ __forceinline__ float value() const { return h; }
    __device__ __forceinline__ void step(float mh, float, float t) { h = fmaf(mh, h, t); }
};
struct TriComp {
    float h, l;
    __device__ __forceinline__ void zero() { h = l = 0.f; }
    __device__ __forceinline__ void set(float v)
    {
        h = v;
        l = 0.f;
    }
    __device__ __forceinline__ float value() const { return h + l; }
    __device__ __forceinline__ void step(float mh, float ml, float t)
    {
        const float y = fmaf(mh, h, t);
        const float r = fmaf(ml, h, __fadd_rn(fmaf(mh, h, -y), t));
        l = fmaf(mh, l, r);
        h = y;
    }
};

// One warp per real column: entering state of every segment, in place over
// the aggregates.  rev: the segments were written in reversed order (q = 0
// is the last, possibly short, segment of the column).
__device__ __forceinline__ void tri_scan(float* arr, const SolveParams& p, int VF, int nseg, int K, bool rev)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = (blockDim.x + 31) >> 5;
    for (int col = warp; col < VF; col += nwarps) {
        const int v = min((int)(blockIdx.x * VF + col) >> 1, p.wc - 1);
        const float4 t = __ldg(&p.tri[2 * v + 1]);  // hi / lo of rho^RPT and rho^len_last
        const float wrap = __ldg(&p.tri[2 * v]).z;  // 1 / (1 - rho^H)
        float* a = arr + col * 32 * K;
        const int qshort = rev ? 0 : nseg - 1;
        float A = 1.f, B = 0.f;
        for (int k = 0; k < K; ++k) {
            const int q = lane * K + k;
            if (q < nseg) {
                const float ak = q == qshort ? t.z : t.x, al = q == qshort ? t.w : t.y;
                B = fmaf(al, B, fmaf(ak, B, a[k * 32 + lane]));
                A *= ak;
            }
        }
        float Ai = A, Bi = B;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const float Ap = __shfl_up_sync(0xffffffffu, Ai, d), Bp = __shfl_up_sync(0xffffffffu, Bi, d);
            if (lane >= d) {
                Bi = fmaf(Ai, Bp, Bi);
                Ai *= Ap;
            }
        }
        const float tot = __shfl_sync(0xffffffffu, Bi, 31);
        float Ae = __shfl_up_sync(0xffffffffu, Ai, 1), Be = __shfl_up_sync(0xffffffffu, Bi, 1);
        if (lane == 0) {
            Ae = 1.f;
            Be = 0.f;
        }
        float S = fmaf(Ae, tot * wrap, Be);  // cyclic: the state entering segment 0 is total / (1 - rho^H)
        for (int k = 0; k < K; ++k) {
            const int q = lane * K + k;
            if (q < nseg) {
                const float ak = q == qshort ? t.z : t.x, al = q == qshort ? t.w : t.y;
                const float Tk = a[k * 32 + lane];
                a[k * 32 + lane] = S;
                S = fmaf(al, S, fmaf(ak, S, Tk));
            }
        }
    }
}

// The phases of one thread's strip (RPT rows x TC floats in registers).
// FULL: nlive == RPT, no per-row predicates; the kernel branches per phase so
// every thread reaches the barriers between the phases at the same place.
template <int RPT, int TC, bool FULL, class ST>
struct TriStrip {
    static __device__ __forceinline__ bool on(int i, int nlive) { return FULL || i < nlive; }
    static __device__ __forceinline__ void load(const float* base, size_t pitchf, int nlive, float (&x)[RPT][TC])
    {
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
            if (on(i, nlive)) {
                TriVec<TC>::ld(base + i * pitchf, x[i]);
            } else {
#pragma unroll
                for (int k = 0; k < TC; ++k) x[i][k] = 0.f;
            }
        }
    }
    // aggregate of the segment from a zero state; UP: rows in increasing order
    template <bool UP>
    static __device__ __forceinline__ void aggregate(const float (&x)[RPT][TC], int nlive, float rh, float rl,
                                                     ST (&S)[TC])
    {
#pragma unroll
        for (int k = 0; k < TC; ++k) S[k].zero();
#pragma unroll
        for (int j = 0; j < RPT; ++j) {
            const int i = UP ? j : RPT - 1 - j;
            if (on(i, nlive))
#pragma unroll
                for (int k = 0; k < TC; ++k) S[k].step(rh, rl, x[i][k]);
        }
    }
    // causal factor from the entering state S: y[n] = x[n] + rho y[n-1], in place
    static __device__ __forceinline__ void causal(float (&x)[RPT][TC], int nlive, float rh, float rl, ST (&S)[TC])
    {
#pragma unroll
        for (int i = 0; i < RPT; ++i)
            if (on(i, nlive))
#pragma unroll
                for (int k = 0; k < TC; ++k) {
                    S[k].step(rh, rl, x[i][k]);
                    x[i][k] = S[k].value();
                }
    }
    // anticausal factor z[n] = y[n] + rho z[n+1], scaled and stored
    static __device__ __forceinline__ void anticausal_store(const float (&x)[RPT][TC], int nlive, float rh, float rl,
                                                            float sc, ST (&S)[TC], float* base, size_t pitchf)
    {
#pragma unroll
        for (int i = RPT - 1; i >= 0; --i)
            if (on(i, nlive)) {
                float o[TC];
#pragma unroll
                for (int k = 0; k < TC; ++k) {
                    S[k].step(rh, rl, x[i][k]);
                    o[k] = S[k].value() * sc;
                }
                TriVec<TC>::st(base + i * pitchf, o);
            }
    }
};

// both factors of one thread's strip with the state type ST; every thread of
// the CTA takes the same ST (the barriers are CTA-uniform)
template <int RPT, int TC, class ST>
__device__ __forceinline__ void tri_strip(const SolveParams& p, float* base, size_t pitchf, int nlive, float4 t0,
                                          float* arr1, float* arr2, int ct, int s, int nseg, int K, int VF)
{
    using F = TriStrip<RPT, TC, true, ST>;   // full segments: no per-row predicates
    using R = TriStrip<RPT, TC, false, ST>;  // the ragged last segment, dead threads
    const float rh = t0.x, rl = t0.y, sc = t0.w;
    // one path per warp: a warp that holds the ragged segment (or dead
    // threads) runs the predicated phases for all its threads
    const bool full = __all_sync(0xffffffffu, nlive == RPT);
    float x[RPT][TC];
    ST S[TC];
    if (full) F::load(base, pitchf, nlive, x); else R::load(base, pitchf, nlive, x);

    if (full) F::template aggregate<true>(x, nlive, rh, rl, S); else R::template aggregate<true>(x, nlive, rh, rl, S);
    if (s < nseg)
#pragma unroll
        for (int k = 0; k < TC; ++k) arr1[(ct * TC + k) * 32 * K + tri_pos(s, K)] = S[k].value();
    __syncthreads();
    tri_scan(arr1, p, VF, nseg, K, false);
    __syncthreads();
#pragma unroll
    for (int k = 0; k < TC; ++k) S[k].set(s < nseg ? arr1[(ct * TC + k) * 32 * K + tri_pos(s, K)] : 0.f);
    if (full) F::causal(x, nlive, rh, rl, S); else R::causal(x, nlive, rh, rl, S);

    if (full) F::template aggregate<false>(x, nlive, rh, rl, S); else R::template aggregate<false>(x, nlive, rh, rl, S);
    if (s < nseg)
#pragma unroll
        for (int k = 0; k < TC; ++k) arr2[(ct * TC + k) * 32 * K + tri_pos(nseg - 1 - s, K)] = S[k].value();
    __syncthreads();
    tri_scan(arr2, p, VF, nseg, K, true);
    __syncthreads();
#pragma unroll
    for (int k = 0; k < TC; ++k) S[k].set(s < nseg ? arr2[(ct * TC + k) * 32 * K + tri_pos(nseg - 1 - s, K)] : 0.f);
    if (full) F::anticausal_store(x, nlive, rh, rl, sc, S, base, pitchf);
    else R::anticausal_store(x, nlive, rh, rl, sc, S, base, pitchf);
}

// grid (ceil(2 wc / VF), planes), block = NCT * nseg rounded up to a warp
// register budget: the strip (RPT x TC values per thread) + ~24
template <int RPT, int TC, int MAXT>
constexpr int tri_minb()
{
    constexpr int regs = RPT * TC <= 8 ? 32 : RPT * TC <= 32 ? 64 : (BLFLS_TRI_REGS64);
    return 65536 / (regs * MAXT) > 0 ? 65536 / (regs * MAXT) : 1;
}

// Strips whose pole is close to 1 (the lowest spectrum columns: the CTA's
// first column has rho > kTriCompPole) run the compensated recursion: a float
// state rounds with a bias of eps / (1 - rho) of the value that the column
// FFT does not have (c4, rho = 0.978: full-pipeline max-abs 1.3e-5 against
// the FFT's 3.2e-6; compensated: 2.5e-6).  A few percent of the CTAs.
constexpr float kTriCompPole = 0.85f;

template <int RPT, int TC, int NCT, int MAXT>
__global__ void __launch_bounds__(MAXT, tri_minb<RPT, TC, MAXT>())
    k_col_tri(const SolveParams p, int nseg, int K, float pole)
{
    constexpr int VF = TC * NCT;
    extern __shared__ float smt[];  // [2][VF][32 K] segment aggregates / entering states
    if (p.lohi_reset != nullptr && blockIdx.x == 0 && blockIdx.y == 0)
        for (int i = threadIdx.x; i < p.lohi_reset_n; i += blockDim.x) {
            p.lohi_reset[2 * i] = 0xffffffffu;  // ordered +inf / -inf (k_reset_lohi)
            p.lohi_reset[2 * i + 1] = 0u;
        }
    const int H = p.H;
    const int ct = threadIdx.x % NCT, s = threadIdx.x / NCT;
    const int fidx = blockIdx.x * VF + ct * TC;  // float index within the spectrum row
    const size_t pitchf = 2 * (size_t)p.spitch;
    const bool live = s < nseg && fidx < 2 * p.wc;
    const int y0 = s * RPT;
    const int nlive = live ? min(RPT, H - y0) : 0;
    float* base = reinterpret_cast<float*>(p.spec) + ((size_t)blockIdx.y * H + (live ? y0 : 0)) * pitchf +
                  (live ? fidx : 0);
    const int v = min(fidx >> 1, p.wc - 1);
    const float4 t0 = __ldg(&p.tri[2 * v]);  // rho hi, rho lo, 1 / (1 - rho^H), scale
    // rho falls with v: the CTA's first column decides for the whole CTA
    const bool comp = __ldg(&p.tri[2 * min((int)(blockIdx.x * VF) >> 1, p.wc - 1)]).x > pole;
    float* arr1 = smt;
    float* arr2 = smt + VF * 32 * K;
    if (comp)
        tri_strip<RPT, TC, TriComp>(p, base, pitchf, nlive, t0, arr1, arr2, ct, s, nseg, K, VF);
    else
        tri_strip<RPT, TC, TriPlain>(p, base, pitchf, nlive, t0, arr1, arr2, ct, s, nseg, K, VF);
}

template <int RPT, int TC, int NCT>
cudaError_t launch_tri_t(const SolveParams& p, int planes, cudaStream_t st)
{
    constexpr int VF = TC * NCT;
    const int nseg = (p.H + RPT - 1) / RPT;
    const int K = (nseg + 31) / 32;
    const int threads = ((NCT * nseg + 31) / 32) * 32;
    if (threads > 1024) return cudaErrorInvalidConfiguration;
    const size_t smem = (size_t)2 * VF * 32 * K * sizeof(float);
    dim3 grid((2 * p.wc + VF - 1) / VF, planes);
    const float pole = 0.01f * knob("BLFLS_TRI_COMP", (int)(100 * kTriCompPole));  // experiments: 200 = never
    if (threads <= 256)
        k_col_tri<RPT, TC, NCT, 256><<<grid, threads, smem, st>>>(p, nseg, K, pole);
    else if (threads <= 512)
        k_col_tri<RPT, TC, NCT, 512><<<grid, threads, smem, st>>>(p, nseg, K, pole);
    else
        k_col_tri<RPT, TC, NCT, 1024><<<grid, threads, smem, st>>>(p, nseg, K, pole);
    return cudaGetLastError();
}

}  // namespace

// rows per thread of the tridiagonal column pass: 32 (64 strip values per
// thread, 128 registers, 512 resident threads per SM) when the launch fills
// the GPU several times over (c4, c5: streaming from HBM, 128 KB of loads in
// flight per SM), else 16 (twice the threads at 64 registers: c1-c3 are one
// or two waves, latency-bound).  Measured with the bench's stage timers,
// cold L2 (profiles/r02_tri_ab.txt).
int tri_rows_per_thread(int H, int wc, int planes, int nsm)
{
    const int forced = knob("BLFLS_TRI_RPT", 0);
    if (forced == 8 || forced == 16 || forced == 32) return forced;
    const long strips = (long)planes * ((2 * wc + 7) / 8);
    const long threads32 = strips * 4 * ((H + 31) / 32);
    return threads32 >= 5L * 256 * nsm && H >= 1024 ? 32 : 16;
}

// Host tables in double, two float4 per column.  The pole rho and the segment
// multipliers are kept as hi + lo float pairs (x' = hi x + lo x in two FMAs):
// a pole rounded to one float moves the response of the low-frequency columns
// by 2 eps / (1 - rho) (c4: 5e-6 of the value).
//   tri[2v]     = (rho hi, rho lo, 1 / (1 - rho^H), rho / (lambda W))
//   tri[2v + 1] = (rho^RPT hi, lo, rho^len_last hi, lo)
// rho / (lambda W) = 2 / ((b + sqrt(c (c + 4 lambda))) W)
void tri_tables(int H, int W, int wc, double lambda, int rpt, std::vector<float4>& tri)
{
    tri.resize(2 * (size_t)wc);
    const int nseg = (H + rpt - 1) / rpt;
    const int len_last = H - (nseg - 1) * rpt;
    auto hi = [](double x) { return (float)x; };
    auto lo = [](double x) { return (float)(x - (double)(float)x); };
    for (int v = 0; v < wc; ++v) {
        const double sx = std::sin(M_PI * v / W);
        const double c = 1.0 + lambda * 4.0 * sx * sx;
        const double b = c + 2.0 * lambda;
        const double root = b + std::sqrt(c * (c + 4.0 * lambda));
        const double rho = 2.0 * lambda / root;
        const double m = std::pow(rho, rpt), ml = std::pow(rho, len_last);
        tri[2 * v] = make_float4(hi(rho), lo(rho), (float)(1.0 / (1.0 - std::pow(rho, H))), (float)(2.0 / (root * W)));
        tri[2 * v + 1] = make_float4(hi(m), lo(m), hi(ml), lo(ml));
    }
}

bool tri_supported(int H, int rpt) { return 4 * ((H + rpt - 1) / rpt) <= 1024 && H >= 2; }

cudaError_t launch_col_tri(const SolveParams& p, int planes, int nsm, cudaStream_t st)
{
    // thread shape: TC floats per thread x NCT thread columns (VF = TC NCT = 8
    // floats = one 32-byte sector per spectrum row and CTA).  Default: one
    // complex value per thread and row (8-byte loads, 4 thread columns); at
    // RPT = 32 that is 64 data registers, 2 CTAs of 256 threads per SM (c5:
    // 1.47 ms per iteration, 4.45 TB/s; the scalar 8-column shape 1.66 ms).
    // Launches far below one wave (c1) take the scalar shape: twice the
    // threads per strip (c1 column pass 17.7 -> 9.9 us per step).
    const int nseg = (p.H + p.tri_rpt - 1) / p.tri_rpt;
    const long threads = (long)planes * ((2 * p.wc + 7) / 8) * 4 * nseg;
    const bool scalar = threads < 256L * nsm && 8 * nseg <= 1024;
#ifdef BLFLS_EXPERIMENTS
    const int shape = knob("BLFLS_TRI_SHAPE", scalar ? 0 : 1);
#define BLFLS_TRI_GO(R)                                                                    \
    if (p.tri_rpt == R) {                                                                  \
        if (shape == 0 && 8 * nseg <= 1024) return launch_tri_t<R, 1, 8>(p, planes, st);   \
        if (shape == 2 && 8 * nseg <= 1024) return launch_tri_t<R, 2, 8>(p, planes, st);   \
        if (shape == 3 && 16 * nseg <= 1024) return launch_tri_t<R, 1, 16>(p, planes, st); \
        return launch_tri_t<R, 2, 4>(p, planes, st);                                       \
    }
    BLFLS_TRI_GO(32)
    BLFLS_TRI_GO(16)
    BLFLS_TRI_GO(8)
#undef BLFLS_TRI_GO
#else
    if (p.tri_rpt == 32) return launch_tri_t<32, 2, 4>(p, planes, st);
    if (p.tri_rpt == 16) return scalar ? launch_tri_t<16, 1, 8>(p, planes, st) : launch_tri_t<16, 2, 4>(p, planes, st);
#endif
    return cudaErrorInvalidConfiguration;
}

}  // namespace blfls
