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

// One recursion step x' = m x + t in the state type ST.  float: the multiplier
// as a hi + lo pair (two FMAs); double (the low-frequency columns, below): one
// DFMA with m = hi + lo.
template <class ST>
struct TriMul;
template <>
struct TriMul<float> {
    float hi, lo;
    __device__ __forceinline__ TriMul(float h, float l) : hi(h), lo(l) {}
    __device__ __forceinline__ float step(float S, float t) const { return fmaf(lo, S, fmaf(hi, S, t)); }
    __device__ __forceinline__ float value() const { return hi; }
};
template <>
struct TriMul<double> {
    double m;
    __device__ __forceinline__ TriMul(float h, float l) : m((double)h + (double)l) {}
    __device__ __forceinline__ double step(double S, double t) const { return fma(m, S, t); }
    __device__ __forceinline__ double value() const { return m; }
};

// One warp per real column: entering state of every segment, in place over
// the aggregates.  rev: the segments were written in reversed order (q = 0
// is the last, possibly short, segment of the column).
template <class ST>
__device__ __forceinline__ void tri_scan(ST* arr, const SolveParams& p, int VF, int nseg, int K, bool rev)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = (blockDim.x + 31) >> 5;
    for (int col = warp; col < VF; col += nwarps) {
        const int v = min((int)(blockIdx.x * VF + col) >> 1, p.wc - 1);
        const float4 t = __ldg(&p.tri[2 * v + 1]);  // hi / lo of rho^RPT and rho^len_last
        const ST wrap = __ldg(&p.tri[2 * v]).z;     // 1 / (1 - rho^H)
        const TriMul<ST> mfull(t.x, t.y), mshort(t.z, t.w);
        ST* a = arr + col * 32 * K;
        const int qshort = rev ? 0 : nseg - 1;
        ST A = 1, B = 0;
        for (int k = 0; k < K; ++k) {
            const int q = lane * K + k;
            if (q < nseg) {
                const TriMul<ST>& m = q == qshort ? mshort : mfull;
                B = m.step(B, a[k * 32 + lane]);
                A *= m.value();
            }
        }
        ST Ai = A, Bi = B;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const ST Ap = __shfl_up_sync(0xffffffffu, Ai, d), Bp = __shfl_up_sync(0xffffffffu, Bi, d);
            if (lane >= d) {
                Bi = Ai * Bp + Bi;
                Ai *= Ap;
            }
        }
        const ST tot = __shfl_sync(0xffffffffu, Bi, 31);
        ST Ae = __shfl_up_sync(0xffffffffu, Ai, 1), Be = __shfl_up_sync(0xffffffffu, Bi, 1);
        if (lane == 0) {
            Ae = 1;
            Be = 0;
        }
        ST S = Ae * (tot * wrap) + Be;  // cyclic: the state entering segment 0 is total / (1 - rho^H)
        for (int k = 0; k < K; ++k) {
            const int q = lane * K + k;
            if (q < nseg) {
                const TriMul<ST>& m = q == qshort ? mshort : mfull;
                const ST Tk = a[k * 32 + lane];
                a[k * 32 + lane] = S;
                S = m.step(S, Tk);
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
    static __device__ __forceinline__ void aggregate(const float (&x)[RPT][TC], int nlive, const TriMul<ST>& rho,
                                                     ST (&S)[TC])
    {
#pragma unroll
        for (int k = 0; k < TC; ++k) S[k] = 0;
#pragma unroll
        for (int j = 0; j < RPT; ++j) {
            const int i = UP ? j : RPT - 1 - j;
            if (on(i, nlive))
#pragma unroll
                for (int k = 0; k < TC; ++k) S[k] = rho.step(S[k], x[i][k]);
        }
    }
    // causal factor from the entering state S: y[n] = x[n] + rho y[n-1], in place
    static __device__ __forceinline__ void causal(float (&x)[RPT][TC], int nlive, const TriMul<ST>& rho, ST (&S)[TC])
    {
#pragma unroll
        for (int i = 0; i < RPT; ++i)
            if (on(i, nlive))
#pragma unroll
                for (int k = 0; k < TC; ++k) {
                    S[k] = rho.step(S[k], x[i][k]);
                    x[i][k] = (float)S[k];
                }
    }
    // anticausal factor z[n] = y[n] + rho z[n+1], scaled and stored
    static __device__ __forceinline__ void anticausal_store(const float (&x)[RPT][TC], int nlive, const TriMul<ST>& rho,
                                                            float sc, ST (&S)[TC], float* base, size_t pitchf)
    {
#pragma unroll
        for (int i = RPT - 1; i >= 0; --i)
            if (on(i, nlive)) {
                float o[TC];
#pragma unroll
                for (int k = 0; k < TC; ++k) {
                    S[k] = rho.step(S[k], x[i][k]);
                    o[k] = (float)S[k] * sc;
                }
                TriVec<TC>::st(base + i * pitchf, o);
            }
    }
};

// both factors of one thread's strip in the state type ST; every thread of the
// CTA takes the same ST (the barriers are CTA-uniform)
template <int RPT, int TC, class ST>
__device__ __forceinline__ void tri_strip(const SolveParams& p, float* base, size_t pitchf, int nlive, float4 t0,
                                          ST* arr1, ST* arr2, int ct, int s, int nseg, int K, int VF)
{
    using F = TriStrip<RPT, TC, true, ST>;   // full segments: no per-row predicates
    using R = TriStrip<RPT, TC, false, ST>;  // the ragged last segment, dead threads
    const TriMul<ST> rho(t0.x, t0.y);
    const float sc = t0.w;
    const bool full = nlive == RPT;
    float x[RPT][TC];
    ST S[TC];
    if (full) F::load(base, pitchf, nlive, x); else R::load(base, pitchf, nlive, x);

    if (full) F::template aggregate<true>(x, nlive, rho, S); else R::template aggregate<true>(x, nlive, rho, S);
    if (s < nseg)
#pragma unroll
        for (int k = 0; k < TC; ++k) arr1[(ct * TC + k) * 32 * K + tri_pos(s, K)] = S[k];
    __syncthreads();
    tri_scan<ST>(arr1, p, VF, nseg, K, false);
    __syncthreads();
    if (s < nseg)
#pragma unroll
        for (int k = 0; k < TC; ++k) S[k] = arr1[(ct * TC + k) * 32 * K + tri_pos(s, K)];
    if (full) F::causal(x, nlive, rho, S); else R::causal(x, nlive, rho, S);

    if (full) F::template aggregate<false>(x, nlive, rho, S); else R::template aggregate<false>(x, nlive, rho, S);
    if (s < nseg)
#pragma unroll
        for (int k = 0; k < TC; ++k) arr2[(ct * TC + k) * 32 * K + tri_pos(nseg - 1 - s, K)] = S[k];
    __syncthreads();
    tri_scan<ST>(arr2, p, VF, nseg, K, true);
    __syncthreads();
    if (s < nseg)
#pragma unroll
        for (int k = 0; k < TC; ++k) S[k] = arr2[(ct * TC + k) * 32 * K + tri_pos(nseg - 1 - s, K)];
    if (full) F::anticausal_store(x, nlive, rho, sc, S, base, pitchf);
    else R::anticausal_store(x, nlive, rho, sc, S, base, pitchf);
}

// grid (ceil(2 wc / VF), planes), block = NCT * nseg rounded up to a warp
// register budget: the strip (RPT x TC values per thread) + ~24
template <int RPT, int TC, int MAXT>
constexpr int tri_minb()
{
    constexpr int regs = RPT * TC <= 8 ? 32 : RPT * TC <= 32 ? 64 : 128;
    return 65536 / (regs * MAXT) > 0 ? 65536 / (regs * MAXT) : 1;
}

// Strips whose pole is close to 1 (the lowest spectrum columns: the CTA's
// first column has rho > kTriDoublePole) keep the recursion state in double:
// on smooth data a float state rounds the same way at every step, a bias of
// eps / (1 - rho) of the value that the column FFT does not have (c4, rho =
// 0.978: full-pipeline max-abs 1.3e-5 -> the FFT's 3e-6).  A few percent of
// the CTAs; the strip values stay float.
constexpr float kTriDoublePole = 0.85f;

template <int RPT, int TC, int NCT, int MAXT>
__global__ void __launch_bounds__(MAXT, tri_minb<RPT, TC, MAXT>()) k_col_tri(const SolveParams p, int nseg, int K)
{
    constexpr int VF = TC * NCT;
    extern __shared__ __align__(8) double smt[];  // [2][VF][32 K] segment aggregates / entering states
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
    const bool dbl = __ldg(&p.tri[2 * min((int)(blockIdx.x * VF) >> 1, p.wc - 1)]).x > kTriDoublePole;
    if (dbl) {
        tri_strip<RPT, TC, double>(p, base, pitchf, nlive, t0, smt, smt + VF * 32 * K, ct, s, nseg, K, VF);
    } else {
        float* smf = reinterpret_cast<float*>(smt);
        tri_strip<RPT, TC, float>(p, base, pitchf, nlive, t0, smf, smf + VF * 32 * K, ct, s, nseg, K, VF);
    }
}

template <int RPT, int TC, int NCT>
cudaError_t launch_tri_t(const SolveParams& p, int planes, cudaStream_t st)
{
    constexpr int VF = TC * NCT;
    const int nseg = (p.H + RPT - 1) / RPT;
    const int K = (nseg + 31) / 32;
    const int threads = ((NCT * nseg + 31) / 32) * 32;
    if (threads > 1024) return cudaErrorInvalidConfiguration;
    const size_t smem = (size_t)2 * VF * 32 * K * sizeof(double);
    dim3 grid((2 * p.wc + VF - 1) / VF, planes);
    if (threads <= 256)
        k_col_tri<RPT, TC, NCT, 256><<<grid, threads, smem, st>>>(p, nseg, K);
    else if (threads <= 512)
        k_col_tri<RPT, TC, NCT, 512><<<grid, threads, smem, st>>>(p, nseg, K);
    else
        k_col_tri<RPT, TC, NCT, 1024><<<grid, threads, smem, st>>>(p, nseg, K);
    return cudaGetLastError();
}

}  // namespace

// rows per thread of the tridiagonal column pass: 32 (one strip = 4 thread
// columns x H / 32 segments; measured fastest on every BASELINE size,
// profiles/r02_tri_ab.txt); 16 for short columns so a strip still fills
// four warps
int tri_rows_per_thread(int H, int wc, int planes, int nsm)
{
    const int forced = knob("BLFLS_TRI_RPT", 0);
    if (forced == 8 || forced == 16 || forced == 32) return forced;
    (void)wc, (void)planes, (void)nsm;
    return H >= 1024 ? 32 : 16;
}

// Host tables in double, two float4 per column.  The pole rho and the segment
// multipliers are kept as hi + lo float pairs (x' = hi x + lo x in two FMAs):
// a pole rounded to one float moves the response of the low-frequency columns
// by 2 eps / (1 - rho) (c4: 5e-6 of the value).
//   tri[2v]     = (rho hi, rho lo, 1 / (1 - rho^H), rho / (lambda W))
//   tri[2v + 1] = (rho^RPT hi, lo, rho^len_last hi, lo)
// rho / (lambda W) = 2 / ((b + sqrt(c (c + 4 lambda))) W)
void tri_tables(int H, int W, int wc, double lambda, int rpt, std::vector<float4>& tri, std::vector<float>& scale)
{
    tri.resize(2 * (size_t)wc);
    scale.clear();
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

cudaError_t launch_col_tri(const SolveParams& p, int planes, cudaStream_t st)
{
    // thread shape: TC floats per thread x NCT thread columns (VF = TC NCT
    // floats = VF / 2 spectrum columns per CTA).  Default: one complex value
    // per thread and row (8-byte loads), 4 columns = one 32-byte sector per
    // row and CTA; at RPT = 32 that is 64 data registers, 2 CTAs of 256
    // threads per SM with 128 KB of loads in flight (c5: 1.47 ms per
    // iteration, 4.45 TB/s; the scalar 8-column shape 1.66 ms).
#ifdef BLFLS_EXPERIMENTS
    const int shape = knob("BLFLS_TRI_SHAPE", 1);
    const int nseg = (p.H + p.tri_rpt - 1) / p.tri_rpt;
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
    if (p.tri_rpt == 16) return launch_tri_t<16, 2, 4>(p, planes, st);
#endif
    return cudaErrorInvalidConfiguration;
}

}  // namespace blfls
