// fft.cuh -- shared-memory Stockham mixed-radix FFT engine (device side).
//
// Replaces the reference's FFTW calls (src/fft2d.cpp:17-52).  A CTA holds V
// complex vectors of length n in ONE shared buffer; every stage reads each
// thread's butterfly inputs into registers, barriers, then writes the outputs
// back to the same buffer (no ping-pong, so a strip of V vectors costs V*n*8
// bytes).  Threads are split into V groups of TV = blockDim/V threads, one
// group per vector, so butterfly indices need no division by n.  Layouts:
//   ROWS: element j of vector v at buf[v*n + j]    thread -> v = tid / TV
//   COLS: element j of vector v at buf[j*V + v]    thread -> v = tid % V
//         (V adjacent spectrum columns: consecutive threads hit consecutive
//         banks and global loads are V*8-byte row segments)
// Stockham stage, radix p, stride s (product of earlier radices):
//   butterfly bb in [0, n/p): k = bb % s, q = bb / s, a_r = x[bb + r n/p]
//   y[k + s (p q + t)] = tw[q t s] * sum_r a_r w_p^{r t}
// tw[j] = exp(-2 pi i j / n) from double-precision host tables; the inverse
// conjugates every twiddle.  Radices 2, 3, 4, 5 are specialised; other primes
// up to 13 use the generic stage, compiled only into the GENERIC kernels that
// the plan selects for such (test-only) sizes.
#pragma once

#include "blfls_internal.cuh"

namespace blfls {

__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b)
{
    return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }
// multiply by +i (sg = +1) or -i (sg = -1)
__device__ __forceinline__ float2 cmuli(float2 a, float sg) { return make_float2(-sg * a.y, sg * a.x); }
__device__ __forceinline__ float2 cconj(float2 a) { return make_float2(a.x, -a.y); }

// Compile-time cos / sin of 2 pi m / P (Taylor series in double; the
// arguments are reduced to [0, pi]) for the odd-prime radices of the
// compile-time engine: they become FFMA immediates, not table loads.
constexpr double ct_pi = 3.14159265358979323846;
constexpr double ct_taylor_sin(double x)
{
    double term = x, sum = x;
    for (int k = 1; k < 30; ++k) {
        term *= -x * x / ((2.0 * k) * (2.0 * k + 1.0));
        sum += term;
    }
    return sum;
}
constexpr double ct_taylor_cos(double x)
{
    double term = 1.0, sum = 1.0;
    for (int k = 1; k < 30; ++k) {
        term *= -x * x / ((2.0 * k - 1.0) * (2.0 * k));
        sum += term;
    }
    return sum;
}
template <int P>
struct DftConst {
    float c[P], s[P];  // cos, sin of 2 pi m / P
    constexpr DftConst() : c(), s()
    {
        for (int m = 0; m < P; ++m) {
            c[m] = (float)ct_taylor_cos(2.0 * ct_pi * m / P);
            s[m] = (float)ct_taylor_sin(2.0 * ct_pi * m / P);
        }
    }
};

// Direct DFT of odd prime length P (7, 11, 13, 17) with the conjugate-pair
// symmetry: s_r = a_r + a_{P-r}, d_r = a_r - a_{P-r} (r = 1..h, h = (P-1)/2);
// A_t = a_0 + sum_r s_r cos(2 pi rt/P), B_t = sum_r d_r sin(2 pi rt/P);
// y_t = A_t + i sg B_t, y_{P-t} = A_t - i sg B_t: 4 h^2 real FMAs per P outputs.
template <int P>
__device__ __forceinline__ void dft_prime(float2 (&a)[P], float sg)
{
    constexpr int h = (P - 1) / 2;
    constexpr DftConst<P> K{};
    float2 sr[h + 1], dr[h + 1];
    float2 y0 = a[0];
#pragma unroll
    for (int r = 1; r <= h; ++r) {
        sr[r] = cadd(a[r], a[P - r]);
        dr[r] = csub(a[r], a[P - r]);
        y0 = cadd(y0, sr[r]);
    }
    float2 out[P];
    out[0] = y0;
#pragma unroll
    for (int t = 1; t <= h; ++t) {
        float2 A = a[0], B = make_float2(0.f, 0.f);
#pragma unroll
        for (int r = 1; r <= h; ++r) {
            const int m = (r * t) % P;
            const float c = K.c[m], sn = K.s[m];  // cos / sin of 2 pi m / P (sin odd in m)
            A = make_float2(fmaf(sr[r].x, c, A.x), fmaf(sr[r].y, c, A.y));
            B = make_float2(fmaf(dr[r].x, sn, B.x), fmaf(dr[r].y, sn, B.y));
        }
        const float2 jb = cmuli(B, sg);
        out[t] = cadd(A, jb);
        out[P - t] = csub(A, jb);
    }
#pragma unroll
    for (int t = 0; t < P; ++t) a[t] = out[t];
}

template <int P>
__device__ __forceinline__ void dft_small(float2 (&a)[P], float sg /* -1 fwd, +1 inv */)
{
    if constexpr (P == 2) {
        const float2 t = a[1];
        a[1] = csub(a[0], t);
        a[0] = cadd(a[0], t);
    } else if constexpr (P == 3) {
        const float c = -0.5f, d = sg * 0.86602540378443864676f;
        const float2 t1 = cadd(a[1], a[2]);
        const float2 t2 = csub(a[1], a[2]);
        const float2 m = make_float2(fmaf(c, t1.x, a[0].x), fmaf(c, t1.y, a[0].y));
        const float2 jt = cmuli(cscale(t2, d), 1.0f);
        a[0] = cadd(a[0], t1);
        a[1] = cadd(m, jt);
        a[2] = csub(m, jt);
    } else if constexpr (P == 4) {
        const float2 s02 = cadd(a[0], a[2]), d02 = csub(a[0], a[2]);
        const float2 s13 = cadd(a[1], a[3]), d13 = csub(a[1], a[3]);
        const float2 jd = cmuli(d13, sg);  // sg*i*(a1-a3)
        a[0] = cadd(s02, s13);
        a[2] = csub(s02, s13);
        a[1] = cadd(d02, jd);
        a[3] = csub(d02, jd);
    } else if constexpr (P == 8) {
        // radix-2 DIF step (twiddles w8^k) then two radix-4 DFTs
        constexpr float r = 0.70710678118654752440f;
        float2 b[4], c[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            b[k] = cadd(a[k], a[k + 4]);
            c[k] = csub(a[k], a[k + 4]);
        }
        c[1] = make_float2(r * (c[1].x - sg * c[1].y), r * (c[1].y + sg * c[1].x));    // * (r, sg r)
        c[2] = cmuli(c[2], sg);                                                         // * (0, sg)
        c[3] = make_float2(r * (-c[3].x - sg * c[3].y), r * (-c[3].y + sg * c[3].x));  // * (-r, sg r)
        dft_small<4>(b, sg);
        dft_small<4>(c, sg);
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            a[2 * m] = b[m];
            a[2 * m + 1] = c[m];
        }
    } else if constexpr (P == 5) {
        const float c1 = 0.30901699437494742410f, c2 = -0.80901699437494742410f;
        const float s1 = 0.95105651629515357212f * sg, s2 = 0.58778525229247312917f * sg;
        const float2 t1 = cadd(a[1], a[4]), t2 = cadd(a[2], a[3]);
        const float2 t3 = csub(a[1], a[4]), t4 = csub(a[2], a[3]);
        const float2 m1 = make_float2(a[0].x + c1 * t1.x + c2 * t2.x, a[0].y + c1 * t1.y + c2 * t2.y);
        const float2 m2 = make_float2(a[0].x + c2 * t1.x + c1 * t2.x, a[0].y + c2 * t1.y + c1 * t2.y);
        const float2 j1 = cmuli(make_float2(s1 * t3.x + s2 * t4.x, s1 * t3.y + s2 * t4.y), 1.0f);
        const float2 j2 = cmuli(make_float2(s2 * t3.x - s1 * t4.x, s2 * t3.y - s1 * t4.y), 1.0f);
        a[0] = cadd(a[0], cadd(t1, t2));
        a[1] = cadd(m1, j1);
        a[4] = csub(m1, j1);
        a[2] = cadd(m2, j2);
        a[3] = csub(m2, j2);
    } else {
        dft_prime<P>(a, sg);
    }
}

// per-thread view of a CTA holding V vectors
struct FftLane {
    int v;    // vector owned by this thread
    int t;    // index within the vector's thread group
    int TV;   // threads per vector
};

template <bool COLS>
__device__ __forceinline__ FftLane fft_lane(int V, int log2V)
{
    FftLane l;
    l.TV = blockDim.x >> log2V;
    if (COLS) {
        l.v = threadIdx.x & (V - 1);
        l.t = threadIdx.x >> log2V;
    } else {
        l.v = threadIdx.x / l.TV;
        l.t = threadIdx.x - l.v * l.TV;
    }
    return l;
}

template <bool COLS>
__device__ __forceinline__ int fft_addr(const FftLane& l, int j, int n, int V)
{
    return COLS ? j * V + l.v : l.v * n + j;
}

// E = complex values a thread holds across the stage barrier
template <int P, int E, bool COLS>
__device__ __forceinline__ void fft_stage(float2* buf, const FftLane& l, int n, int V, int s,
                                          const float2* __restrict__ tw, bool inv)
{
    constexpr int NB = (E + P - 1) / P;
    const int nbp = n / P;
    const float sg = inv ? 1.0f : -1.0f;
    float2 a[NB][P];
#pragma unroll
    for (int i = 0; i < NB; ++i) {
        const int bb = l.t + i * l.TV;
        if (bb < nbp) {
#pragma unroll
            for (int r = 0; r < P; ++r) a[i][r] = buf[fft_addr<COLS>(l, bb + r * nbp, n, V)];
        }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < NB; ++i) {
        const int bb = l.t + i * l.TV;
        if (bb < nbp) {
            const int q = bb / s, k = bb - q * s;
            dft_small<P>(a[i], sg);
            const int obase = k + s * P * q;
            buf[fft_addr<COLS>(l, obase, n, V)] = a[i][0];
#pragma unroll
            for (int t = 1; t < P; ++t) {
                float2 w = __ldg(&tw[q * t * s]);
                if (inv) w.y = -w.y;
                buf[fft_addr<COLS>(l, obase + s * t, n, V)] = cmul(a[i][t], w);
            }
        }
    }
    __syncthreads();
}

// Generic odd prime radix (7, 11, 13), O(p^2) per butterfly; test sizes only.
template <int E, bool COLS>
__device__ void fft_stage_generic(float2* buf, const FftLane& l, int n, int V, int s, int P,
                                  const float2* __restrict__ tw, bool inv)
{
    const int nbp = n / P;
    const int NB = (nbp + l.TV - 1) / l.TV;  // plan guarantees NB * P <= 2E
    float2 a[2 * E];
    for (int i = 0; i < NB; ++i) {
        const int bb = l.t + i * l.TV;
        if (bb < nbp)
            for (int r = 0; r < P; ++r) a[i * P + r] = buf[fft_addr<COLS>(l, bb + r * nbp, n, V)];
    }
    __syncthreads();
    for (int i = 0; i < NB; ++i) {
        const int bb = l.t + i * l.TV;
        if (bb < nbp) {
            const int q = bb / s, k = bb - q * s;
            for (int t = 0; t < P; ++t) {
                float2 acc = make_float2(0.f, 0.f);
                for (int r = 0; r < P; ++r) {
                    float2 w = __ldg(&tw[((r * t) % P) * nbp]);
                    if (inv) w.y = -w.y;
                    acc = cadd(acc, cmul(a[i * P + r], w));
                }
                float2 w2 = __ldg(&tw[q * t * s]);
                if (inv) w2.y = -w2.y;
                buf[fft_addr<COLS>(l, k + s * (P * q + t), n, V)] = cmul(acc, w2);
            }
        }
    }
    __syncthreads();
}

// Direct DFT stage for primes above 13 (reflect-padded sizes such as
// 1952 = 2^5 * 61 or 1112 = 2^3 * 139): a batched P x P matrix product
// y[t][g] = sum_r w^{(r t) mod P} a[r][g] over the V * n / P butterfly
// groups g of the CTA.  Register tiling: a work item is kDirG groups x kDirT
// outputs t; per r it loads kDirG inputs and kDirT roots (a shared table of
// the P roots, indices advanced incrementally) for kDirG * kDirT complex
// MACs.  The outer twiddle and the Stockham placement are applied on the way
// to `scratch`; the stage is then copied back.  The root table sits after
// the scratch buffer (RtFft::smem_bytes).
constexpr int kDirT = 4;  // outputs t per item
constexpr int kDirG = 4;  // groups per item
template <bool COLS>
__device__ void fft_stage_direct(float2* buf, float2* scratch, const FftLane& l, int n, int V, int s,
                                 int P, const float2* __restrict__ tw, bool inv)
{
    const int nbp = n / P;
    float2* roots = scratch + (size_t)V * n;  // [P]
    for (int m = threadIdx.x; m < P; m += blockDim.x) {
        float2 w = __ldg(&tw[m * nbp]);  // w_P^m
        if (inv) w.y = -w.y;
        roots[m] = w;
    }
    __syncthreads();
    const int groups = V * nbp;  // g -> (vector g / nbp, butterfly g % nbp)
    const int ngb = (groups + kDirG - 1) / kDirG, ntb = (P + kDirT - 1) / kDirT;
    for (int item = threadIdx.x; item < ngb * ntb; item += blockDim.x) {
        const int gb = item % ngb, tb = item / ngb;
        const int t0 = tb * kDirT;
        int addr_in[kDirG];
#pragma unroll
        for (int j = 0; j < kDirG; ++j) {
            const int g = min(gb * kDirG + j, groups - 1);
            const int v = g / nbp, bb = g - v * nbp;
            addr_in[j] = COLS ? bb * V + v : v * n + bb;
        }
        const int rstep = COLS ? nbp * V : nbp;  // address step of r
        float2 acc[kDirG][kDirT];
#pragma unroll
        for (int j = 0; j < kDirG; ++j)
#pragma unroll
            for (int i = 0; i < kDirT; ++i) acc[j][i] = make_float2(0.f, 0.f);
        int e[kDirT];  // (r * t) mod P
#pragma unroll
        for (int i = 0; i < kDirT; ++i) e[i] = 0;
        for (int r = 0; r < P; ++r) {
            float2 a[kDirG], w[kDirT];
#pragma unroll
            for (int j = 0; j < kDirG; ++j) a[j] = buf[addr_in[j] + r * rstep];
#pragma unroll
            for (int i = 0; i < kDirT; ++i) {
                w[i] = roots[e[i]];
                e[i] += min(t0 + i, P - 1);
                if (e[i] >= P) e[i] -= P;
            }
#pragma unroll
            for (int j = 0; j < kDirG; ++j)
#pragma unroll
                for (int i = 0; i < kDirT; ++i) {
                    acc[j][i].x = fmaf(a[j].x, w[i].x, fmaf(-a[j].y, w[i].y, acc[j][i].x));
                    acc[j][i].y = fmaf(a[j].x, w[i].y, fmaf(a[j].y, w[i].x, acc[j][i].y));
                }
        }
#pragma unroll
        for (int j = 0; j < kDirG; ++j) {
            const int g = gb * kDirG + j;
            if (g >= groups) break;
            const int v = g / nbp, bb = g - v * nbp;
            const int q = bb / s, k = bb - q * s;
#pragma unroll
            for (int i = 0; i < kDirT; ++i) {
                const int t = t0 + i;
                if (t < P) {
                    float2 w2 = __ldg(&tw[q * t * s]);
                    if (inv) w2.y = -w2.y;
                    const int o = k + s * (P * q + t);
                    scratch[COLS ? o * V + v : v * n + o] = cmul(acc[j][i], w2);
                }
            }
        }
    }
    __syncthreads();
    for (int o = l.t; o < n; o += l.TV) buf[fft_addr<COLS>(l, o, n, V)] = scratch[fft_addr<COLS>(l, o, n, V)];
    __syncthreads();
}

// Full transform of the CTA's V vectors (unnormalised; inverse = conjugate twiddles).
template <int E, bool COLS, bool GENERIC>
__device__ void fft_run(float2* buf, const FftDesc& d, int V, int log2V, bool inv)
{
    const FftLane l = fft_lane<COLS>(V, log2V);
    int s = 1;
    for (int st = 0; st < d.nstages; ++st) {
        const int p = d.radix[st];
        if (GENERIC && p > 13)
            fft_stage_direct<COLS>(buf, buf + (size_t)V * d.n, l, d.n, V, s, p, d.tw, inv);
        else if (p == 4)
            fft_stage<4, E, COLS>(buf, l, d.n, V, s, d.tw, inv);
        else if (p == 2)
            fft_stage<2, E, COLS>(buf, l, d.n, V, s, d.tw, inv);
        else if (p == 3)
            fft_stage<3, E, COLS>(buf, l, d.n, V, s, d.tw, inv);
        else if (p == 5)
            fft_stage<5, E, COLS>(buf, l, d.n, V, s, d.tw, inv);
        else if constexpr (GENERIC)
            fft_stage_generic<E, COLS>(buf, l, d.n, V, s, p, d.tw, inv);
        s *= p;
    }
}

// Bluestein: X_k = c_k sum_j (x_j c_j) h_{k-j}, c_m = exp(sg pi i m^2 / n),
// h = conj(c) -- a cyclic convolution of length M computed with two M-point
// transforms of the runtime engine in `work` (V * M complex after the strip).
template <int E, bool COLS>
__device__ void fft_bluestein(float2* buf, float2* work, const FftDesc& d, const BlueDesc& b, int V,
                              int log2V, bool inv)
{
    const FftLane l = fft_lane<COLS>(V, log2V);
    const int n = d.n, M = b.m.n;
    for (int j = l.t; j < M; j += l.TV) {
        float2 a = make_float2(0.f, 0.f);
        if (j < n) {
            float2 c = __ldg(&b.chirp[j]);
            if (inv) c.y = -c.y;
            a = cmul(buf[fft_addr<COLS>(l, j, n, V)], c);
        }
        work[fft_addr<COLS>(l, j, M, V)] = a;
    }
    __syncthreads();
    fft_run<E, COLS, false>(work, b.m, V, log2V, false);
    const float2* H = inv ? b.hi : b.hf;
    for (int j = l.t; j < M; j += l.TV) {
        const int o = fft_addr<COLS>(l, j, M, V);
        work[o] = cmul(work[o], __ldg(&H[j]));
    }
    __syncthreads();
    fft_run<E, COLS, false>(work, b.m, V, log2V, true);
    for (int k = l.t; k < n; k += l.TV) {
        float2 c = __ldg(&b.chirp[k]);
        if (inv) c.y = -c.y;
        buf[fft_addr<COLS>(l, k, n, V)] = cmul(work[fft_addr<COLS>(l, k, M, V)], c);
    }
    __syncthreads();
}

}  // namespace blfls

// ===================================================================
// Compile-time engine: length N, V vectors per CTA, TV threads per vector.
// Every index (stage stride, butterfly count, predicate) folds to a
// constant.  Instantiated for the BASELINE sizes (capi.cu / k_solve.cu).
namespace blfls {

constexpr int ct_count(int n, int p) { return n % p == 0 ? 1 + ct_count(n / p, p) : 0; }
// power-of-two part as radix 8s, then one 4 or 2; then 3s, 5s, and the odd
// primes 7, 11, 13, 17 (reflect-padded sizes, e.g. 1056 = 2^5 3 11)
constexpr int ct_n8(int n) { return ct_count(n, 2) / 3; }
constexpr int ct_rest(int n) { return ct_count(n, 2) % 3; }  // 0, 1 (radix 2) or 2 (radix 4)
constexpr int ct_nstages(int n)
{
    return ct_n8(n) + (ct_rest(n) ? 1 : 0) + ct_count(n, 3) + ct_count(n, 5) + ct_count(n, 7) +
           ct_count(n, 11) + ct_count(n, 13) + ct_count(n, 17);
}
constexpr int ct_radix(int n, int i)
{
    if (i < ct_n8(n)) return 8;
    i -= ct_n8(n);
    if (ct_rest(n)) {
        if (i == 0) return ct_rest(n) == 2 ? 4 : 2;
        i -= 1;
    }
    for (int p : {3, 5, 7, 11, 13, 17}) {
        if (i < ct_count(n, p)) return p;
        i -= ct_count(n, p);
    }
    return 1;
}
constexpr int ct_stride(int n, int i)
{
    int s = 1;
    for (int k = 0; k < i; ++k) s *= ct_radix(n, k);
    return s;
}
constexpr bool ct_supported(int n)
{
    int m = n;
    for (int p : {2, 3, 5, 7, 11, 13, 17})
        while (m % p == 0) m /= p;
    return m == 1;
}

// Shared-memory padding of the compile-time engine: the first Stockham
// stages write with a stride of 8 complex (rows) or 8 rows of V complex
// (columns), which would map 16 lanes onto 1-2 bank pairs.  One pad element
// per 8 (rows) / V pad elements per 8*V (columns) spreads them over all banks.
template <int V>
constexpr int ct_log2(int v) { return v <= 1 ? 0 : 1 + ct_log2<V>(v / 2); }
// Rows of a power-of-two length take one pad slot per 16 complex instead:
// with 8-byte elements a half-warp's 16 consecutive reads (every stage's
// inputs and the row epilogues) then stay inside one 128-byte bank line --
// per 8 they straddle a pad slot and conflict 2-way -- while the stride-8
// first-stage writes still spread over all banks (c5 row r2c 9.25 -> 8.75
// ms per step, c4 178 -> 168 us; c3's 960-point rows measured slower, so
// mixed-radix lengths keep the per-8 pad).
template <int N>
constexpr int ct_row_pad_block() { return (N & (N - 1)) == 0 ? 16 : 8; }
template <int V, bool COLS, int PB = 8>
__device__ __forceinline__ int ct_pad(int flat)
{
    if (COLS) {
        constexpr int L = ct_log2<V>(V);
        return flat + ((flat >> (3 + L)) << L);
    }
    return flat + flat / PB;
}

template <int N, int V, int TV, bool COLS, bool INV, int P, int S>
__device__ __forceinline__ void ct_stage(float2* buf, int v, int t, const float2* __restrict__ tw)
{
    constexpr int NBP = N / P;
    constexpr int NB = (NBP + TV - 1) / TV;
    constexpr bool PRED = NB * TV != NBP;
    constexpr float sg = INV ? 1.0f : -1.0f;
    constexpr int PB = COLS ? 8 : ct_row_pad_block<N>();  // elements per pad slot
    auto addr = [&](int j) { return ct_pad<V, COLS, PB>(COLS ? j * V + v : v * N + j); };
    // ct_pad adds one pad slot per 8 (rows) / per 8 V (columns) elements, so
    // indices j + m D with D a multiple of 8 map to addr(j) + m D (9/8) (x V
    // for columns): the butterfly's P inputs (D = NBP) and, when the stage
    // stride S is a multiple of 8 (or S = 1 with P | 8, outputs inside one
    // 8-block), its P outputs are a base address plus compile-time offsets.
    constexpr bool LIN_IN = NBP % PB == 0;
    constexpr bool LIN_OUT = S % PB == 0 || (S == 1 && PB % P == 0);
    constexpr int VS = COLS ? V : 1;
    constexpr int STR_IN = LIN_IN ? NBP / PB * (PB + 1) * VS : 0;
    constexpr int STR_OUT = S == 1 ? VS : (LIN_OUT ? S / PB * (PB + 1) * VS : 0);
    float2 a[NB][P];
#pragma unroll
    for (int i = 0; i < NB; ++i) {
        const int bb = t + i * TV;
        if (!PRED || bb < NBP) {
            if constexpr (LIN_IN) {
                const float2* src = buf + addr(bb);
#pragma unroll
                for (int r = 0; r < P; ++r) a[i][r] = src[r * STR_IN];
            } else {
#pragma unroll
                for (int r = 0; r < P; ++r) a[i][r] = buf[addr(bb + r * NBP)];
            }
        }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < NB; ++i) {
        const int bb = t + i * TV;
        if (!PRED || bb < NBP) {
            const int q = bb / S, k = bb - q * S;
            dft_small<P>(a[i], sg);
            const int obase = k + S * P * q;
            float2* dst = buf + addr(obase);
            auto out_at = [&](int tt) -> float2& {
                if constexpr (LIN_OUT)
                    return dst[tt * STR_OUT];
                else
                    return buf[addr(obase + S * tt)];
            };
            out_at(0) = a[i][0];
            // twiddles w^t, w = tw[q S]: one coalesced load, powers by complex
            // multiplication (relative error <= (P-1) ulp-level products)
            float2 w1 = __ldg(&tw[q * S]);
            if (INV) w1.y = -w1.y;
            float2 wt = w1;
#pragma unroll
            for (int tt = 1; tt < P; ++tt) {
                out_at(tt) = cmul(a[i][tt], wt);
                if (tt + 1 < P) wt = cmul(wt, w1);  // w^(t+1)
            }
        }
    }
    __syncthreads();
}

template <int N, int V, int TV, bool COLS, bool INV, int I>
__device__ __forceinline__ void ct_stages(float2* buf, int v, int t, const float2* __restrict__ tw)
{
    if constexpr (I < ct_nstages(N)) {
        ct_stage<N, V, TV, COLS, INV, ct_radix(N, I), ct_stride(N, I)>(buf, v, t, tw);
        ct_stages<N, V, TV, COLS, INV, I + 1>(buf, v, t, tw);
    }
}

// engine policies used by the solve kernels
template <int N_, int V_, int TV_>
struct CtFft {
    static constexpr int N = N_, V = V_, TV = TV_, THREADS = V_ * TV_;
    static constexpr bool kCompileTime = true;
    // row r2c launch bounds: the fold phase is load-latency bound, so the
    // CT row pass runs at 2048 resident threads per SM (32 registers)
    static constexpr int kMaxThreads = THREADS, kRowMinBlocks = 2048 / THREADS;
    const float2* tw;
    __device__ __forceinline__ int n() const { return N; }
    __device__ __forceinline__ int vecs() const { return V; }
    template <bool COLS>
    __device__ __forceinline__ int pad(int flat) const { return ct_pad<V, COLS, COLS ? 8 : ct_row_pad_block<N_>()>(flat); }
    __device__ __forceinline__ int threads() const { return THREADS; }  // compile-time
    __host__ __device__ static constexpr size_t smem_bytes(bool cols)
    {
        const int last = V * N - 1;
        const int L = ct_log2<V>(V);
        const int padded = cols ? last + ((last >> (3 + L)) << L) : last + last / ct_row_pad_block<N_>();
        return (size_t)(padded + 1) * sizeof(float2);
    }
    template <bool COLS>
    __device__ __forceinline__ void run(float2* buf, bool inv) const
    {
        const int v = COLS ? (int)threadIdx.x % V : (int)threadIdx.x / TV;
        const int t = COLS ? (int)threadIdx.x / V : (int)threadIdx.x % TV;
        if (inv)
            ct_stages<N, V, TV, COLS, true, 0>(buf, v, t, tw);
        else
            ct_stages<N, V, TV, COLS, false, 0>(buf, v, t, tw);
    }
};

template <int E, bool GENERIC>
struct RtFft {
    static constexpr bool kCompileTime = false;
    static constexpr int kMaxThreads = 1024, kRowMinBlocks = 1;
    FftDesc d;
    int V, log2V;
    __device__ __forceinline__ int n() const { return d.n; }
    __device__ __forceinline__ int vecs() const { return V; }
    bool direct;  // a prime factor above 13: the direct stage needs a scratch buffer
    int pmax;     // largest prime factor (the direct stage's root table)
    bool bluestein;
    BlueDesc blue;
    template <bool COLS>
    __device__ __forceinline__ int pad(int flat) const { return flat; }
    __device__ __forceinline__ int threads() const { return blockDim.x; }
    size_t smem_bytes(bool) const
    {
        // Bluestein: the strip plus the length-M work vectors; direct stages:
        // a scratch copy of the strip plus the root table
        if (bluestein) return (size_t)V * (d.n + blue.m.n) * sizeof(float2);
        return (size_t)V * d.n * sizeof(float2) * (direct ? 2 : 1) +
               (direct ? (size_t)pmax * sizeof(float2) : 0);
    }
    template <bool COLS>
    __device__ __forceinline__ void run(float2* buf, bool inv) const
    {
        if (bluestein)
            fft_bluestein<E, COLS>(buf, buf + (size_t)V * d.n, d, blue, V, log2V, inv);
        else
            fft_run<E, COLS, GENERIC>(buf, d, V, log2V, inv);
    }
};

}  // namespace blfls
