// fft.cuh -- shared-memory Stockham mixed-radix FFT engine (device side).
//
// Replaces the reference's FFTW calls (src/fft2d.cpp:17-52).  A CTA holds V
// complex vectors of length n in ONE shared buffer; every stage reads each
// thread's butterfly inputs into registers, barriers, then writes the outputs
// back to the same buffer (no ping-pong, so a column strip of V vectors uses
// V*n*8 bytes).  Layouts:
//   ROWS: element j of vector v at buf[v*n + j]   (vectors along a row)
//   COLS: element j of vector v at buf[j*V + v]   (V adjacent spectrum columns,
//         so consecutive threads touch consecutive banks)
// Radices 2, 3, 4, 5 are specialised; any other prime up to 31 goes through a
// generic radix stage (used only by odd test sizes).
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

// values per thread held across a stage barrier
constexpr int kFftRegs = 16;

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
    }
}

template <bool COLS>
__device__ __forceinline__ int fft_addr(int v, int j, int n, int V)
{
    return COLS ? j * V + v : v * n + j;
}

template <int P, bool COLS>
__device__ __forceinline__ void fft_stage(float2* buf, int n, int V, int s,
                                          const float2* __restrict__ tw, bool inv)
{
    constexpr int NB = (kFftRegs + P - 1) / P;
    const int nbp = n / P;
    const int total = V * nbp;
    const int T = blockDim.x;
    const float sg = inv ? 1.0f : -1.0f;
    float2 a[NB][P];
#pragma unroll
    for (int i = 0; i < NB; ++i) {
        const int b = threadIdx.x + i * T;
        if (b < total) {
            const int v = COLS ? b % V : b / nbp;
            const int bb = COLS ? b / V : b % nbp;
#pragma unroll
            for (int r = 0; r < P; ++r) a[i][r] = buf[fft_addr<COLS>(v, bb + r * nbp, n, V)];
        }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < NB; ++i) {
        const int b = threadIdx.x + i * T;
        if (b < total) {
            const int v = COLS ? b % V : b / nbp;
            const int bb = COLS ? b / V : b % nbp;
            const int k = bb % s, q = bb / s;
            dft_small<P>(a[i], sg);
            const int obase = k + s * P * q;
            buf[fft_addr<COLS>(v, obase, n, V)] = a[i][0];
#pragma unroll
            for (int t = 1; t < P; ++t) {
                float2 w = __ldg(&tw[q * t * s]);
                if (inv) w.y = -w.y;
                buf[fft_addr<COLS>(v, obase + s * t, n, V)] = cmul(a[i][t], w);
            }
        }
    }
    __syncthreads();
}

// Generic odd prime radix (7..31), O(p^2) per butterfly, local-memory staging.
template <bool COLS>
__device__ void fft_stage_generic(float2* buf, int n, int V, int s, int P,
                                  const float2* __restrict__ tw, bool inv)
{
    const int nbp = n / P;
    const int total = V * nbp;
    const int T = blockDim.x;
    const int NB = (total + T - 1) / T;  // plan guarantees NB * P <= 32
    float2 a[32];
    for (int i = 0; i < NB; ++i) {
        const int b = threadIdx.x + i * T;
        if (b < total) {
            const int v = COLS ? b % V : b / nbp;
            const int bb = COLS ? b / V : b % nbp;
            for (int r = 0; r < P; ++r) a[i * P + r] = buf[fft_addr<COLS>(v, bb + r * nbp, n, V)];
        }
    }
    __syncthreads();
    const int wstep = n / P;
    for (int i = 0; i < NB; ++i) {
        const int b = threadIdx.x + i * T;
        if (b < total) {
            const int v = COLS ? b % V : b / nbp;
            const int bb = COLS ? b / V : b % nbp;
            const int k = bb % s, q = bb / s;
            for (int t = 0; t < P; ++t) {
                float2 acc = make_float2(0.f, 0.f);
                for (int r = 0; r < P; ++r) {
                    float2 w = __ldg(&tw[((r * t) % P) * wstep]);
                    if (inv) w.y = -w.y;
                    const float2 pr = cmul(a[i * P + r], w);
                    acc = cadd(acc, pr);
                }
                float2 w2 = __ldg(&tw[q * t * s]);
                if (inv) w2.y = -w2.y;
                buf[fft_addr<COLS>(v, k + s * (P * q + t), n, V)] = cmul(acc, w2);
            }
        }
    }
    __syncthreads();
}

// Full transform of V vectors in `buf` (unnormalised; inverse = conjugate twiddles).
template <bool COLS>
__device__ void fft_run(float2* buf, const FftDesc& d, int V, bool inv)
{
    int s = 1;
    for (int st = 0; st < d.nstages; ++st) {
        const int p = d.radix[st];
        switch (p) {
            case 2: fft_stage<2, COLS>(buf, d.n, V, s, d.tw, inv); break;
            case 3: fft_stage<3, COLS>(buf, d.n, V, s, d.tw, inv); break;
            case 4: fft_stage<4, COLS>(buf, d.n, V, s, d.tw, inv); break;
            case 5: fft_stage<5, COLS>(buf, d.n, V, s, d.tw, inv); break;
            default: fft_stage_generic<COLS>(buf, d.n, V, s, p, d.tw, inv); break;
        }
        s *= p;
    }
}

}  // namespace blfls
