// fft2.cuh -- high-radix Stockham engine (device side) for the solve kernels.
//
// Same transform as fft.cuh (FFTW's convention, src/fft2d.cpp:17-52), built
// to move fewer bytes through shared memory: every stage is a radix-P DFT of
// up to 32 points held in registers (composite P as an in-register
// Cooley-Tukey with compile-time roots), so a 1024-point vector takes two
// stages instead of four (8 8 8 2).  The first stage can read its inputs
// straight from global memory and the last stage can write its outputs
// straight to global memory (both coalesced: consecutive butterflies touch
// consecutive elements), so a row pass touches shared memory only for the
// exchanges between stages.
//
// Stage i (radix P, stride S = product of the earlier radices), butterfly
// bb in [0, N/P): k = bb % S, q = bb / S, inputs a_r = x[bb + r N/P],
// outputs y[k + S (P q + t)] = w^{t} DFT_P(a)_t with w = tw[q S] (conjugated
// for the inverse).  The radices are packed first-fit-decreasing from the
// prime factors of N under PMAX (1024 -> 32 32, 960 -> 30 32,
// 1080 -> 30 18 2, 2048 -> 32 32 2).
#pragma once

#include "fft.cuh"

namespace blfls {

struct Plan2 {
    int n;       // stages
    int r[12];   // radices
};

constexpr Plan2 c2_plan(int N, int PMAX)
{
    int f[32] = {};
    int nf = 0, m = N;
    for (int p = 2; p <= m && nf < 32; ++p)
        while (m % p == 0) {
            f[nf++] = p;
            m /= p;
        }
    Plan2 s{};
    for (int i = nf - 1; i >= 0; --i) {  // largest prime first
        int j = 0;
        while (j < s.n && s.r[j] * f[i] > PMAX) ++j;
        if (j == s.n) s.r[s.n++] = 1;
        s.r[j] *= f[i];
    }
    return s;
}

// the same radices in reverse order (the inverse column transform of the
// fused forward / inverse pass, s2_fwd_last_inv_first)
constexpr Plan2 c2_reverse(Plan2 p)
{
    Plan2 r{};
    r.n = p.n;
    for (int i = 0; i < p.n; ++i) r.r[i] = p.r[p.n - 1 - i];
    return r;
}

// first factor of an in-register composite DFT of P points
constexpr int c2_split(int P)
{
    if ((P & (P - 1)) == 0) return P == 16 ? 4 : 8;  // 16 = 4 x 4, 32 = 8 x 4
    for (int p : {4, 2, 3, 5, 7, 11, 13, 17})
        if (P % p == 0 && P > p) return p;
    return P;
}

constexpr bool c2_is_leaf(int P)
{
    return P == 1 || P == 2 || P == 3 || P == 4 || P == 5 || P == 7 || P == 8 || P == 11 || P == 13 ||
           P == 17;
}

// cos / sin of 2 pi m / P with exact zeros and ones (folded by the compiler)
template <int P>
struct DftConst2 {
    float c[P], s[P];
    constexpr DftConst2() : c(), s()
    {
        for (int m = 0; m < P; ++m) {
            double cc = 0.0, ss = 0.0;
            if (4 * m == P) { cc = 0.0; ss = 1.0; }
            else if (2 * m == P) { cc = -1.0; ss = 0.0; }
            else if (4 * m == 3 * P) { cc = 0.0; ss = -1.0; }
            else if (m == 0) { cc = 1.0; ss = 0.0; }
            else {
                // reduce to [-pi, pi] for the Taylor series
                double x = 2.0 * ct_pi * m / P;
                if (x > ct_pi) x -= 2.0 * ct_pi;
                cc = ct_taylor_cos(x);
                ss = ct_taylor_sin(x);
            }
            c[m] = (float)cc;
            s[m] = (float)ss;
        }
    }
};

// a * (c + i s) with c, s compile-time constants after unrolling
__device__ __forceinline__ float2 cmul_k(float2 a, float c, float s)
{
    if (s == 0.f) {
        if (c == 1.f) return a;
        if (c == -1.f) return make_float2(-a.x, -a.y);
        return make_float2(a.x * c, a.y * c);
    }
    if (c == 0.f) {
        if (s == 1.f) return make_float2(-a.y, a.x);
        if (s == -1.f) return make_float2(a.y, -a.x);
        return make_float2(-s * a.y, s * a.x);
    }
    return make_float2(fmaf(a.x, c, -s * a.y), fmaf(a.x, s, c * a.y));
}

// In-register DFT of P points: X_k = sum_n a_n exp(-+ 2 pi i n k / P)
template <int P, bool INV>
__device__ __forceinline__ void dft_reg(float2 (&a)[P])
{
    if constexpr (P == 1) {
        return;
    } else if constexpr (c2_is_leaf(P)) {
        dft_small<P>(a, INV ? 1.0f : -1.0f);
    } else {
        constexpr int P1 = c2_split(P), P2 = P / P1;
        constexpr DftConst2<P> K{};
        float2 y[P];
        // n = P2 n1 + n2, k = k1 + P1 k2
#pragma unroll
        for (int n2 = 0; n2 < P2; ++n2) {
            float2 b[P1];
#pragma unroll
            for (int n1 = 0; n1 < P1; ++n1) b[n1] = a[P2 * n1 + n2];
            dft_reg<P1, INV>(b);
#pragma unroll
            for (int k1 = 0; k1 < P1; ++k1) {
                const int m = (n2 * k1) % P;
                y[k1 * P2 + n2] = cmul_k(b[k1], K.c[m], INV ? K.s[m] : -K.s[m]);
            }
        }
#pragma unroll
        for (int k1 = 0; k1 < P1; ++k1) {
            float2 c[P2];
#pragma unroll
            for (int n2 = 0; n2 < P2; ++n2) c[n2] = y[k1 * P2 + n2];
            dft_reg<P2, INV>(c);
#pragma unroll
            for (int k2 = 0; k2 < P2; ++k2) a[k1 + P1 * k2] = c[k2];
        }
    }
}

// Engine geometry: length N, V vectors per CTA, TV threads per vector,
// radices <= PMAX.  Shared layout (one pad slot per 2^LG elements):
//   rows:    element j of vector v at v * RS + j + (j >> LG)
//   columns: element u of vector v at (u + (u >> LG)) * V + v
template <int N_, int V_, int TV_, int PMAX_, bool REV_ = false>
struct Fft2 {
    static constexpr int N = N_, V = V_, TV = TV_, THREADS = V_ * TV_, PMAX = PMAX_;
    static constexpr Plan2 fplan = c2_plan(N_, PMAX_);
    static constexpr Plan2 plan = REV_ ? c2_reverse(fplan) : fplan;
    using Rev = Fft2<N_, V_, TV_, PMAX_, !REV_>;
    static constexpr int NST = plan.n;
    static constexpr int radix(int i) { return plan.r[i]; }
    static constexpr int stride(int i)
    {
        int s = 1;
        for (int k = 0; k < i; ++k) s *= plan.r[k];
        return s;
    }
    static constexpr int LG = fplan.r[0] <= 16 ? 4 : 5;  // one layout for both radix orders
    static constexpr int PADN = N_ + (N_ >> LG) + 1;  // padded vector length
    __device__ static __forceinline__ int ra(int v, int j) { return v * PADN + j + (j >> LG); }
    __device__ static __forceinline__ int ca(int v, int u) { return (u + (u >> LG)) * V_ + v; }
    static constexpr size_t smem_bytes() { return (size_t)PADN * V_ * sizeof(float2); }
};

// One Stockham stage over the thread's butterflies.  ld(j) returns input j,
// st(o, y) stores output o.  MID: a barrier between all loads and all stores
// (in-place shared-memory stages).
template <class G, bool INV, int I, bool MID, class Ld, class St>
__device__ __forceinline__ void s2_stage(int t, const float2* __restrict__ tw, Ld&& ld, St&& st)
{
    constexpr int N = G::N, TV = G::TV;
    constexpr int P = G::radix(I), S = G::stride(I);
    constexpr int NBP = N / P;
    constexpr int NB = (NBP + TV - 1) / TV;
    constexpr bool PRED = NB * TV != NBP;
    constexpr bool LAST = S * P == N;  // q == 0: no outer twiddles
    float2 a[NB][P];
#pragma unroll
    for (int i = 0; i < NB; ++i) {
        const int bb = t + i * TV;
        if (!PRED || bb < NBP) {
#pragma unroll
            for (int r = 0; r < P; ++r) a[i][r] = ld(bb + r * NBP);
        }
    }
    if constexpr (MID) __syncthreads();
#pragma unroll
    for (int i = 0; i < NB; ++i) {
        const int bb = t + i * TV;
        if (!PRED || bb < NBP) {
            dft_reg<P, INV>(a[i]);
            if constexpr (LAST) {
#pragma unroll
                for (int tt = 0; tt < P; ++tt) st(bb + S * tt, a[i][tt]);
            } else {
                const int q = bb / S, k = bb - q * S;
                const int obase = k + S * P * q;
                st(obase, a[i][0]);
                float2 w1 = __ldg(&tw[q * S]);
                if (INV) w1.y = -w1.y;
                if constexpr (P <= 8) {
                    float2 wt = w1;
#pragma unroll
                    for (int tt = 1; tt < P; ++tt) {
                        st(obase + S * tt, cmul(a[i][tt], wt));
                        if (tt + 1 < P) wt = cmul(wt, w1);
                    }
                } else {
                    // w^t = (w^8)^(t/8) w^(t%8): w^8 from the table, at most
                    // 7 + P/8 - 1 sequential products per power
                    float2 wl[8];
                    wl[1] = w1;
#pragma unroll
                    for (int b = 2; b < 8; ++b) wl[b] = cmul(wl[b - 1], w1);
                    float2 w8 = __ldg(&tw[8 * q * S]);
                    if (INV) w8.y = -w8.y;
                    float2 wh = w8;
#pragma unroll
                    for (int tt = 1; tt < P; ++tt) {
                        if (tt >= 16 && tt % 8 == 0) wh = cmul(wh, w8);
                        const float2 w = tt < 8 ? wl[tt] : (tt % 8 == 0 ? wh : cmul(wh, wl[tt % 8]));
                        st(obase + S * tt, cmul(a[i][tt], w));
                    }
                }
            }
        }
    }
}

// The last stage of a forward transform on plan G fused with the first stage
// of the inverse on the reversed plan G::Rev.  Stockham's last stage maps
// the inputs {bb + r N/P} of butterfly bb to the outputs {bb + t N/P}, and
// the reversed plan's first stage (same radix P, stride 1) reads exactly
// {bb + r N/P} for the same bb: the thread keeps its butterflies in
// registers across the two stages, applying scale(u) to element u in
// between, instead of a shared-memory round trip and a barrier.  ld reads
// the forward's input u (shared memory), st stores the inverse stage-0
// output o.  The caller syncs before and after (in-place buffer).
template <class G, class Ld, class Sc, class St>
__device__ __forceinline__ void s2_fwd_last_inv_first(int t, const float2* __restrict__ tw, Ld&& ld, Sc&& scale,
                                                      St&& st)
{
    using R = typename G::Rev;
    constexpr int N = G::N, TV = G::TV;
    constexpr int P = G::radix(G::NST - 1);
    static_assert(R::radix(0) == P && R::stride(0) == 1 && G::stride(G::NST - 1) * P == N, "reversed plan");
    constexpr int NBP = N / P;
    constexpr int NB = (NBP + TV - 1) / TV;
    constexpr bool PRED = NB * TV != NBP;
    float2 a[NB][P];
#pragma unroll
    for (int i = 0; i < NB; ++i) {
        const int bb = t + i * TV;
        if (!PRED || bb < NBP) {
#pragma unroll
            for (int r = 0; r < P; ++r) a[i][r] = ld(bb + r * NBP);
        }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < NB; ++i) {
        const int bb = t + i * TV;
        if (!PRED || bb < NBP) {
            dft_reg<P, false>(a[i]);  // forward: y[bb + t N/P] = a[i][t]
#pragma unroll
            for (int r = 0; r < P; ++r) a[i][r] = cscale(a[i][r], scale(bb + r * NBP));
            dft_reg<P, true>(a[i]);  // inverse stage 0 (stride 1): q = bb, outputs P bb + t
            const int obase = P * bb;
            st(obase, a[i][0]);
            float2 w1 = __ldg(&tw[bb]);
            w1.y = -w1.y;
            if constexpr (P <= 8) {
                float2 wt = w1;
#pragma unroll
                for (int tt = 1; tt < P; ++tt) {
                    st(obase + tt, cmul(a[i][tt], wt));
                    if (tt + 1 < P) wt = cmul(wt, w1);
                }
            } else {
                float2 wl[8];
                wl[1] = w1;
#pragma unroll
                for (int b = 2; b < 8; ++b) wl[b] = cmul(wl[b - 1], w1);
                float2 w8 = __ldg(&tw[8 * bb]);
                w8.y = -w8.y;
                float2 wh = w8;
#pragma unroll
                for (int tt = 1; tt < P; ++tt) {
                    if (tt >= 16 && tt % 8 == 0) wh = cmul(wh, w8);
                    const float2 w = tt < 8 ? wl[tt] : (tt % 8 == 0 ? wh : cmul(wh, wl[tt % 8]));
                    st(obase + tt, cmul(a[i][tt], w));
                }
            }
        }
    }
}

// stages [I, E) in place in shared memory (barrier after each)
template <class G, bool COLS, bool INV, int I, int E>
__device__ __forceinline__ void s2_smem_stages(float2* buf, int v, int t, const float2* __restrict__ tw)
{
    if constexpr (I < E) {
        auto ld = [&](int j) { return buf[COLS ? G::ca(v, j) : G::ra(v, j)]; };
        auto st = [&](int j, float2 z) { buf[COLS ? G::ca(v, j) : G::ra(v, j)] = z; };
        s2_stage<G, INV, I, true>(t, tw, ld, st);
        __syncthreads();
        s2_smem_stages<G, COLS, INV, I + 1, E>(buf, v, t, tw);
    }
}

}  // namespace blfls
