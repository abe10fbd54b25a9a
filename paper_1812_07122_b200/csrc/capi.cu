// capi.cu -- the extern "C" boundary (include/blfls/blfls.h): plans,
// workspaces, validation with the reference's error semantics, and the
// per-iteration kernel sequence
//
//   min/max(f) -> grad+BLF(f) -> row r2c (+ divergence fold) -> column solve
//   -> row c2r (+ next min/max)
//
// replayed as a cached CUDA graph on the plan's own stream.
#include <algorithm>
#include <complex>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "blfls_internal.cuh"

namespace blfls {

#ifdef BLFLS_EXPERIMENTS
int knob(const char* name, int def)
{
    const char* e = std::getenv(name);
    return e ? std::atoi(e) : def;
}
#endif

cudaError_t launch_grad_blf(const BlfParams& p, int mode, int batch, cudaStream_t st);
cudaError_t launch_row_r2c(const SolveParams& p, const FftGeom& g, int planes, bool odd,
                           cudaStream_t st);
cudaError_t launch_col(const SolveParams& p, const FftGeom& g, int planes, cudaStream_t st);
cudaError_t launch_row_c2r(const SolveParams& p, const FftGeom& g, int planes, bool odd,
                           cudaStream_t st);
cudaError_t launch_minmax(const float* x, size_t per_image, int batch, uint32_t* lohi, int nsm,
                          cudaStream_t st);
cudaError_t launch_reset_lohi(uint32_t* lohi, int n, cudaStream_t st);
cudaError_t launch_count_nonfinite(const float* x, size_t n, unsigned* count, int nsm, cudaStream_t st);
cudaError_t launch_scale_by_range(float* x, size_t per_image, int batch, const uint32_t* lohi,
                                  int to_raw, cudaStream_t st);
cudaError_t launch_generate(int H, int W, int planes, const uint64_t* seeds, int K, double sigma,
                            double p_sp, float* out, cudaStream_t st);
cudaError_t measure_mufu(int device, double* ex2_per_s, double* clock_hz);
cudaError_t launch_reflect_pad(const float* src, float* dst, int H, int W, int pad, size_t planes,
                               int nsm, cudaStream_t st);
cudaError_t launch_grid_blf(const GridParams& p, int nsm, cudaStream_t st, int* launches);
bool ct_geometry(bool cols, int n, int nvec, int planes, int nsm, int* V, int* threads);

}  // namespace blfls

using namespace blfls;

namespace {

thread_local std::string g_err;

blfls_status fail(blfls_status st, const std::string& msg)
{
    g_err = msg;
    return st;
}

blfls_status cuda_fail(cudaError_t e, const char* where)
{
    g_err = std::string(where) + ": " + cudaGetErrorString(e);
    return e == cudaErrorMemoryAllocation ? BLFLS_ENOMEM : BLFLS_ECUDA;
}

#define CK(expr)                                               \
    do {                                                       \
        cudaError_t e_ = (expr);                               \
        if (e_ != cudaSuccess) return cuda_fail(e_, #expr);    \
    } while (0)

struct DevFft {
    FftGeom g{};
    float2* tw = nullptr;
    // Bluestein tables (device): chirp (n), M-point twiddles, kernel spectra
    float2* chirp = nullptr;
    float2* btw = nullptr;
    float2* hf = nullptr;
    float2* hi = nullptr;
};

// Bluestein for lengths with a prime factor above this (the direct stage
// below it); BLFLS_BLUESTEIN_MINP overrides (0 disables Bluestein)
int bluestein_min_prime()
{
    static const int v = knob("BLFLS_BLUESTEIN_MINP", 150);  // measured: P = 61, 43 faster direct, P = 139 a tie
    return v;
}

bool smooth235(int m)
{
    for (int p : {2, 3, 5})
        while (m % p == 0) m /= p;
    return m == 1;
}

// host mixed-radix (2, 3, 5) FFT in double, sign -1 forward (table setup only)
void host_fft(std::vector<std::complex<double>>& a, int sign)
{
    const int n = (int)a.size();
    if (n == 1) return;
    int p = n % 2 == 0 ? 2 : (n % 3 == 0 ? 3 : 5);
    const int m = n / p;
    std::vector<std::vector<std::complex<double>>> sub(p, std::vector<std::complex<double>>(m));
    for (int j = 0; j < m; ++j)
        for (int r = 0; r < p; ++r) sub[r][j] = a[(size_t)j * p + r];
    for (auto& v : sub) host_fft(v, sign);
    for (int k = 0; k < n; ++k) {
        std::complex<double> acc = 0.0;
        for (int r = 0; r < p; ++r) {
            const double ang = sign * 2.0 * M_PI * (double)(((long long)r * k) % n) / n;
            acc += sub[r][k % m] * std::complex<double>(std::cos(ang), std::sin(ang));
        }
        a[k] = acc;
    }
}

bool factorize(int n, std::vector<int>& radix)
{
    radix.clear();
    int m = n;
    while (m % 4 == 0) { radix.push_back(4); m /= 4; }
    while (m % 2 == 0) { radix.push_back(2); m /= 2; }
    for (int p : {3, 5}) while (m % p == 0) { radix.push_back(p); m /= p; }
    // any other prime: 7..13 register-staged generic stage, larger ones the
    // direct DFT stage (sizes produced by reflect padding)
    for (int p = 7; (long)p * p <= m; p += 2)
        while (m % p == 0) { radix.push_back(p); m /= p; }
    if (m > 1) radix.push_back(m);
    return (int)radix.size() <= kMaxFftRadices;
}

// threads per vector so that every stage fits the E-register budget of fft_stage
int threads_per_vector(const std::vector<int>& radix, int n, int E)
{
    int tv = 1;
    for (int p : radix) {
        if (p > 13) continue;  // direct stage: any thread count
        const int nbp = n / p;
        const int nb = p <= 5 ? (E + p - 1) / p : (2 * E) / p;
        if (nb < 1) return 1 << 30;
        tv = std::max(tv, (nbp + nb - 1) / nb);
    }
    return tv;
}

// V (power of two, <= Vmax) vectors of length n per CTA, <= 1024 threads,
// <= smem_cap bytes of shared memory; largest V first, then the smaller E.
bool plan_fft(int n, int Vmax, size_t smem_cap, bool cols, bool odd, int nvec, int planes, int nsm,
              DevFft& out, std::vector<int>& radix)
{
    if (!factorize(n, radix)) return false;
    bool generic = false, direct = false;
    int pmax = 1;
    for (int p : radix) {
        generic |= p > 5;
        direct |= p > 13;
        pmax = std::max(pmax, p);
    }
    int cv = 0, ct = 0;
    if (!odd && ct_geometry(cols, n, nvec, planes, nsm, &cv, &ct)) {
        FftGeom& g = out.g;
        g.V = cv;
        g.log2V = 0;
        while ((1 << g.log2V) < cv) ++g.log2V;
        g.threads = ct;
        g.E = 16;
        g.generic = false;
        g.direct = false;
        g.ct = true;
        return true;
    }
    const int bmin = bluestein_min_prime();
    if (bmin > 0 && pmax > bmin) {
        // Bluestein: the transform becomes a cyclic convolution of 5-smooth length M
        int M = 2 * n - 1;
        while (!smooth235(M)) ++M;
        std::vector<int> mrad;
        factorize(M, mrad);
        for (int V = Vmax; V >= 1; V >>= 1) {
            if ((size_t)V * (n + M) * 8 > smem_cap) continue;
            for (int E : {8, 16}) {
                int tv = threads_per_vector(mrad, M, E);
                while ((tv * V) % 32 != 0) ++tv;
                if ((long)tv * V > 1024) continue;
                FftGeom& g = out.g;
                g.V = V;
                g.log2V = 0;
                while ((1 << g.log2V) < V) ++g.log2V;
                g.threads = tv * V;
                g.E = E;
                g.generic = false;
                g.direct = false;
                g.pmax = pmax;
                g.ct = false;
                g.bluestein = true;
                g.blue.m.n = M;
                g.blue.m.nstages = (int)mrad.size();
                for (size_t i = 0; i < mrad.size(); ++i) g.blue.m.radix[i] = mrad[i];
                return true;
            }
        }
    }
    for (int V = Vmax; V >= 1; V >>= 1) {
        // direct stages: strip + scratch copy + root table of the largest prime
        if ((size_t)V * n * 8 * (direct ? 2 : 1) + (direct ? (size_t)pmax * 8 : 0) > smem_cap) continue;
        for (int E : {8, 16}) {
            int tv = threads_per_vector(radix, n, E);
            // whole warps per CTA: the block reductions shuffle over full warps
            while ((tv * V) % 32 != 0) ++tv;
            if ((long)tv * V > 1024) continue;
            FftGeom& g = out.g;
            g.V = V;
            g.log2V = 0;
            while ((1 << g.log2V) < V) ++g.log2V;
            g.threads = tv * V;
            g.E = E;
            g.generic = generic;
            g.direct = direct;
            g.pmax = pmax;
            g.ct = false;
            return true;
        }
    }
    return false;
}

std::vector<float2> twiddles(int n)
{
    std::vector<float2> t(n);
    for (int j = 0; j < n; ++j) {
        const double a = -2.0 * M_PI * (double)j / (double)n;
        t[j] = make_float2((float)std::cos(a), (float)std::sin(a));
    }
    return t;
}

struct EventPair {
    cudaEvent_t a, b;
    int stage;
};

}  // namespace

struct blfls_plan_s {
    blfls_params prm{};
    int radius = 0;
    int mode = 0;  // BLF kernel mode: 0 self, 1 per-channel guide, 2 shared gray guide
    int nsm = 148;
    cudaStream_t ps = nullptr;
    cudaEvent_t ev_in = nullptr, ev_out = nullptr;
    // plane-grouped solve: each group's half spectrum stays L2-resident across
    // its r2c -> column -> c2r kernels; two groups in flight on ps / ps2
    int solve_group = 0;           // planes per group (0: one launch over all planes)
    cudaStream_t ps2 = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    // FFT
    bool odd = false;
    int wc = 0, spitch = 0;
    DevFft rowf, colf;
    float* gain_x = nullptr;
    float* gain_y = nullptr;
    float2* post = nullptr;
    float4* tri = nullptr;       // tridiagonal column pass tables (k_col_tri.cu)
    int tri_rpt = 0;
    // workspace (max_batch images)
    size_t plane = 0, img_elems = 0;  // user (unpadded) plane H*W
    // reflect padding: the BLF and the solve run on the padded grid Hp x Wp
    int pad = 0, Hp = 0, Wp = 0;
    size_t pplane = 0;
    float* fpad = nullptr;   // padded current image
    float* gpad = nullptr;   // padded guide
    // bilateral-grid backend workspace (backend == BLFLS_BACKEND_GRID)
    GridParams grid{};
    int grid_planes = 0;     // planes per grid launch (2 slots each)
    // domain-transform backend workspace (backend == BLFLS_BACKEND_DT)
    DtParams dt{};
    int dt_planes = 0;       // planes per DT launch group (2 slots each)
    int dt_iters = 0;
    float* buf[2] = {nullptr, nullptr};
    float* tx = nullptr;
    float* ty = nullptr;
    float2* spec = nullptr;
    float* in_dev = nullptr;     // host-pointer staging (stage entry points)
    float* guide_dev = nullptr;
    float* out_dev = nullptr;
    // blfls_run with host pointers: two staging slots, H2D / D2H on their own
    // streams, so consecutive BLFLS_ASYNC calls overlap copies with compute
    struct HostSlot {
        float* in = nullptr;
        float* guide = nullptr;
        float* out = nullptr;
        cudaEvent_t h2d = nullptr, comp = nullptr, d2h = nullptr;
        bool used = false;
    } slot[2];
    int next_slot = 0;
    cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
    unsigned* nonfinite_acc = nullptr;  // deferred non-finite count of ASYNC calls
    uint32_t* lohi = nullptr;    // [2][max_batch][2]
    uint32_t* glohi = nullptr;   // [max_batch][2]
    unsigned* nonfinite = nullptr;
    BlfParams blf{};
    // graph cache: instantiated iteration sequences keyed on their pointers
    struct GraphEntry {
        cudaGraphExec_t exec = nullptr;
        const void* in = nullptr;
        const void* guide = nullptr;
        void* out = nullptr;
        int batch = -1, iters = -1;
        long long last = 0;
        long long launches = 0;
    } graphs[4];
    long long graph_clock = 0;
    // stats
    blfls_stats stats{};
    long long launches = 0;
    std::vector<EventPair> timing;
    bool time_stages = false;
};

namespace {

blfls_status set_device(blfls_plan_t p)
{
    CK(cudaSetDevice(p->prm.device));
    return BLFLS_OK;
}

// --------------------------------------------------------------- stages --

void stage_begin(blfls_plan_t p, int stage, cudaStream_t st)
{
    if (!p->time_stages) return;
    EventPair e{};
    cudaEventCreate(&e.a);
    cudaEventCreate(&e.b);
    e.stage = stage;
    cudaEventRecord(e.a, st);
    p->timing.push_back(e);
}

void stage_end(blfls_plan_t p, cudaStream_t st)
{
    if (!p->time_stages) return;
    cudaEventRecord(p->timing.back().b, st);
}

SolveParams solve_params(blfls_plan_t p)
{
    SolveParams s{};
    s.H = p->Hp;
    s.W = p->Wp;
    s.C = p->prm.channels;
    s.oH = p->prm.height;
    s.oW = p->prm.width;
    s.opad = p->pad;
    s.spitch = p->spitch;
    s.wc = p->wc;
    s.lambda = (float)p->prm.lambda;
    s.inv_hw = (float)(1.0 / ((double)s.H * (double)s.W));
    s.gain_x = p->gain_x;
    s.gain_y = p->gain_y;
    s.post = p->post;
    s.spec = p->spec;
    s.tri = p->tri;
    s.tri_rpt = p->tri_rpt;
    return s;
}

blfls_status enq_solve(blfls_plan_t p, const float* f, const float* tx, const float* ty, float* out,
                       uint32_t* lohi_out, int batch, cudaStream_t st)
{
    const int planes = batch * p->prm.channels;
    SolveParams s = solve_params(p);
    s.f = f;
    s.tx = tx;
    s.ty = ty;
    s.out = out;
    s.lohi_out = lohi_out;
    s.mode = 3;
    s.plane0 = 0;
    const int grp = p->solve_group;
    if (grp <= 0 || grp >= planes) {
        stage_begin(p, 2, st);
        CK(launch_row_r2c(s, p->rowf.g, planes, p->odd, st));
        stage_end(p, st);
        // the tridiagonal column pass resets the (lo, hi) slots of the c2r epilogue
        const bool fused_reset = lohi_out != nullptr && s.tri != nullptr;
        if (fused_reset) {
            s.lohi_reset = lohi_out;
            s.lohi_reset_n = batch;
        }
        stage_begin(p, 3, st);
        CK(launch_col(s, p->colf.g, planes, st));
        stage_end(p, st);
        if (lohi_out && !fused_reset) {
            CK(launch_reset_lohi(lohi_out, batch, st));
            p->launches++;
        }
        stage_begin(p, 4, st);
        CK(launch_row_c2r(s, p->rowf.g, planes, p->odd, st));
        stage_end(p, st);
        p->launches += 3;
        return BLFLS_OK;
    }
    // grouped: spectrum regions 0 / 1 alternate between the two streams
    const size_t pimg = p->pplane;                      // padded inputs
    const size_t pout = p->plane;                       // cropped outputs
    const size_t pspec = (size_t)p->Hp * p->spitch;
    if (lohi_out) {
        CK(launch_reset_lohi(lohi_out, batch, st));
        p->launches++;
    }
    stage_begin(p, 2, st);  // the whole grouped solve is timed as stage 2
    CK(cudaEventRecord(p->ev_fork, st));
    CK(cudaStreamWaitEvent(p->ps2, p->ev_fork, 0));
    int k = 0;
    for (int p0 = 0; p0 < planes; p0 += grp, ++k) {
        const int np = std::min(grp, planes - p0);
        cudaStream_t cs = (k & 1) ? p->ps2 : st;
        SolveParams g = s;
        g.plane0 = p0;
        g.f = f + p0 * pimg;
        g.tx = tx ? tx + p0 * pimg : nullptr;
        g.ty = ty ? ty + p0 * pimg : nullptr;
        g.out = out + p0 * pout;
        g.spec = p->spec + (size_t)(k & 1) * grp * pspec;
        CK(launch_row_r2c(g, p->rowf.g, np, p->odd, cs));
        CK(launch_col(g, p->colf.g, np, cs));
        CK(launch_row_c2r(g, p->rowf.g, np, p->odd, cs));
        p->launches += 3;
    }
    CK(cudaEventRecord(p->ev_join, p->ps2));
    CK(cudaStreamWaitEvent(st, p->ev_join, 0));
    stage_end(p, st);
    return BLFLS_OK;
}

blfls_status enq_grid(blfls_plan_t p, const float* f, const float* guide, const uint32_t* lohi,
                      float* tx, float* ty, int batch, int normalized, cudaStream_t st)
{
    GridParams g = p->grid;
    g.f = f;
    g.guide = guide;
    g.tx = tx;
    g.ty = ty;
    g.lohi = lohi;
    g.glohi = p->glohi;
    g.normalized = normalized;
    const int planes = batch * p->prm.channels;
    stage_begin(p, 1, st);
    for (int p0 = 0; p0 < planes; p0 += p->grid_planes) {
        g.plane0 = p0;
        g.slots = 2 * std::min(p->grid_planes, planes - p0);
        int n = 0;
        CK(launch_grid_blf(g, p->nsm, st, &n));
        p->launches += n;
    }
    stage_end(p, st);
    p->stats.blf_launches++;
    return BLFLS_OK;
}

blfls_status enq_dt(blfls_plan_t p, const float* f, const float* guide, const uint32_t* lohi,
                    float* tx, float* ty, int batch, int normalized, cudaStream_t st)
{
    DtParams d = p->dt;
    d.f = f;
    d.guide = guide;
    d.tx = tx;
    d.ty = ty;
    d.lohi = lohi;
    d.glohi = p->glohi;
    d.normalized = normalized;
    const int planes = batch * p->prm.channels;
    stage_begin(p, 1, st);
    for (int p0 = 0; p0 < planes; p0 += p->dt_planes) {
        d.plane0 = p0;
        d.slots = 2 * std::min(p->dt_planes, planes - p0);
        const int n = launch_dt_filter(d, p->dt_iters, p->prm.sigma_s, p->nsm, st);
        if (n < 0) CK(cudaGetLastError());
        p->launches += n;
    }
    stage_end(p, st);
    p->stats.blf_launches++;
    return BLFLS_OK;
}

blfls_status enq_blf(blfls_plan_t p, const float* f, const float* guide, const uint32_t* lohi,
                     float* tx, float* ty, int batch, int y0, int y1, int out_rows, int normalized,
                     cudaStream_t st)
{
    if (p->prm.backend == BLFLS_BACKEND_DT) {
        if (y0 != 0 || y1 != p->Hp) return fail(BLFLS_EUNSUPPORTED, "dt backend: no row bands");
        return enq_dt(p, f, guide, lohi, tx, ty, batch, normalized, st);
    }
    if (p->prm.backend == BLFLS_BACKEND_GRID) {
        if (y0 != 0 || y1 != p->Hp) return fail(BLFLS_EUNSUPPORTED, "grid backend: no row bands");
        return enq_grid(p, f, guide, lohi, tx, ty, batch, normalized, st);
    }
    BlfParams b = p->blf;
    b.f = f;
    b.guide = guide;
    b.tx = tx;
    b.ty = ty;
    b.lohi = lohi;
    b.glohi = p->glohi;
    b.y0 = y0;
    b.y1 = y1;
    b.out_rows = out_rows;
    b.normalized_out = normalized;
    stage_begin(p, 1, st);
    CK(launch_grad_blf(b, p->mode, batch, st));
    stage_end(p, st);
    p->launches++;
    p->stats.blf_launches++;
    return BLFLS_OK;
}

blfls_status enq_minmax(blfls_plan_t p, const float* x, size_t per_image, int batch, uint32_t* lohi,
                        cudaStream_t st)
{
    stage_begin(p, 0, st);
    CK(launch_minmax(x, per_image, batch, lohi, p->nsm, st));
    stage_end(p, st);
    p->launches += 2;
    return BLFLS_OK;
}

// the whole cascade on device pointers
blfls_status enq_run(blfls_plan_t p, const float* in, const float* guide, float* out, int batch,
                     int iters, cudaStream_t st)
{
    const size_t per_image = (size_t)p->prm.channels * p->plane;
    const int mb = p->prm.max_batch;
    blfls_status r;
    if (guide) {
        r = enq_minmax(p, guide, (size_t)p->prm.guide_channels * p->plane, batch, p->glohi, st);
        if (r) return r;
    }
    // The image's own (lo, hi) (normalize_to_unit, image.cpp:46-60) only
    // enters the range kernel when the image guides itself: the solve is
    // affine-equivariant (den(0,0) = 1, conj(otf)(0) = 0), so with a separate
    // guide the normalise / denormalise pair cancels exactly and the
    // brute-force kernels never read it (the grid / DT backends normalise the
    // image like the reference and do).  Skipped for guided brute force: the
    // iteration-1 min/max pass (c5: 3.2 GB, 0.5 ms per step) and the c2r
    // epilogue's reductions.
    const bool need_range = !(p->prm.backend == BLFLS_BACKEND_BRUTE && p->prm.guide_channels > 0);
    if (need_range) {
        r = enq_minmax(p, in, per_image, batch, p->lohi, st);
        if (r) return r;
    }
    const float* g_use = guide;
    if (guide && p->pad > 0) {  // pipelines.cpp:82-83: the guide is padded once
        CK(launch_reflect_pad(guide, p->gpad, p->prm.height, p->prm.width, p->pad,
                              (size_t)batch * p->prm.guide_channels, p->nsm, st));
        p->launches++;
        g_use = p->gpad;
    }
    const float* cur = in;
    for (int k = 0; k < iters; ++k) {
        const bool last = k == iters - 1;
        float* nxt = last ? out : p->buf[k & 1];
        uint32_t* lo_cur = p->lohi + (size_t)(k & 1) * 2 * mb;
        uint32_t* lo_nxt = (last || !need_range) ? nullptr : p->lohi + (size_t)((k + 1) & 1) * 2 * mb;
        const float* f = cur;
        if (p->pad > 0) {  // pipelines.cpp:76-78: reflect-pad every smooth() input
            CK(launch_reflect_pad(cur, p->fpad, p->prm.height, p->prm.width, p->pad,
                                  (size_t)batch * p->prm.channels, p->nsm, st));
            p->launches++;
            f = p->fpad;
        }
        r = enq_blf(p, f, g_use, lo_cur, p->tx, p->ty, batch, 0, p->Hp, p->Hp, 0, st);
        if (r) return r;
        r = enq_solve(p, f, p->tx, p->ty, nxt, lo_nxt, batch, st);  // c2r crops (pipelines.cpp:92)
        if (r) return r;
        cur = nxt;
    }
    return BLFLS_OK;
}

blfls_status validate_batch(blfls_plan_t p, int batch)
{
    if (!p) return fail(BLFLS_EINVAL, "null plan");
    if (batch < 1 || batch > p->prm.max_batch)
        return fail(BLFLS_EINVAL, "batch must be in [1, max_batch]");
    return BLFLS_OK;
}

blfls_status check_finite(blfls_plan_t p, const float* x, size_t n, cudaStream_t st, const char* what)
{
    CK(cudaMemsetAsync(p->nonfinite, 0, sizeof(unsigned), st));
    CK(launch_count_nonfinite(x, n, p->nonfinite, p->nsm, st));
    unsigned h = 0;
    CK(cudaMemcpyAsync(&h, p->nonfinite, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (h) return fail(BLFLS_ENONFINITE, std::string(what) + ": non-finite sample in input image");
    return BLFLS_OK;
}

// join the caller's stream into the plan stream and back
blfls_status fork_in(blfls_plan_t p, cudaStream_t user)
{
    CK(cudaEventRecord(p->ev_in, user));
    CK(cudaStreamWaitEvent(p->ps, p->ev_in, 0));
    return BLFLS_OK;
}

blfls_status join_out(blfls_plan_t p, cudaStream_t user, unsigned flags)
{
    CK(cudaEventRecord(p->ev_out, p->ps));
    CK(cudaStreamWaitEvent(user, p->ev_out, 0));
    if (flags & BLFLS_SYNC) CK(cudaStreamSynchronize(user));
    return BLFLS_OK;
}

void free_plan(blfls_plan_t p)
{
    if (!p) return;
    cudaSetDevice(p->prm.device);
    for (auto& g : p->graphs)
        if (g.exec) cudaGraphExecDestroy(g.exec);
    for (auto& sl : p->slot) {
        if (sl.in) cudaFree(sl.in);
        if (sl.guide) cudaFree(sl.guide);
        if (sl.out) cudaFree(sl.out);
        if (sl.h2d) cudaEventDestroy(sl.h2d);
        if (sl.comp) cudaEventDestroy(sl.comp);
        if (sl.d2h) cudaEventDestroy(sl.d2h);
    }
    if (p->nonfinite_acc) cudaFree(p->nonfinite_acc);
    if (p->s_h2d) cudaStreamDestroy(p->s_h2d);
    if (p->s_d2h) cudaStreamDestroy(p->s_d2h);
    for (auto& e : p->timing) {
        cudaEventDestroy(e.a);
        cudaEventDestroy(e.b);
    }
    void* ptrs[] = {p->tri, p->gain_x, p->gain_y, p->post, p->buf[0], p->buf[1], p->tx, p->ty, p->spec,
                    p->in_dev, p->guide_dev, p->out_dev, p->lohi, p->glohi, p->nonfinite,
                    p->rowf.tw, p->colf.tw, p->rowf.chirp, p->rowf.btw, p->rowf.hf, p->rowf.hi,
                    p->colf.chirp, p->colf.btw, p->colf.hf, p->colf.hi, p->fpad, p->gpad, p->grid.wgrid, p->grid.vgrid,
                    p->grid.blurred, p->grid.erange, p->dt.cth, p->dt.ctv, p->dt.pc, p->dt.x, p->dt.g01};
    for (void* q : ptrs)
        if (q) cudaFree(q);
    if (p->ev_in) cudaEventDestroy(p->ev_in);
    if (p->ev_fork) cudaEventDestroy(p->ev_fork);
    if (p->ev_join) cudaEventDestroy(p->ev_join);
    if (p->ps2) cudaStreamDestroy(p->ps2);
    if (p->ev_out) cudaEventDestroy(p->ev_out);
    if (p->ps) cudaStreamDestroy(p->ps);
    delete p;
}

}  // namespace

namespace blfls {
blfls_status report(blfls_status st, const std::string& msg) { return fail(st, msg); }
}  // namespace blfls

extern "C" {

const char* blfls_last_error(void) { return g_err.c_str(); }
const char* blfls_version(void) { return "blfls-b200 0.1 (sm_100a)"; }
int blfls_abi_version(void) { return BLFLS_ABI_VERSION; }

blfls_status blfls_plan_create(const blfls_params* prm, blfls_plan_t* out)
{
    if (!prm || !out) return fail(BLFLS_EINVAL, "null argument");
    *out = nullptr;
    const blfls_params& q = *prm;
    // image.cpp:14-17, solver.cpp:35-36
    if (q.height < 2 || q.width < 2)
        return fail(BLFLS_EINVAL, "plan: height and width must be >= 2");
    if (q.channels != 1 && q.channels != 3)
        return fail(BLFLS_EINVAL, "plan: channels must be 1 or 3");
    if (q.guide_channels != 0 && q.guide_channels != 1 && q.guide_channels != q.channels)
        return fail(BLFLS_EINVAL, "plan: guide channels must be 0, 1 or match the image");
    // bilateral.cpp:12-16
    if (!(q.sigma_s > 0.0) || !std::isfinite(q.sigma_s) || !(q.sigma_r > 0.0) ||
        !std::isfinite(q.sigma_r))
        return fail(BLFLS_EINVAL, "bilateral: sigma_s and sigma_r must be positive and finite");
    // solver.cpp:15-21
    if (!(q.lambda >= 0.0) || !std::isfinite(q.lambda))
        return fail(BLFLS_EINVAL, "solver: lambda must be finite and >= 0");
    if (q.max_batch < 1) return fail(BLFLS_EINVAL, "plan: max_batch must be >= 1");
    if (q.pad < 0) return fail(BLFLS_EINVAL, "solver: pad must be >= 0");  // solver.cpp:19-20
    if (q.pad > 4096) return fail(BLFLS_EUNSUPPORTED, "plan: pad above 4096");
    if (q.backend != BLFLS_BACKEND_BRUTE && q.backend != BLFLS_BACKEND_GRID &&
        q.backend != BLFLS_BACKEND_DT)
        return fail(BLFLS_EINVAL, "plan: unknown gradient-filter backend");
    if (q.backend == BLFLS_BACKEND_DT && q.dt_iterations < 0)  // domain_transform.cpp:27-28
        return fail(BLFLS_EINVAL, "nc_filter: iterations must be >= 1");
    const bool grid = q.backend == BLFLS_BACKEND_GRID;
    const bool brute = q.backend == BLFLS_BACKEND_BRUTE;  // the only one with a window radius
    const int radius = !brute ? 0 : (q.radius < 0 ? (int)std::ceil(3.0 * q.sigma_s) : q.radius);
    if (radius > kMaxRadius)
        return fail(BLFLS_EUNSUPPORTED, "plan: radius above " + std::to_string(kMaxRadius));

    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(BLFLS_ECUDA, "no CUDA device (this library has no CPU fallback)");
    if (q.device < 0 || q.device >= ndev) return fail(BLFLS_EINVAL, "plan: bad device ordinal");

    auto* p = new blfls_plan_s();
    p->prm = q;
    p->radius = radius;
    p->mode = q.guide_channels == 0 ? 0 : (q.guide_channels == 1 && q.channels == 3 ? 2 : 1);
    auto bail = [&](blfls_status st) {
        free_plan(p);
        return st;
    };
    if (cudaSetDevice(q.device) != cudaSuccess) return bail(fail(BLFLS_ECUDA, "cudaSetDevice failed"));
    cudaDeviceProp prop{};
    cudaGetDeviceProperties(&prop, q.device);
    if (prop.major < 10)
        return bail(fail(BLFLS_ECUDA, std::string("device is not sm_100-class: ") + prop.name));
    p->nsm = prop.multiProcessorCount;

    const int C = q.channels;
    p->pad = q.pad;
    p->Hp = q.height + 2 * q.pad;
    p->Wp = q.width + 2 * q.pad;
    // everything spectral and the BLF run on the padded grid
    const int H = p->Hp, W = p->Wp;
    p->odd = (W % 2) != 0;
    p->wc = W / 2 + 1;
    p->spitch = ((p->wc + 15) / 16) * 16;
    const int nrow = p->odd ? W : W / 2;
    std::vector<int> rrad, crad;
    // rows: about 2048 complex values per CTA
    int vrow = 1;
    while (vrow * 2 * nrow <= 2048 && vrow < 16) vrow *= 2;
    if (!plan_fft(nrow, vrow, 64 * 1024, false, p->odd, H, q.max_batch * C, p->nsm, p->rowf, rrad))
        return bail(fail(BLFLS_EUNSUPPORTED, "FFT: width " + std::to_string(W) +
                                                 " too large for the shared-memory row FFT"));
    if (!plan_fft(H, 16, 128 * 1024, true, false, p->wc, q.max_batch * C, p->nsm, p->colf, crad))
        return bail(fail(BLFLS_EUNSUPPORTED, "FFT: height " + std::to_string(H) +
                                                 " too large for the shared-memory column FFT"));

    if (knob("BLFLS_DEBUG_FFT", 0)) {
        for (const DevFft* f : {&p->rowf, &p->colf})
            std::fprintf(stderr, "blfls fft n=%d ct=%d bluestein=%d (M=%d) direct=%d pmax=%d V=%d threads=%d E=%d\n",
                         f->g.desc.n, (int)f->g.ct, (int)f->g.bluestein, f->g.blue.m.n, (int)f->g.direct,
                         f->g.pmax, f->g.V, f->g.threads, f->g.E);
    }
    // tables (double -> float)
    {
        auto tr = twiddles(nrow);
        auto tc = twiddles(H);
        std::vector<float> gx(p->wc), gy(H);
        std::vector<float2> post(p->wc);
        for (int v = 0; v < p->wc; ++v) {
            const double sx = std::sin(M_PI * v / W);
            gx[v] = (float)(4.0 * sx * sx);
            const double a = -2.0 * M_PI * v / W;
            post[v] = make_float2((float)std::cos(a), (float)std::sin(a));
        }
        for (int u = 0; u < H; ++u) {
            const double sy = std::sin(M_PI * u / H);
            gy[u] = (float)(4.0 * sy * sy);
        }
        if (cudaMalloc(&p->rowf.tw, sizeof(float2) * nrow) != cudaSuccess ||
            cudaMalloc(&p->colf.tw, sizeof(float2) * H) != cudaSuccess ||
            cudaMalloc(&p->gain_x, sizeof(float) * p->wc) != cudaSuccess ||
            cudaMalloc(&p->gain_y, sizeof(float) * H) != cudaSuccess ||
            cudaMalloc(&p->post, sizeof(float2) * p->wc) != cudaSuccess)
            return bail(fail(BLFLS_ENOMEM, "plan: table allocation failed"));
        cudaMemcpy(p->rowf.tw, tr.data(), sizeof(float2) * nrow, cudaMemcpyHostToDevice);
        cudaMemcpy(p->colf.tw, tc.data(), sizeof(float2) * H, cudaMemcpyHostToDevice);
        cudaMemcpy(p->gain_x, gx.data(), sizeof(float) * p->wc, cudaMemcpyHostToDevice);
        cudaMemcpy(p->gain_y, gy.data(), sizeof(float) * H, cudaMemcpyHostToDevice);
        cudaMemcpy(p->post, post.data(), sizeof(float2) * p->wc, cudaMemcpyHostToDevice);
        // the solve's column pass as a cyclic tridiagonal solve (BLFLS_COL_TRI=0
        // in the experiments build keeps the column FFT pair)
        const int rpt = tri_rows_per_thread(H, p->wc, q.max_batch * C, p->nsm);
        if (knob("BLFLS_COL_TRI", 1) != 0 && tri_supported(H, rpt)) {
            std::vector<float4> t4;
            tri_tables(H, W, p->wc, q.lambda, rpt, t4);
            if (cudaMalloc(&p->tri, sizeof(float4) * t4.size()) != cudaSuccess)
                return bail(fail(BLFLS_ENOMEM, "plan: table allocation failed"));
            cudaMemcpy(p->tri, t4.data(), sizeof(float4) * t4.size(), cudaMemcpyHostToDevice);
            p->tri_rpt = rpt;
        }
        auto fill = [](DevFft& f, int n, const std::vector<int>& rad) {
            f.g.desc.n = n;
            f.g.desc.nstages = (int)rad.size();
            for (size_t i = 0; i < rad.size(); ++i) f.g.desc.radix[i] = rad[i];
            f.g.desc.tw = f.tw;
        };
        fill(p->rowf, nrow, rrad);
        fill(p->colf, H, crad);
        for (DevFft* f : {&p->rowf, &p->colf}) {
            if (!f->g.bluestein) continue;
            const int n = f->g.desc.n, M = f->g.blue.m.n;
            std::vector<float2> ch(n);
            std::vector<std::complex<double>> hk(M, 0.0), hk_inv(M, 0.0);
            for (int j = 0; j < n; ++j) {  // c_j = exp(-pi i j^2 / n), angle reduced mod 2 pi
                const double a = -M_PI * (double)(((long long)j * j) % (2LL * n)) / n;
                const std::complex<double> c(std::cos(a), std::sin(a));
                ch[j] = make_float2((float)c.real(), (float)c.imag());
                hk[j] = std::conj(c);  // forward kernel h = conj(c); inverse: c
                hk_inv[j] = c;
                if (j) {
                    hk[M - j] = std::conj(c);
                    hk_inv[M - j] = c;
                }
            }
            host_fft(hk, -1);
            host_fft(hk_inv, -1);
            std::vector<float2> hf(M), hi(M);
            for (int k = 0; k < M; ++k) {
                hf[k] = make_float2((float)(hk[k].real() / M), (float)(hk[k].imag() / M));
                hi[k] = make_float2((float)(hk_inv[k].real() / M), (float)(hk_inv[k].imag() / M));
            }
            auto tm = twiddles(M);
            if (cudaMalloc(&f->chirp, sizeof(float2) * n) != cudaSuccess ||
                cudaMalloc(&f->btw, sizeof(float2) * M) != cudaSuccess ||
                cudaMalloc(&f->hf, sizeof(float2) * M) != cudaSuccess ||
                cudaMalloc(&f->hi, sizeof(float2) * M) != cudaSuccess)
                return bail(fail(BLFLS_ENOMEM, "plan: Bluestein table allocation failed"));
            cudaMemcpy(f->chirp, ch.data(), sizeof(float2) * n, cudaMemcpyHostToDevice);
            cudaMemcpy(f->btw, tm.data(), sizeof(float2) * M, cudaMemcpyHostToDevice);
            cudaMemcpy(f->hf, hf.data(), sizeof(float2) * M, cudaMemcpyHostToDevice);
            cudaMemcpy(f->hi, hi.data(), sizeof(float2) * M, cudaMemcpyHostToDevice);
            f->g.blue.m.tw = f->btw;
            f->g.blue.chirp = f->chirp;
            f->g.blue.hf = f->hf;
            f->g.blue.hi = f->hi;
        }
    }

    // BLF constants
    {
        BlfParams& b = p->blf;
        b.H = H;
        b.W = W;
        b.C = C;
        b.GC = q.guide_channels;
        b.radius = radius;
        b.poly_period = -1;
        b.poly_period = knob("BLFLS_POLY_PERIOD", b.poly_period);
        b.legacy_joint3 = 0;
        b.legacy_joint3 = -knob("BLFLS_PACKED_JOINT3", 0);
        b.x2_poly = -1;  // r01 sweep: packed kernel slower (FP32 pipe co-saturated); experiment only
        b.x2_poly = knob("BLFLS_X2", b.x2_poly);
        b.cols_per_thread = 4;
        b.cols_per_thread = knob("BLFLS_COLS", b.cols_per_thread);
        b.tile_rows = 0;
        b.tile_rows = knob("BLFLS_TILE_ROWS", b.tile_rows);
        b.joint3_rows = 2;
        b.joint3_rows = knob("BLFLS_J3_ROWS", b.joint3_rows);
        b.range_coef = (float)std::sqrt(1.4426950408889634 / (8.0 * q.sigma_r * q.sigma_r));
        for (int d = 0; d <= kMaxRadius; ++d) {
            const double c = -(double)d * d / (2.0 * q.sigma_s * q.sigma_s) * 1.4426950408889634;
            b.cs[d] = (float)c;
            b.wrow[d] = (float)std::exp2(c);
        }
        for (int i = 0; i < 2 * kMaxRadius + 2; ++i) {
            const int a = std::min(std::abs(i - radius), radius), c = std::min(std::abs(i - radius - 1), radius);
            b.cep[i] = make_float2(b.cs[a], b.cs[c]);
        }
        b.rfold[0] = 1.0f;
        for (int i = 1; i < 2 * kMaxRadius + 2; ++i) {
            const int d = i - radius;  // window row; wy(d - 1) / wy(d)
            const double e = ((double)d * d - (double)(d - 1) * (d - 1)) / (2.0 * q.sigma_s * q.sigma_s);
            b.rfold[i] = d <= radius ? (float)std::exp(std::min(e, 80.0)) : 1.0f;
        }
        // shared-memory envelope of the generic kernel
        const int narr = p->mode == 0 ? 2 : (p->mode == 1 ? 4 : 8);
        const size_t smem = (size_t)narr * (16 + 2 * radius) * (((64 + 2 * radius) + 3) & ~3) * 4;
        if (brute && smem > 227 * 1024)
            return bail(fail(BLFLS_EUNSUPPORTED, "plan: radius too large for the shared-memory tile"));
    }
    if (grid) {
        // bilateral.cpp:126-134 with sampling = (sigma_s, sigma_r); guide01 in [0, 1]
        GridParams& g = p->grid;
        g.H = H;
        g.W = W;
        g.C = C;
        g.GC = q.guide_channels;
        g.ss = q.sigma_s;
        g.sr = q.sigma_r;
        g.gw = (int)std::floor((W - 1) / q.sigma_s) + 1 + 4;
        g.gh = (int)std::floor((H - 1) / q.sigma_s) + 1 + 4;
        const double gdmax = std::floor(1.0 / q.sigma_r) + 1 + 4 + 1;
        if (gdmax > 1e6 || (double)g.gw * g.gh * gdmax > 2e9)
            return bail(fail(BLFLS_EUNSUPPORTED, "grid backend: grid too large for these sigmas"));
        // a cell holds <= (sigma_s + 2)^2 pixels of 2^39-scaled fixed-point values
        if (q.sigma_s > 4096.0)
            return bail(fail(BLFLS_EUNSUPPORTED, "grid backend: sigma_s > 4096 overflows the splat"));
        g.gdmax = (int)gdmax;
        g.cells = (size_t)g.gw * g.gh * g.gdmax;
        const size_t per_plane = 2 * 4 * g.cells * sizeof(double);  // 2 slots x 4 grids
        int np = (int)std::max<size_t>(1, (size_t)(1u << 30) / per_plane);
        np = std::min(np, q.max_batch * C);
        p->grid_planes = np;
        const size_t n = (size_t)2 * np * g.cells;
        if (cudaMalloc(&g.wgrid, sizeof(double) * n) != cudaSuccess ||
            cudaMalloc(&g.vgrid, sizeof(double) * n) != cudaSuccess ||
            cudaMalloc(&g.blurred, sizeof(double) * 2 * n) != cudaSuccess ||
            cudaMalloc(&g.erange, sizeof(unsigned long long) * 4 * np) != cudaSuccess)
            return bail(fail(BLFLS_ENOMEM, "plan: grid workspace allocation failed"));
    }
    if (q.backend == BLFLS_BACKEND_DT) {
        if (p->Hp > 65535)  // window grid rows
            return bail(fail(BLFLS_EUNSUPPORTED, "dt backend: padded height above 65535"));
        DtParams& d = p->dt;
        d.H = p->Hp;
        d.W = p->Wp;
        d.C = C;
        d.GC = q.guide_channels;
        d.ratio = q.sigma_s / q.sigma_r;
        d.plane = (size_t)p->Hp * p->Wp;
        d.pcplane = (size_t)(p->Hp + 1) * (p->Wp + 1);
        p->dt_iters = q.dt_iterations == 0 ? 3 : q.dt_iterations;
        if (!dt_configure(p->dt_iters, q.sigma_s))
            return bail(fail(BLFLS_EUNSUPPORTED, "dt backend: sigma_s too large for the window tile"));
        const size_t per_plane = 2 * sizeof(double) * (4 * d.plane + d.pcplane);  // 2 slots
        int np = (int)std::max<size_t>(1, (size_t)(1u << 30) / per_plane);
        np = std::min(np, q.max_batch * C);
        p->dt_planes = np;
        const size_t ns = (size_t)2 * np;
        if (cudaMalloc(&d.cth, sizeof(double) * ns * d.plane) != cudaSuccess ||
            cudaMalloc(&d.ctv, sizeof(double) * ns * d.plane) != cudaSuccess ||
            cudaMalloc(&d.x, sizeof(double) * ns * d.plane) != cudaSuccess ||
            cudaMalloc(&d.g01, sizeof(double) * ns * d.plane) != cudaSuccess ||
            cudaMalloc(&d.pc, sizeof(double) * ns * d.pcplane) != cudaSuccess)
            return bail(fail(BLFLS_ENOMEM, "plan: domain-transform workspace allocation failed"));
    }

    // workspace
    p->plane = (size_t)q.height * q.width;
    p->pplane = (size_t)H * W;
    p->img_elems = (size_t)q.max_batch * C * p->plane;
    const size_t pad_elems = (size_t)q.max_batch * C * p->pplane;
    const size_t spec_elems = (size_t)q.max_batch * C * H * p->spitch;
    if (p->pad > 0 &&
        (cudaMalloc(&p->fpad, sizeof(float) * pad_elems) != cudaSuccess ||
         (q.guide_channels &&
          cudaMalloc(&p->gpad, sizeof(float) * q.max_batch * q.guide_channels * p->pplane) != cudaSuccess)))
        return bail(fail(BLFLS_ENOMEM, "plan: padded workspace allocation failed"));
    if (cudaMalloc(&p->buf[0], sizeof(float) * p->img_elems) != cudaSuccess ||
        cudaMalloc(&p->buf[1], sizeof(float) * p->img_elems) != cudaSuccess ||
        cudaMalloc(&p->tx, sizeof(float) * pad_elems) != cudaSuccess ||
        cudaMalloc(&p->ty, sizeof(float) * pad_elems) != cudaSuccess ||
        cudaMalloc(&p->spec, sizeof(float2) * spec_elems) != cudaSuccess ||
        cudaMalloc(&p->lohi, sizeof(uint32_t) * 4 * q.max_batch) != cudaSuccess ||
        cudaMalloc(&p->glohi, sizeof(uint32_t) * 2 * q.max_batch) != cudaSuccess ||
        cudaMalloc(&p->nonfinite, sizeof(unsigned)) != cudaSuccess)
        return bail(fail(BLFLS_ENOMEM, "plan: workspace allocation failed"));
    {
        // one launch per pass over all planes: with the high-radix column /
        // c2r passes the streaming solve beats plane groups that keep each
        // spectrum L2-resident (c5: 7.64 ms per iteration vs 7.8-9.1 for
        // groups of 6..1 planes, r01 B200); BLFLS_SOLVE_GROUP=n (experiment)
        // runs groups of n planes on two streams
        int grp = 0;
        grp = knob("BLFLS_SOLVE_GROUP", grp);
        p->solve_group = grp;
    }
    if (cudaStreamCreateWithFlags(&p->ps2, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&p->ev_join, cudaEventDisableTiming) != cudaSuccess)
        return bail(fail(BLFLS_ECUDA, "plan: stream creation failed"));
    if (cudaStreamCreateWithFlags(&p->ps, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&p->ev_in, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&p->ev_out, cudaEventDisableTiming) != cudaSuccess)
        return bail(fail(BLFLS_ECUDA, "plan: stream creation failed"));
    p->stats.radius = radius;
    *out = p;
    return BLFLS_OK;
}

blfls_status blfls_plan_destroy(blfls_plan_t p)
{
    free_plan(p);
    return BLFLS_OK;
}

namespace {

// Launch the cached graph of the iteration sequence for these pointers
// (capturing and instantiating it on first use).
blfls_status launch_graph(blfls_plan_t p, const float* din, const float* dguide, float* dout, int batch,
                          int iters, cudaStream_t st)
{
    blfls_plan_s::GraphEntry* hit = nullptr;
    for (auto& g : p->graphs)
        if (g.exec && g.in == din && g.guide == dguide && g.out == dout && g.batch == batch &&
            g.iters == iters)
            hit = &g;
    if (!hit) {
        hit = &p->graphs[0];
        for (auto& g : p->graphs)
            if (!g.exec || g.last < hit->last) hit = &g;
        if (hit->exec) {
            cudaGraphExecDestroy(hit->exec);
            hit->exec = nullptr;
        }
        p->launches = 0;
        cudaGraph_t g;
        CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        blfls_status r = enq_run(p, din, dguide, dout, batch, iters, st);
        cudaError_t ce = cudaStreamEndCapture(st, &g);
        if (r) return r;
        if (ce != cudaSuccess) return cuda_fail(ce, "cudaStreamEndCapture");
        ce = cudaGraphInstantiate(&hit->exec, g, 0);
        cudaGraphDestroy(g);
        if (ce != cudaSuccess) return cuda_fail(ce, "cudaGraphInstantiate");
        hit->in = din;
        hit->guide = dguide;
        hit->out = dout;
        hit->batch = batch;
        hit->iters = iters;
        hit->launches = p->launches;
    }
    hit->last = ++p->graph_clock;
    p->stats.kernel_launches = hit->launches;
    CK(cudaGraphLaunch(hit->exec, st));
    return BLFLS_OK;
}

blfls_status ensure_host_slots(blfls_plan_t p)
{
    if (p->s_h2d) return BLFLS_OK;
    CK(cudaStreamCreateWithFlags(&p->s_h2d, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&p->s_d2h, cudaStreamNonBlocking));
    if (!p->nonfinite_acc) {
        CK(cudaMalloc(&p->nonfinite_acc, sizeof(unsigned)));
        CK(cudaMemset(p->nonfinite_acc, 0, sizeof(unsigned)));
    }
    for (auto& sl : p->slot) {
        CK(cudaMalloc(&sl.in, sizeof(float) * p->img_elems));
        CK(cudaMalloc(&sl.out, sizeof(float) * p->img_elems));
        if (p->prm.guide_channels)
            CK(cudaMalloc(&sl.guide, sizeof(float) * p->prm.max_batch * p->prm.guide_channels * p->plane));
        CK(cudaEventCreateWithFlags(&sl.h2d, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&sl.comp, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&sl.d2h, cudaEventDisableTiming));
    }
    return BLFLS_OK;
}

}  // namespace

namespace {

// Images per chunk of an ASYNC host-pointer call: a large host batch is
// streamed through the two staging slots in chunks (images are independent,
// so the results are the same bits), so chunk k + 1's H2D and chunk k - 1's
// D2H overlap chunk k's compute instead of the whole batch's copies
// bracketing the whole batch's compute.  Chunks of >= 64 MB of input, at most
// 8 per call; BLFLS_HOST_CHUNKS=n overrides the count (1: off).
int host_chunk_images(blfls_plan_t p, int batch)
{
    static const int env = knob("BLFLS_HOST_CHUNKS", 0);
    if (batch < 2) return batch;
    const size_t per_image = sizeof(float) * p->plane * (p->prm.channels + p->prm.guide_channels);
    int n = env > 0 ? env : (int)std::min<size_t>(8, (size_t)batch * per_image / (64u << 20));
    n = std::max(1, std::min(n, batch));
    return (batch + n - 1) / n;
}

blfls_status run_impl(blfls_plan_t p, const float* img, const float* guide, int batch, int iters, float* out,
                      void* stream, unsigned flags);

}  // namespace

blfls_status blfls_run(blfls_plan_t p, const float* img, const float* guide, int batch, int iters,
                       float* out, void* stream, unsigned flags)
{
    blfls_status r = validate_batch(p, batch);
    if (r) return r;
    if (iters < 1) return fail(BLFLS_EINVAL, "blf_ls: iters must be >= 1");
    if (!img || !out) return fail(BLFLS_EINVAL, "blf_ls: null image/output");
    if ((p->prm.guide_channels == 0) != (guide == nullptr))
        return fail(BLFLS_EINVAL, "smooth: guidance image shape does not match input");
    if ((r = set_device(p))) return r;
    if ((flags & BLFLS_HOST_PTRS) && (flags & BLFLS_ASYNC) && !(flags & BLFLS_TIME_STAGES)) {
        const int per = host_chunk_images(p, batch);
        if (per < batch) {
            const size_t ci = (size_t)p->prm.channels * p->plane, cg = (size_t)p->prm.guide_channels * p->plane;
            for (int b0 = 0; b0 < batch; b0 += per) {
                const int nb = std::min(per, batch - b0);
                if ((r = run_impl(p, img + b0 * ci, guide ? guide + b0 * cg : nullptr, nb, iters, out + b0 * ci,
                                  stream, flags)))
                    return r;
            }
            return BLFLS_OK;
        }
    }
    return run_impl(p, img, guide, batch, iters, out, stream, flags);
}

namespace {

blfls_status run_impl(blfls_plan_t p, const float* img, const float* guide, int batch, int iters, float* out,
                      void* stream, unsigned flags)
{
    blfls_status r;
    cudaStream_t us = (cudaStream_t)stream;
    const size_t n = (size_t)batch * p->prm.channels * p->plane;
    const size_t ng = guide ? (size_t)batch * p->prm.guide_channels * p->plane : 0;
    const bool host = flags & BLFLS_HOST_PTRS;
    const bool async_host = (flags & BLFLS_ASYNC) && host;
    // ASYNC device calls: ordered on the caller's stream as usual, but the
    // non-finite check is counted on the device and reported by blfls_sync
    // (no host round trip per call)
    const bool async_dev = (flags & BLFLS_ASYNC) && !host;
    const bool async = async_host || async_dev;
    // ASYNC host calls are ordered by blfls_sync, not by the caller's stream:
    // joining it would chain call k+1's H2D behind call k's D2H
    if (!async_host && (r = fork_in(p, us))) return r;
    if (async_dev && !p->nonfinite_acc) {
        CK(cudaMalloc(&p->nonfinite_acc, sizeof(unsigned)));
        CK(cudaMemset(p->nonfinite_acc, 0, sizeof(unsigned)));
    }
    cudaStream_t st = p->ps;
    const float* din = img;
    const float* dguide = guide;
    float* dout = out;
    blfls_plan_s::HostSlot* sl = nullptr;
    if (host) {
        if ((r = ensure_host_slots(p))) return r;
        sl = &p->slot[p->next_slot];
        p->next_slot ^= 1;
        // H2D on its own stream once the slot's previous input was consumed
        if (!async) CK(cudaStreamWaitEvent(p->s_h2d, p->ev_in, 0));
        if (sl->used) CK(cudaStreamWaitEvent(p->s_h2d, sl->comp, 0));
        CK(cudaMemcpyAsync(sl->in, img, sizeof(float) * n, cudaMemcpyHostToDevice, p->s_h2d));
        if (guide)
            CK(cudaMemcpyAsync(sl->guide, guide, sizeof(float) * ng, cudaMemcpyHostToDevice, p->s_h2d));
        CK(cudaEventRecord(sl->h2d, p->s_h2d));
        CK(cudaStreamWaitEvent(st, sl->h2d, 0));
        if (sl->used) CK(cudaStreamWaitEvent(st, sl->d2h, 0));  // slot output drained
        din = sl->in;
        dguide = guide ? sl->guide : nullptr;
        dout = sl->out;
    }
    if (flags & BLFLS_CHECK_FINITE) {
        if (async) {
            // deferred: counted on the device, reported by blfls_sync
            CK(launch_count_nonfinite(din, n, p->nonfinite_acc, p->nsm, st));
            if (dguide) CK(launch_count_nonfinite(dguide, ng, p->nonfinite_acc, p->nsm, st));
        } else {
            if ((r = check_finite(p, din, n, st, "smooth"))) return r;
            if (dguide && (r = check_finite(p, dguide, ng, st, "normalize_to_unit"))) return r;
        }
    }
    p->stats.blf_launches = 0;
    p->time_stages = (flags & BLFLS_TIME_STAGES) != 0;
    const bool use_graph = !(flags & (BLFLS_NO_GRAPH | BLFLS_TIME_STAGES));
    if (use_graph) {
        if ((r = launch_graph(p, din, dguide, dout, batch, iters, st))) return r;
    } else {
        p->launches = 0;
        r = enq_run(p, din, dguide, dout, batch, iters, st);
        p->time_stages = false;
        if (r) return r;
        p->stats.kernel_launches = p->launches;
    }
    const int G = p->mode == 2 ? 1 : p->prm.channels;
    const double taps = p->prm.backend == BLFLS_BACKEND_GRID ? 0.0
                                                            : (double)(2 * p->radius + 1) * (2 * p->radius + 1);
    p->stats.exps = taps * (double)p->pplane * 2.0 * batch * G * iters;
    p->stats.blf_launches = iters;
    if (!host) return join_out(p, us, flags);
    CK(cudaEventRecord(sl->comp, st));
    CK(cudaStreamWaitEvent(p->s_d2h, sl->comp, 0));
    CK(cudaMemcpyAsync(out, sl->out, sizeof(float) * n, cudaMemcpyDeviceToHost, p->s_d2h));
    CK(cudaEventRecord(sl->d2h, p->s_d2h));
    sl->used = true;
    if (async) return BLFLS_OK;
    CK(cudaStreamWaitEvent(us, sl->d2h, 0));
    CK(cudaEventSynchronize(sl->d2h));
    return BLFLS_OK;
}

}  // namespace

blfls_status blfls_sync(blfls_plan_t p)
{
    if (!p) return fail(BLFLS_EINVAL, "null plan");
    blfls_status r;
    if ((r = set_device(p))) return r;
    CK(cudaStreamSynchronize(p->ps));
    if (p->s_h2d) {
        CK(cudaStreamSynchronize(p->s_h2d));
        CK(cudaStreamSynchronize(p->s_d2h));
    }
    if (p->nonfinite_acc) {
        unsigned h = 0;
        CK(cudaMemcpy(&h, p->nonfinite_acc, sizeof(unsigned), cudaMemcpyDeviceToHost));
        CK(cudaMemset(p->nonfinite_acc, 0, sizeof(unsigned)));
        if (h) return fail(BLFLS_ENONFINITE, "smooth: non-finite sample in input image");
    }
    return BLFLS_OK;
}

blfls_status blfls_filter_gradients(blfls_plan_t p, const float* img, const float* guide, int batch,
                                    float* tx, float* ty, void* stream, unsigned flags)
{
    blfls_status r = validate_batch(p, batch);
    if (r) return r;
    if (p->pad) return fail(BLFLS_EUNSUPPORTED, "stage entry points require pad == 0");
    if (r) return r;
    if ((p->prm.guide_channels == 0) != (guide == nullptr))
        return fail(BLFLS_EINVAL, "smooth: guidance image shape does not match input");
    if ((r = set_device(p))) return r;
    cudaStream_t us = (cudaStream_t)stream;
    if ((r = fork_in(p, us))) return r;
    cudaStream_t st = p->ps;
    const size_t n = (size_t)batch * p->prm.channels * p->plane;
    const size_t ng = guide ? (size_t)batch * p->prm.guide_channels * p->plane : 0;
    const bool host = flags & BLFLS_HOST_PTRS;
    const float* din = img;
    const float* dguide = guide;
    float* dtx = tx;
    float* dty = ty;
    if (host) {
        CK(cudaMemcpyAsync(p->buf[0], img, sizeof(float) * n, cudaMemcpyHostToDevice, st));
        din = p->buf[0];
        if (guide) {
            if (!p->guide_dev)
                CK(cudaMalloc(&p->guide_dev,
                              sizeof(float) * p->prm.max_batch * p->prm.guide_channels * p->plane));
            CK(cudaMemcpyAsync(p->guide_dev, guide, sizeof(float) * ng, cudaMemcpyHostToDevice, st));
            dguide = p->guide_dev;
        }
        dtx = p->tx;
        dty = p->ty;
    }
    if (flags & BLFLS_CHECK_FINITE) {
        if ((r = check_finite(p, din, n, st, "smooth"))) return r;
        if (dguide && (r = check_finite(p, dguide, ng, st, "normalize_to_unit"))) return r;
    }
    if (dguide && (r = enq_minmax(p, dguide, (size_t)p->prm.guide_channels * p->plane, batch, p->glohi, st)))
        return r;
    if ((r = enq_minmax(p, din, (size_t)p->prm.channels * p->plane, batch, p->lohi, st))) return r;
    if ((r = enq_blf(p, din, dguide, p->lohi, dtx, dty, batch, 0, p->prm.height, p->prm.height, 1, st)))
        return r;
    if (host) {
        CK(cudaMemcpyAsync(tx, dtx, sizeof(float) * n, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(ty, dty, sizeof(float) * n, cudaMemcpyDeviceToHost, st));
    }
    return join_out(p, us, flags | (host ? BLFLS_SYNC : 0));
}

blfls_status blfls_filter_gradients_rows(blfls_plan_t p, const float* img, const float* guide, int y0,
                                         int y1, float* tx, float* ty, void* stream, unsigned flags)
{
    blfls_status r = validate_batch(p, 1);
    if (r) return r;
    if (p->pad) return fail(BLFLS_EUNSUPPORTED, "stage entry points require pad == 0");
    if (r) return r;
    if (y0 < 0 || y1 > p->prm.height || y0 >= y1) return fail(BLFLS_EINVAL, "rows: bad row range");
    if ((p->prm.guide_channels == 0) != (guide == nullptr))
        return fail(BLFLS_EINVAL, "smooth: guidance image shape does not match input");
    if (flags & BLFLS_HOST_PTRS) return fail(BLFLS_EINVAL, "rows: device pointers only");
    if ((r = set_device(p))) return r;
    cudaStream_t us = (cudaStream_t)stream;
    if ((r = fork_in(p, us))) return r;
    cudaStream_t st = p->ps;
    if (guide && (r = enq_minmax(p, guide, (size_t)p->prm.guide_channels * p->plane, 1, p->glohi, st)))
        return r;
    if ((r = enq_minmax(p, img, (size_t)p->prm.channels * p->plane, 1, p->lohi, st))) return r;
    if ((r = enq_blf(p, img, guide, p->lohi, tx, ty, 1, y0, y1, y1 - y0, 0, st))) return r;
    return join_out(p, us, flags);
}

blfls_status blfls_filter_gradients_rows_peers(blfls_plan_t p, const float* img, const float* guide,
                                               int y0, int y1, float* const* tx_peers,
                                               float* const* ty_peers, int npeers, void* stream,
                                               unsigned flags)
{
    blfls_status r = validate_batch(p, 1);
    if (r) return r;
    if (p->pad) return fail(BLFLS_EUNSUPPORTED, "stage entry points require pad == 0");
    if (p->prm.backend != BLFLS_BACKEND_BRUTE)
        return fail(BLFLS_EUNSUPPORTED, "rows: row bands need the brute-force backend");
    if (npeers < 1 || npeers > kMaxPeers || !tx_peers || !ty_peers)
        return fail(BLFLS_EINVAL, "rows_peers: 1..8 peer buffers");
    if (y0 < 0 || y1 > p->prm.height || y0 >= y1) return fail(BLFLS_EINVAL, "rows: bad row range");
    if ((p->prm.guide_channels == 0) != (guide == nullptr))
        return fail(BLFLS_EINVAL, "smooth: guidance image shape does not match input");
    if (flags & BLFLS_HOST_PTRS) return fail(BLFLS_EINVAL, "rows: device pointers only");
    for (int j = 0; j < npeers; ++j)
        if (!tx_peers[j] || !ty_peers[j]) return fail(BLFLS_EINVAL, "rows_peers: null peer buffer");
    if ((r = set_device(p))) return r;
    cudaStream_t us = (cudaStream_t)stream;
    if ((r = fork_in(p, us))) return r;
    cudaStream_t st = p->ps;
    if (guide && (r = enq_minmax(p, guide, (size_t)p->prm.guide_channels * p->plane, 1, p->glohi, st)))
        return r;
    if ((r = enq_minmax(p, img, (size_t)p->prm.channels * p->plane, 1, p->lohi, st))) return r;
    // the band's targets go straight to every rank's full-height buffers
    BlfParams b = p->blf;
    b.f = img;
    b.guide = guide;
    b.tx = nullptr;
    b.ty = nullptr;
    b.lohi = p->lohi;
    b.glohi = p->glohi;
    b.y0 = y0;
    b.y1 = y1;
    b.out_rows = p->Hp;
    b.normalized_out = 0;
    b.x2_poly = -1;  // the experiment kernels have no peer epilogue
    b.legacy_joint3 = 0;
    b.npeers = npeers;
    for (int j = 0; j < npeers; ++j) {
        b.peer_tx[j] = tx_peers[j];
        b.peer_ty[j] = ty_peers[j];
    }
    CK(launch_grad_blf(b, p->mode, 1, st));
    p->launches++;
    p->stats.blf_launches++;
    return join_out(p, us, flags);
}

blfls_status blfls_solve(blfls_plan_t p, const float* g, const float* tx, const float* ty, int batch,
                         float* u, void* stream, unsigned flags)
{
    blfls_status r = validate_batch(p, batch);
    if (r) return r;
    if ((tx == nullptr) != (ty == nullptr))
        return fail(BLFLS_EINVAL, "lsgrad_solve_fft: target shape does not match image");
    if ((r = set_device(p))) return r;
    cudaStream_t us = (cudaStream_t)stream;
    if ((r = fork_in(p, us))) return r;
    cudaStream_t st = p->ps;
    const size_t n = (size_t)batch * p->prm.channels * p->plane;
    const bool host = flags & BLFLS_HOST_PTRS;
    const float* dg = g;
    const float* dtx = tx;
    const float* dty = ty;
    float* du = u;
    if (host) {
        // with padding the inputs are staged unpadded and reflect-padded into
        // fpad / tx / ty below.  The staging buffers are plan scratch that
        // only p->ps touches (never the ASYNC host slots, whose copies run on
        // s_h2d / s_d2h and may still be in flight): buf[0] and buf[1] hold
        // >= n floats (padded image size), the spectrum holds >= 2 n floats and
        // is first written by the solve's row pass, after the padding kernels
        // consumed the staged targets (stream order on p->ps).
        float* sg = p->buf[0];
        float* stx = p->pad ? p->buf[1] : p->tx;
        float* sty = p->pad ? reinterpret_cast<float*>(p->spec) : p->ty;
        CK(cudaMemcpyAsync(sg, g, sizeof(float) * n, cudaMemcpyHostToDevice, st));
        dg = sg;
        if (tx) {
            CK(cudaMemcpyAsync(stx, tx, sizeof(float) * n, cudaMemcpyHostToDevice, st));
            CK(cudaMemcpyAsync(sty, ty, sizeof(float) * n, cudaMemcpyHostToDevice, st));
            dtx = stx;
            dty = sty;
        }
        du = p->buf[1];
    }
    if (flags & BLFLS_CHECK_FINITE) {
        if ((r = check_finite(p, dg, n, st, "lsgrad_solve_fft"))) return r;
        if (dtx && (r = check_finite(p, dtx, n, st, "lsgrad_solve_fft"))) return r;
        if (dty && (r = check_finite(p, dty, n, st, "lsgrad_solve_fft"))) return r;
    }
    if (p->pad) {
        // solver.cpp:97-99: the image and the targets are reflect-padded as
        // plain rasters; the solve crops (solver.cpp:123)
        const size_t planes = (size_t)batch * p->prm.channels;
        CK(launch_reflect_pad(dg, p->fpad, p->prm.height, p->prm.width, p->pad, planes, p->nsm, st));
        dg = p->fpad;
        if (dtx) {
            CK(launch_reflect_pad(dtx, p->tx, p->prm.height, p->prm.width, p->pad, planes, p->nsm, st));
            CK(launch_reflect_pad(dty, p->ty, p->prm.height, p->prm.width, p->pad, planes, p->nsm, st));
            dtx = p->tx;
            dty = p->ty;
        }
    }
    if ((r = enq_solve(p, dg, dtx, dty, du, nullptr, batch, st))) return r;
    if (host) CK(cudaMemcpyAsync(u, du, sizeof(float) * n, cudaMemcpyDeviceToHost, st));
    return join_out(p, us, flags | (host ? BLFLS_SYNC : 0));
}

static blfls_status fft_entry(blfls_plan_t p, const float* in, int batch, float* outp, void* stream,
                              unsigned flags, bool forward)
{
    blfls_status r = validate_batch(p, batch);
    if (r) return r;
    if (p->pad) return fail(BLFLS_EUNSUPPORTED, "stage entry points require pad == 0");
    if (r) return r;
    if ((r = set_device(p))) return r;
    cudaStream_t us = (cudaStream_t)stream;
    if ((r = fork_in(p, us))) return r;
    cudaStream_t st = p->ps;
    const int planes = batch * p->prm.channels;
    const size_t nreal = (size_t)planes * p->plane;
    const size_t nspec = (size_t)planes * p->prm.height * p->wc;  // packed, caller layout
    const bool host = flags & BLFLS_HOST_PTRS;
    SolveParams s = solve_params(p);
    // caller spectra are packed (pitch wc); the plan spectrum has pitch spitch
    if (forward) {
        const float* din = in;
        if (host) {
            CK(cudaMemcpyAsync(p->buf[0], in, sizeof(float) * nreal, cudaMemcpyHostToDevice, st));
            din = p->buf[0];
        }
        s.f = din;
        s.mode = 1;
        CK(launch_row_r2c(s, p->rowf.g, planes, p->odd, st));
        CK(launch_col(s, p->colf.g, planes, st));
        CK(cudaMemcpy2DAsync(outp, sizeof(float2) * p->wc, p->spec, sizeof(float2) * p->spitch,
                             sizeof(float2) * p->wc, (size_t)planes * p->prm.height,
                             host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, st));
    } else {
        CK(cudaMemcpy2DAsync(p->spec, sizeof(float2) * p->spitch, in, sizeof(float2) * p->wc,
                             sizeof(float2) * p->wc, (size_t)planes * p->prm.height,
                             host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, st));
        float* dout = host ? p->buf[1] : outp;
        s.out = dout;
        s.mode = 2;
        CK(launch_col(s, p->colf.g, planes, st));
        CK(launch_row_c2r(s, p->rowf.g, planes, p->odd, st));
        if (host) CK(cudaMemcpyAsync(outp, dout, sizeof(float) * nreal, cudaMemcpyDeviceToHost, st));
    }
    (void)nspec;
    return join_out(p, us, flags | (host ? BLFLS_SYNC : 0));
}

blfls_status blfls_rfft2(blfls_plan_t p, const float* x, int batch, float* spec, void* stream,
                         unsigned flags)
{
    return fft_entry(p, x, batch, spec, stream, flags, true);
}

blfls_status blfls_irfft2(blfls_plan_t p, const float* spec, int batch, float* out, void* stream,
                          unsigned flags)
{
    return fft_entry(p, spec, batch, out, stream, flags, false);
}

blfls_status blfls_generate(int height, int width, int n_planes, const uint64_t* seeds, int n_sites,
                            double noise_sigma, double p_sp, float* out, void* stream, int device)
{
    if (height < 1 || width < 1 || n_planes < 1 || n_sites < 1 || n_sites > 1024 || !seeds || !out)
        return fail(BLFLS_EINVAL, "generate: bad arguments");
    CK(cudaSetDevice(device));
    cudaStream_t st = (cudaStream_t)stream;
    struct Seeds {  // released on every exit path (stream-ordered)
        cudaStream_t st;
        uint64_t* d = nullptr;
        ~Seeds()
        {
            if (d) cudaFreeAsync(d, st);
        }
    } ds{st};
    CK(cudaMallocAsync(&ds.d, sizeof(uint64_t) * n_planes, st));
    CK(cudaMemcpyAsync(ds.d, seeds, sizeof(uint64_t) * n_planes, cudaMemcpyHostToDevice, st));
    CK(launch_generate(height, width, n_planes, ds.d, n_sites, noise_sigma, p_sp, out, st));
    CK(cudaStreamSynchronize(st));
    return BLFLS_OK;
}

blfls_status blfls_forward_gradients(const float* img, int planes, int height, int width, float* gx,
                                     float* gy, int device, void* stream, unsigned flags)
{
    if (!img || !gx || !gy || planes < 1 || height < 1 || width < 1)
        return fail(BLFLS_EINVAL, "forward_gradients: bad arguments");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(BLFLS_ECUDA, "no CUDA device (this library has no CPU fallback)");
    if (device < 0 || device >= ndev) return fail(BLFLS_EINVAL, "forward_gradients: bad device ordinal");
    CK(cudaSetDevice(device));
    cudaDeviceProp prop{};
    CK(cudaGetDeviceProperties(&prop, device));
    cudaStream_t st = (cudaStream_t)stream;
    const size_t n = (size_t)planes * height * width;
    struct Tmp {
        cudaStream_t st;
        float* v[3] = {nullptr, nullptr, nullptr};
        ~Tmp()
        {
            for (float* q : v)
                if (q) cudaFreeAsync(q, st);
        }
    } t{st};
    const float* src = img;
    float *ox = gx, *oy = gy;
    const bool host = flags & BLFLS_HOST_PTRS;
    if (host) {
        for (float*& q : t.v) CK(cudaMallocAsync(&q, sizeof(float) * n, st));
        CK(cudaMemcpyAsync(t.v[0], img, sizeof(float) * n, cudaMemcpyHostToDevice, st));
        src = t.v[0];
        ox = t.v[1];
        oy = t.v[2];
    }
    CK(launch_forward_gradients(src, ox, oy, planes, height, width, prop.multiProcessorCount, st));
    if (host) {
        CK(cudaMemcpyAsync(gx, ox, sizeof(float) * n, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(gy, oy, sizeof(float) * n, cudaMemcpyDeviceToHost, st));
    }
    if (host || (flags & BLFLS_SYNC)) CK(cudaStreamSynchronize(st));
    return BLFLS_OK;
}

blfls_status blfls_blf_brute(const float* src, int cs, const float* guide, int cg, int height,
                             int width, int batch, int radius, double sigma_s, double sigma_r,
                             float* out, int device, void* stream, unsigned flags)
{
    // bilateral.cpp:12-24 (validate_params / validate_pair)
    if (!(sigma_s > 0.0) || !std::isfinite(sigma_s) || !(sigma_r > 0.0) || !std::isfinite(sigma_r))
        return fail(BLFLS_EINVAL, "bilateral: sigma_s and sigma_r must be positive and finite");
    if (!src || !out || height < 1 || width < 1 || batch < 1 || (cs != 1 && cs != 3))
        return fail(BLFLS_EINVAL, "blf_brute: bad arguments");
    if (!guide) cg = cs;
    if (cg != 1 && cg != cs)
        return fail(BLFLS_EINVAL, "bilateral: guide channels must be 1 or match src");
    const int R = radius < 0 ? (int)std::ceil(3.0 * sigma_s) : radius;
    if (R > 4096 || blf_plain_smem(cg, cs, R) > 227 * 1024)
        return fail(BLFLS_EUNSUPPORTED, "blf_brute: radius " + std::to_string(R) +
                                            " exceeds the shared-memory tile");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(BLFLS_ECUDA, "no CUDA device (this library has no CPU fallback)");
    if (device < 0 || device >= ndev) return fail(BLFLS_EINVAL, "blf_brute: bad device ordinal");
    CK(cudaSetDevice(device));
    cudaStream_t st = (cudaStream_t)stream;
    const size_t ns = (size_t)batch * cs * height * width, ng = (size_t)batch * cg * height * width;
    const bool host = flags & BLFLS_HOST_PTRS;
    std::vector<float> tab(2 * (R + 1));
    for (int d = 0; d <= R; ++d) {  // bilateral.cpp:42-47 in the exp2 domain
        const double c = -(double)d * d / (2.0 * sigma_s * sigma_s) * 1.4426950408889634;
        tab[d] = (float)c;
        tab[R + 1 + d] = (float)std::exp2(c);
    }
    struct Tmp {  // stream-ordered temporaries, released on every exit path
        cudaStream_t st;
        float* tab = nullptr;
        float* s = nullptr;
        float* g = nullptr;
        float* o = nullptr;
        unsigned* bad = nullptr;
        ~Tmp()
        {
            for (void* q : {(void*)tab, (void*)s, (void*)g, (void*)o, (void*)bad})
                if (q) cudaFreeAsync(q, st);
        }
    } t{st};
    CK(cudaMallocAsync(&t.tab, sizeof(float) * tab.size(), st));
    CK(cudaMemcpyAsync(t.tab, tab.data(), sizeof(float) * tab.size(), cudaMemcpyHostToDevice, st));
    const float* ds = src;
    const float* dg = guide ? guide : src;
    float* dout = out;
    if (host) {
        CK(cudaMallocAsync(&t.s, sizeof(float) * ns, st));
        CK(cudaMallocAsync(&t.o, sizeof(float) * ns, st));
        CK(cudaMemcpyAsync(t.s, src, sizeof(float) * ns, cudaMemcpyHostToDevice, st));
        ds = t.s;
        dg = t.s;
        if (guide) {
            CK(cudaMallocAsync(&t.g, sizeof(float) * ng, st));
            CK(cudaMemcpyAsync(t.g, guide, sizeof(float) * ng, cudaMemcpyHostToDevice, st));
            dg = t.g;
        }
        dout = t.o;
    }
    if (flags & BLFLS_CHECK_FINITE) {  // bilateral.cpp:31-32 (require_finite)
        CK(cudaMallocAsync(&t.bad, sizeof(unsigned), st));
        CK(cudaMemsetAsync(t.bad, 0, sizeof(unsigned), st));
        cudaDeviceProp prop{};
        CK(cudaGetDeviceProperties(&prop, device));
        CK(launch_count_nonfinite(ds, ns, t.bad, prop.multiProcessorCount, st));
        if (guide) CK(launch_count_nonfinite(dg, ng, t.bad, prop.multiProcessorCount, st));
        unsigned nbad = 0;
        CK(cudaMemcpyAsync(&nbad, t.bad, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (nbad) return fail(BLFLS_ENONFINITE, "blf_brute: image contains non-finite values");
    }
    CK(launch_blf_plain(ds, cs, dg, cg, dout, batch, height, width, R, sigma_s, sigma_r, t.tab, st));
    if (host) CK(cudaMemcpyAsync(out, t.o, sizeof(float) * ns, cudaMemcpyDeviceToHost, st));
    if (host || (flags & BLFLS_SYNC)) CK(cudaStreamSynchronize(st));
    return BLFLS_OK;
}

blfls_status blfls_gaussian_blur(const float* in, int channels, int height, int width, double sigma,
                                 float* out, int device, void* stream, unsigned flags)
{
    // image.cpp:116-117
    if (!(sigma > 0.0) || !std::isfinite(sigma))
        return fail(BLFLS_EINVAL, "gaussian_blur: sigma must be positive and finite");
    if (!in || !out || channels < 1 || height < 1 || width < 1 || in == out)
        return fail(BLFLS_EINVAL, "gaussian_blur: bad arguments");
    if ((size_t)std::ceil(3.0 * sigma) > (size_t)1 << 20)
        return fail(BLFLS_EUNSUPPORTED, "gaussian_blur: sigma too large");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(BLFLS_ECUDA, "no CUDA device (this library has no CPU fallback)");
    if (device < 0 || device >= ndev) return fail(BLFLS_EINVAL, "gaussian_blur: bad device ordinal");
    CK(cudaSetDevice(device));
    cudaDeviceProp prop{};
    CK(cudaGetDeviceProperties(&prop, device));
    cudaStream_t st = (cudaStream_t)stream;
    const std::vector<double> k = gaussian_weights(sigma);
    const int r = (int)(k.size() / 2);
    const size_t n = (size_t)channels * height * width;
    const bool host = flags & BLFLS_HOST_PTRS;
    // temporaries are stream-ordered and released on every exit path
    struct Tmp {
        cudaStream_t st;
        double* dk = nullptr;
        double* tmp = nullptr;
        float* din = nullptr;
        float* dout = nullptr;
        ~Tmp()
        {
            for (void* q : {(void*)dk, (void*)tmp, (void*)din, (void*)dout})
                if (q) cudaFreeAsync(q, st);
        }
    } t{st};
    double*& dk = t.dk;
    double*& tmp = t.tmp;
    float*& din = t.din;
    float*& dout = t.dout;
    CK(cudaMallocAsync(&dk, sizeof(double) * k.size(), st));
    CK(cudaMallocAsync(&tmp, sizeof(double) * n, st));
    CK(cudaMemcpyAsync(dk, k.data(), sizeof(double) * k.size(), cudaMemcpyHostToDevice, st));
    const float* src = in;
    float* dst = out;
    if (host) {
        CK(cudaMallocAsync(&din, sizeof(float) * n, st));
        CK(cudaMallocAsync(&dout, sizeof(float) * n, st));
        CK(cudaMemcpyAsync(din, in, sizeof(float) * n, cudaMemcpyHostToDevice, st));
        src = din;
        dst = dout;
    }
    CK(launch_gaussian_blur(src, dst, tmp, dk, r, channels, height, width,
                            prop.multiProcessorCount, st));
    if (host) CK(cudaMemcpyAsync(out, dout, sizeof(float) * n, cudaMemcpyDeviceToHost, st));
    if (host || (flags & BLFLS_SYNC)) CK(cudaStreamSynchronize(st));
    return BLFLS_OK;
}

blfls_status blfls_last_stats(blfls_plan_t p, blfls_stats* s)
{
    if (!p || !s) return fail(BLFLS_EINVAL, "null argument");
    *s = p->stats;
    return BLFLS_OK;
}

blfls_status blfls_stage_times(blfls_plan_t p, double* ms_sum5, long long* launches5)
{
    if (!p || !ms_sum5) return fail(BLFLS_EINVAL, "null argument");
    blfls_status r;
    if ((r = set_device(p))) return r;
    for (int i = 0; i < 5; ++i) {
        ms_sum5[i] = 0.0;
        if (launches5) launches5[i] = 0;
    }
    for (auto& e : p->timing) {
        CK(cudaEventSynchronize(e.b));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, e.a, e.b));
        ms_sum5[e.stage] += ms;
        if (launches5) launches5[e.stage]++;
        cudaEventDestroy(e.a);
        cudaEventDestroy(e.b);
    }
    p->timing.clear();
    return BLFLS_OK;
}

blfls_status blfls_debug_ranges(blfls_plan_t p, float* out)
{
    if (!p || !out) return fail(BLFLS_EINVAL, "null argument");
    blfls_status r;
    if ((r = set_device(p))) return r;
    CK(cudaStreamSynchronize(p->ps));
    std::vector<uint32_t> h(4 * (size_t)p->prm.max_batch);
    CK(cudaMemcpy(h.data(), p->lohi, sizeof(uint32_t) * h.size(), cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < h.size(); ++i) out[i] = ordered_to_float(h[i]);
    return BLFLS_OK;
}

blfls_status blfls_mufu_peak(int device, double* ex2_per_second, double* sm_clock_hz)
{
    if (!ex2_per_second) return fail(BLFLS_EINVAL, "null argument");
    CK(cudaSetDevice(device));
    double rate = 0.0, clk = 0.0;
    cudaError_t e = measure_mufu(device, &rate, &clk);
    if (e != cudaSuccess) return cuda_fail(e, "measure_mufu");
    *ex2_per_second = rate;
    if (sm_clock_hz) *sm_clock_hz = clk;
    return BLFLS_OK;
}

}  // extern "C"
