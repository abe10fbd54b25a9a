// multi.cu -- one host process driving several GPUs through the C ABI
// (blfls_multi_*, declared in blfls.h).  The decompositions of SURVEY.md
// 8(e), built only from the single-device entry points:
//
//   batch: contiguous shards of the batch, one plan + stream + host thread per
//          device entry, each running blfls_run(HOST_PTRS | ASYNC) (its H2D /
//          compute / D2H pipeline, capi.cu run_impl) and blfls_sync.  Images
//          are independent units of epls::smooth (pipelines.cpp:57-94), so no
//          data crosses devices.
//   band : one image in row bands.  Per iteration every entry filters its band
//          (blfls_filter_gradients_rows_peers: the filter kernel stores each
//          target into the full-height tx / ty of EVERY entry, NVLink peer
//          stores between GPUs), then every entry runs the full FFT solve
//          (blfls_solve) redundantly, so it holds the whole next iterate and
//          the next iteration needs no halo exchange.  Cross-device ordering
//          by events only: filter k waits for every entry's solve k - 1
//          (nobody still reads the target buffers it overwrites), solve k
//          waits for every entry's filter k (all bands landed).  No kernel
//          waits on another kernel.
#include <algorithm>
#include <cmath>
#include <string>
#include <thread>
#include <vector>

#include "blfls_internal.cuh"

using blfls::report;

namespace {

#define MCK(expr)                                                                        \
    do {                                                                                 \
        cudaError_t e_ = (expr);                                                         \
        if (e_ != cudaSuccess)                                                           \
            return report(e_ == cudaErrorMemoryAllocation ? BLFLS_ENOMEM : BLFLS_ECUDA,  \
                          std::string(#expr ": ") + cudaGetErrorString(e_));             \
    } while (0)

// [i0, i1) of entry r among n (balanced contiguous split, multigpu.batch_shard)
void shard(int total, int n, int r, int* i0, int* i1)
{
    const int base = total / n, extra = total % n;
    *i0 = r * base + std::min(r, extra);
    *i1 = *i0 + base + (r < extra ? 1 : 0);
}

// row bands of (almost) equal height (multigpu.band_rows)
void band(int height, int n, int r, int* y0, int* y1)
{
    const int per = (height + n - 1) / n;
    bool empty = false;
    for (int b = 0; b < n; ++b)
        if (std::min(b * per, height) >= std::min(std::min(b * per, height) + per, height)) empty = true;
    if (!empty) {
        *y0 = std::min(r * per, height);
        *y1 = std::min(*y0 + per, height);
    } else {
        shard(height, n, r, y0, y1);
    }
}

struct Entry {
    int device = 0;
    blfls_plan_t plan = nullptr;
    // band mode
    cudaStream_t st = nullptr;
    cudaEvent_t ev_filter = nullptr, ev_solve = nullptr;
    float* f[2] = {nullptr, nullptr};
    float* guide = nullptr;
    float* tx = nullptr;
    float* ty = nullptr;
};

}  // namespace

struct blfls_multi_s {
    blfls_params prm{};
    int mode = BLFLS_MULTI_BATCH;
    std::vector<Entry> e;
    size_t plane = 0;
};

namespace {

void release(blfls_multi_s* m)
{
    for (Entry& x : m->e) {
        if (x.st || x.f[0]) cudaSetDevice(x.device);
        if (x.st) cudaStreamSynchronize(x.st);
        for (float* p : {x.f[0], x.f[1], x.guide, x.tx, x.ty})
            if (p) cudaFree(p);
        if (x.ev_filter) cudaEventDestroy(x.ev_filter);
        if (x.ev_solve) cudaEventDestroy(x.ev_solve);
        if (x.st) cudaStreamDestroy(x.st);
        if (x.plan) blfls_plan_destroy(x.plan);
    }
    delete m;
}

blfls_status setup_band(blfls_multi_s* m)
{
    const blfls_params& q = m->prm;
    const size_t n = (size_t)q.channels * m->plane, ng = (size_t)q.guide_channels * m->plane;
    for (Entry& x : m->e) {
        MCK(cudaSetDevice(x.device));
        MCK(cudaStreamCreateWithFlags(&x.st, cudaStreamNonBlocking));
        MCK(cudaEventCreateWithFlags(&x.ev_filter, cudaEventDisableTiming));
        MCK(cudaEventCreateWithFlags(&x.ev_solve, cudaEventDisableTiming));
        MCK(cudaMalloc(&x.f[0], sizeof(float) * n));
        MCK(cudaMalloc(&x.f[1], sizeof(float) * n));
        MCK(cudaMalloc(&x.tx, sizeof(float) * n));
        MCK(cudaMalloc(&x.ty, sizeof(float) * n));
        if (ng) MCK(cudaMalloc(&x.guide, sizeof(float) * ng));
    }
    // every entry stores into every other entry's target buffers
    for (const Entry& a : m->e)
        for (const Entry& b : m->e) {
            if (a.device == b.device) continue;
            int ok = 0;
            MCK(cudaDeviceCanAccessPeer(&ok, a.device, b.device));
            if (!ok)
                return report(BLFLS_EUNSUPPORTED, "multi band: no peer access from device " +
                                                      std::to_string(a.device) + " to " + std::to_string(b.device));
            MCK(cudaSetDevice(a.device));
            const cudaError_t pe = cudaDeviceEnablePeerAccess(b.device, 0);
            if (pe == cudaErrorPeerAccessAlreadyEnabled)
                (void)cudaGetLastError();
            else if (pe != cudaSuccess)
                return report(BLFLS_ECUDA, std::string("cudaDeviceEnablePeerAccess: ") + cudaGetErrorString(pe));
        }
    return BLFLS_OK;
}

bool any_nonfinite(const float* x, size_t n)
{
    for (size_t i = 0; i < n; ++i)
        if (!std::isfinite(x[i])) return true;
    return false;
}

blfls_status run_band(blfls_multi_s* m, const float* img, const float* guide, int iters, float* out,
                      unsigned flags)
{
    const blfls_params& q = m->prm;
    const int n = (int)m->e.size();
    const size_t ni = (size_t)q.channels * m->plane, ng = (size_t)q.guide_channels * m->plane;
    if (flags & BLFLS_CHECK_FINITE) {
        if (any_nonfinite(img, ni)) return report(BLFLS_ENONFINITE, "smooth: non-finite sample in input");
        if (guide && any_nonfinite(guide, ng))
            return report(BLFLS_ENONFINITE, "normalize_to_unit: non-finite sample in input");
    }
    std::vector<float*> txp(n), typ(n);
    for (int r = 0; r < n; ++r) {
        txp[r] = m->e[r].tx;
        typ[r] = m->e[r].ty;
    }
    for (Entry& x : m->e) {
        MCK(cudaSetDevice(x.device));
        MCK(cudaMemcpyAsync(x.f[0], img, sizeof(float) * ni, cudaMemcpyHostToDevice, x.st));
        if (guide) MCK(cudaMemcpyAsync(x.guide, guide, sizeof(float) * ng, cudaMemcpyHostToDevice, x.st));
    }
    int cur = 0;
    blfls_status r;
    for (int k = 0; k < iters; ++k) {
        for (int i = 0; i < n; ++i) {
            Entry& x = m->e[i];
            MCK(cudaSetDevice(x.device));
            if (k > 0)
                for (const Entry& o : m->e) MCK(cudaStreamWaitEvent(x.st, o.ev_solve, 0));
            int y0, y1;
            band(q.height, n, i, &y0, &y1);
            if ((r = blfls_filter_gradients_rows_peers(x.plan, x.f[cur], guide ? x.guide : nullptr, y0, y1,
                                                       txp.data(), typ.data(), n, x.st, BLFLS_DEVICE_PTRS)))
                return r;
            MCK(cudaSetDevice(x.device));
            MCK(cudaEventRecord(x.ev_filter, x.st));
        }
        for (Entry& x : m->e) {
            MCK(cudaSetDevice(x.device));
            for (const Entry& o : m->e) MCK(cudaStreamWaitEvent(x.st, o.ev_filter, 0));
            if ((r = blfls_solve(x.plan, x.f[cur], x.tx, x.ty, 1, x.f[cur ^ 1], x.st, BLFLS_DEVICE_PTRS)))
                return r;
            MCK(cudaSetDevice(x.device));
            MCK(cudaEventRecord(x.ev_solve, x.st));
        }
        cur ^= 1;
    }
    Entry& x0 = m->e[0];
    MCK(cudaSetDevice(x0.device));
    MCK(cudaMemcpyAsync(out, x0.f[cur], sizeof(float) * ni, cudaMemcpyDeviceToHost, x0.st));
    for (Entry& x : m->e) {
        MCK(cudaSetDevice(x.device));
        MCK(cudaStreamSynchronize(x.st));
    }
    return BLFLS_OK;
}

blfls_status run_batch(blfls_multi_s* m, const float* img, const float* guide, int batch, int iters,
                       float* out, unsigned flags)
{
    const blfls_params& q = m->prm;
    const int n = (int)m->e.size();
    const size_t ci = (size_t)q.channels * m->plane, cg = (size_t)q.guide_channels * m->plane;
    std::vector<blfls_status> st(n, BLFLS_OK);
    std::vector<std::string> msg(n);
    auto work = [&](int r) {
        int i0, i1;
        shard(batch, n, r, &i0, &i1);
        if (i1 <= i0) return;
        Entry& x = m->e[r];
        const unsigned fl = (flags & BLFLS_CHECK_FINITE) | BLFLS_HOST_PTRS | BLFLS_ASYNC;
        blfls_status s = blfls_run(x.plan, img + i0 * ci, guide ? guide + i0 * cg : nullptr, i1 - i0, iters,
                                   out + i0 * ci, nullptr, fl);
        const blfls_status s2 = blfls_sync(x.plan);
        if (!s) s = s2;
        st[r] = s;
        if (s) msg[r] = blfls_last_error();
    };
    if (n == 1) {
        work(0);
    } else {
        std::vector<std::thread> th;
        th.reserve(n);
        for (int r = 0; r < n; ++r) th.emplace_back(work, r);
        for (auto& t : th) t.join();
    }
    for (int r = 0; r < n; ++r)
        if (st[r]) return report(st[r], "device entry " + std::to_string(r) + ": " + msg[r]);
    return BLFLS_OK;
}

}  // namespace

extern "C" {

blfls_status blfls_multi_create(const blfls_params* params, const int* devices, int ndevices, int mode,
                                blfls_multi_t* out)
{
    if (!params || !devices || !out) return report(BLFLS_EINVAL, "null argument");
    *out = nullptr;
    if (ndevices < 1 || ndevices > blfls::kMaxPeers) return report(BLFLS_EINVAL, "multi: 1..8 device entries");
    if (mode != BLFLS_MULTI_BATCH && mode != BLFLS_MULTI_BAND) return report(BLFLS_EINVAL, "multi: bad mode");
    if (params->max_batch < 1) return report(BLFLS_EINVAL, "multi: max_batch must be >= 1");
    if (mode == BLFLS_MULTI_BAND) {
        if (params->max_batch != 1) return report(BLFLS_EINVAL, "multi band: one image (max_batch 1)");
        if (params->pad != 0 || params->backend != BLFLS_BACKEND_BRUTE)
            return report(BLFLS_EUNSUPPORTED, "multi band: brute-force backend, pad 0");
        if (params->height < ndevices) return report(BLFLS_EINVAL, "multi band: fewer rows than bands");
    }
    auto* m = new blfls_multi_s;
    m->prm = *params;
    m->mode = mode;
    m->plane = (size_t)params->height * params->width;
    m->e.resize(ndevices);
    for (int i = 0; i < ndevices; ++i) {
        blfls_params q = *params;
        q.device = devices[i];
        q.max_batch = mode == BLFLS_MULTI_BAND ? 1 : (params->max_batch + ndevices - 1) / ndevices;
        m->e[i].device = devices[i];
        const blfls_status s = blfls_plan_create(&q, &m->e[i].plan);
        if (s) {
            const std::string msg = blfls_last_error();
            release(m);
            return report(s, msg);
        }
    }
    if (mode == BLFLS_MULTI_BAND) {
        const blfls_status s = setup_band(m);
        if (s) {
            const std::string msg = blfls_last_error();
            release(m);
            return report(s, msg);
        }
    }
    *out = m;
    return BLFLS_OK;
}

blfls_status blfls_multi_run(blfls_multi_t m, const float* img, const float* guide, int batch, int iters,
                             float* out, unsigned flags)
{
    if (!m) return report(BLFLS_EINVAL, "null multi");
    if (!img || !out) return report(BLFLS_EINVAL, "blf_ls: null image/output");
    if (iters < 1) return report(BLFLS_EINVAL, "blf_ls: iters must be >= 1");
    if (batch < 1 || batch > m->prm.max_batch) return report(BLFLS_EINVAL, "batch outside [1, max_batch]");
    if ((m->prm.guide_channels == 0) != (guide == nullptr))
        return report(BLFLS_EINVAL, "smooth: guidance image shape does not match input");
    if (!(flags & BLFLS_HOST_PTRS)) return report(BLFLS_EINVAL, "multi: host pointers (BLFLS_HOST_PTRS)");
    if (m->mode == BLFLS_MULTI_BAND) return run_band(m, img, guide, iters, out, flags);
    return run_batch(m, img, guide, batch, iters, out, flags);
}

blfls_status blfls_multi_destroy(blfls_multi_t m)
{
    if (m) release(m);
    return BLFLS_OK;
}

blfls_status blfls_host_alloc(size_t bytes, void** ptr)
{
    if (!ptr) return report(BLFLS_EINVAL, "null argument");
    *ptr = nullptr;
    if (bytes == 0) return BLFLS_OK;
    MCK(cudaHostAlloc(ptr, bytes, cudaHostAllocPortable));
    return BLFLS_OK;
}

blfls_status blfls_host_free(void* ptr)
{
    if (ptr) MCK(cudaFreeHost(ptr));
    return BLFLS_OK;
}

}  // extern "C"
