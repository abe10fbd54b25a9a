// blfls_bench.cpp -- end-to-end throughput of the C++ host API (blfls.hpp):
// the reference's call pattern (one spec, repeated smooth() cascades,
// pipelines.cpp:111-115) on float host buffers through a reused blfls::Plan
// (pinned staging, ASYNC: H2D / compute / D2H overlapped across calls), or
// through blfls::MultiPlan when --devices lists several entries.
//
//   blfls_bench --height 2048 --width 2048 --channels 3 --guide-channels 1
//               --batch 64 --radius 7 --sigma-s 7 --sigma-r 0.1 --lambda 1000
//               --iters 3 --steps 5 --warmup 2 [--devices 0,1,...]
//
// Inputs: the BASELINE generator on the device (blfls_generate), copied once
// into pinned host memory.  Timed: K consecutive calls, each copying the batch
// H2D, smoothing it and copying the result D2H, with the non-finite check;
// host wall clock from the first submit to the last sync.  Prints one JSON
// line (MP/s = H W batch iters / seconds per step).
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "blfls/blfls.hpp"

namespace {

struct Args {
    int height = 2048, width = 2048, channels = 3, guide_channels = 1, batch = 64, radius = 7;
    double sigma_s = 7.0, sigma_r = 0.1, lambda = 1000.0;
    int iters = 3, steps = 5, warmup = 2, seed_base = 5000;
    std::vector<int> devices{0};
};

Args parse(int argc, char** argv)
{
    Args a;
    for (int i = 1; i + 1 < argc; i += 2) {
        const std::string k = argv[i];
        const char* v = argv[i + 1];
        if (k == "--height") a.height = std::atoi(v);
        else if (k == "--width") a.width = std::atoi(v);
        else if (k == "--channels") a.channels = std::atoi(v);
        else if (k == "--guide-channels") a.guide_channels = std::atoi(v);
        else if (k == "--batch") a.batch = std::atoi(v);
        else if (k == "--radius") a.radius = std::atoi(v);
        else if (k == "--sigma-s") a.sigma_s = std::atof(v);
        else if (k == "--sigma-r") a.sigma_r = std::atof(v);
        else if (k == "--lambda") a.lambda = std::atof(v);
        else if (k == "--iters") a.iters = std::atoi(v);
        else if (k == "--steps") a.steps = std::atoi(v);
        else if (k == "--warmup") a.warmup = std::atoi(v);
        else if (k == "--seed-base") a.seed_base = std::atoi(v);
        else if (k == "--devices") {
            a.devices.clear();
            for (const char* p = v; *p;) {
                a.devices.push_back(std::atoi(p));
                while (*p && *p != ',') ++p;
                if (*p == ',') ++p;
            }
        } else {
            std::fprintf(stderr, "unknown option %s\n", k.c_str());
            std::exit(2);
        }
    }
    return a;
}

// planes of the BASELINE generator into pinned host memory
void generate(float* host, int h, int w, const std::vector<uint64_t>& seeds, int device)
{
    const size_t plane = (size_t)h * w;
    const size_t chunk = 16;  // planes per device round trip
    float* d = nullptr;
    cudaSetDevice(device);
    if (cudaMalloc(&d, sizeof(float) * plane * chunk) != cudaSuccess) throw std::runtime_error("cudaMalloc");
    for (size_t p0 = 0; p0 < seeds.size(); p0 += chunk) {
        const int n = (int)std::min(chunk, seeds.size() - p0);
        blfls::detail::check(blfls_generate(h, w, n, seeds.data() + p0, 12, 0.03, 0.0, d, nullptr, device));
        cudaMemcpy(host + p0 * plane, d, sizeof(float) * plane * n, cudaMemcpyDeviceToHost);
    }
    cudaFree(d);
}

}  // namespace

int main(int argc, char** argv)
{
    const Args a = parse(argc, argv);
    try {
        const size_t plane = (size_t)a.height * a.width;
        const size_t ni = plane * a.channels * a.batch, ng = plane * a.guide_channels * a.batch;
        blfls::detail::PinnedFloats in, gd, out0, out1;
        float* h_in = in.reserve(ni);
        float* h_g = a.guide_channels ? gd.reserve(ng) : nullptr;
        float* h_out[2] = {out0.reserve(ni), out1.reserve(ni)};
        std::vector<uint64_t> seeds, gseeds;
        for (int b = 0; b < a.batch; ++b) {
            for (int c = 0; c < a.channels; ++c) seeds.push_back((uint64_t)a.seed_base + 10 * b + c);
            if (a.guide_channels) gseeds.push_back((uint64_t)a.seed_base + 500 + b);
        }
        generate(h_in, a.height, a.width, seeds, a.devices[0]);
        if (h_g) generate(h_g, a.height, a.width, gseeds, a.devices[0]);
        const blfls_params prm = blfls::detail::make_params(a.height, a.width, a.channels, a.guide_channels,
                                                            a.radius, a.sigma_s, a.sigma_r, a.lambda, a.batch,
                                                            a.devices[0]);
        const bool multi = a.devices.size() > 1;
        std::unique_ptr<blfls::Plan> plan;
        std::unique_ptr<blfls::MultiPlan> mplan;
        if (multi) mplan.reset(new blfls::MultiPlan(prm, a.devices, BLFLS_MULTI_BATCH));
        else plan.reset(new blfls::Plan(prm));
        auto step = [&](int k) {
            if (multi) mplan->run(h_in, h_g, a.batch, a.iters, h_out[k & 1]);
            else plan->run_async(h_in, h_g, a.batch, a.iters, h_out[k & 1]);
        };
        for (int k = 0; k < a.warmup; ++k) step(k);
        if (!multi) plan->sync();
        const auto t0 = std::chrono::steady_clock::now();
        for (int k = 0; k < a.steps; ++k) step(k);
        if (!multi) plan->sync();
        const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() / a.steps;
        const double mp = (double)plane * a.batch * a.iters / 1e6;
        std::printf("{\"value\": %.3f, \"unit\": \"MP/s\", \"ms_per_step\": %.4f, \"steps\": %d, "
                    "\"h2d_bytes_per_step\": %zu, \"d2h_bytes_per_step\": %zu, \"devices\": %zu, "
                    "\"path\": \"%s\"}\n",
                    mp / s, s * 1e3, a.steps, (ni + ng) * sizeof(float), ni * sizeof(float), a.devices.size(),
                    multi ? "blfls::MultiPlan::run (blfls_multi_run, batch shards, host thread per device)"
                          : "blfls::Plan::run_async (blfls_run HOST_PTRS|ASYNC|CHECK_FINITE, pinned float buffers)");
        return 0;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
}
