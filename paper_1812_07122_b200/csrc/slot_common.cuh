// slot_common.cuh -- per "slot" (image b, channel c, gradient axis a) access
// to the normalised unit-range gradients src01 / guide01 that the reference's
// filter_gradients hands to its per-plane filters (pipelines.cpp:33-53),
// evaluated in double with the reference's rounding.  Shared by the
// bilateral-grid (k_grid.cu) and domain-transform (k_dt.cu) backends; P is
// their parameter block (fields f, guide, lohi, glohi, H, W, C, GC, plane0).
#pragma once

#include "blfls_internal.cuh"

namespace blfls {

// slot -> (image b, channel c, axis a); slot = (plane0 + local plane) * 2 + axis
struct Slot {
    int b, c, axis;
};
template <class P>
__device__ __forceinline__ Slot slot_of(const P& p, int z)
{
    const int gp = p.plane0 * 2 + z;
    Slot s;
    s.axis = gp & 1;
    const int plane = gp >> 1;
    s.b = plane / p.C;
    s.c = plane - s.b * p.C;
    return s;
}

// normalisation (lo, scale) of an image in double, image.cpp:46-60
__device__ __forceinline__ void norm_of(const uint32_t* lohi, int b, double& lo, double& scale)
{
    const double l = (double)ordered_to_float(lohi[2 * b]);
    const double h = (double)ordered_to_float(lohi[2 * b + 1]);
    lo = l;
    scale = h > l ? 1.0 / (h - l) : 0.0;  // constant image -> zeros
}

// ((gn[next] - gn[here]) + 1) * 0.5, every operation rounded as the reference's
__device__ __forceinline__ double grad01(const float* img, int H, int W, int y, int x, int axis,
                                         double lo, double scale)
{
    const int xn = axis == 0 ? (x + 1 == W ? 0 : x + 1) : x;
    const int yn = axis == 0 ? y : (y + 1 == H ? 0 : y + 1);
    const double a = __dmul_rn(__dsub_rn((double)__ldg(img + (size_t)yn * W + xn), lo), scale);
    const double b = __dmul_rn(__dsub_rn((double)__ldg(img + (size_t)y * W + x), lo), scale);
    return __dmul_rn(__dadd_rn(__dsub_rn(a, b), 1.0), 0.5);
}

template <class P>
__device__ __forceinline__ void slot_images(const P& p, const Slot& s, const float*& src,
                                            const float*& gde, double& slo, double& ssc, double& glo,
                                            double& gsc)
{
    const size_t plane = (size_t)p.H * p.W;
    src = p.f + ((size_t)s.b * p.C + s.c) * plane;
    norm_of(p.lohi, s.b, slo, ssc);
    if (p.guide) {
        gde = p.guide + ((size_t)s.b * p.GC + (p.GC == 1 ? 0 : s.c)) * plane;
        norm_of(p.glohi, s.b, glo, gsc);
    } else {
        gde = src;
        glo = slo;
        gsc = ssc;
    }
}

}  // namespace blfls
