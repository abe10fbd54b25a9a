// wls_shim.cpp -- stands in for /root/reference/proj/src/wls.cpp, which needs
// Eigen (absent).  TEST INFRASTRUCTURE ONLY.  wls_solve is out of scope for
// the BLF-LS path and throws; the dense normal-equations oracle
// (wls.cpp:78-144) is restated in oracle/blfls_oracle.c:orc_dense_solve with
// the same 4096-pixel cap and exception types.
#include <stdexcept>

#include "../blfls_oracle.h"
#include "epls/solver.hpp"

namespace epls {

PlanarImage wls_solve(const PlanarImage&, const WlsParams&)
{
    throw std::runtime_error("wls_solve: not built in oracle/_ref (Eigen absent; out of scope)");
}

namespace {
PlanarImage dense(const PlanarImage& g, const GradientField* t, double lambda)
{
    if (g.plane_size() > 4096)
        throw std::length_error("ls_solve_dense_oracle: refusing images beyond 4096 pixels");
    if (!(lambda >= 0.0))
        throw std::invalid_argument("ls_solve_dense_oracle: lambda must be finite and >= 0");
    require_finite(g, "ls_solve_dense_oracle");
    PlanarImage out(g.width(), g.height(), g.channels());
    orc_dense_solve(g.data().data(), t ? t->gx.data().data() : nullptr,
                    t ? t->gy.data().data() : nullptr, g.channels(), g.height(), g.width(), lambda,
                    out.data().data());
    return out;
}
} // namespace

PlanarImage ls_solve_dense_oracle(const PlanarImage& g, double lambda)
{
    return dense(g, nullptr, lambda);
}

PlanarImage ls_solve_dense_oracle(const PlanarImage& g, const GradientField& target, double lambda)
{
    if (!g.same_shape(target.gx) || !g.same_shape(target.gy))
        throw std::invalid_argument("ls_solve_dense_oracle: target shape does not match image");
    return dense(g, &target, lambda);
}

} // namespace epls
