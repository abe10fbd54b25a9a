// fft_backend.cpp -- replacement for the reference's FFTW seam
// (/root/reference/proj/src/fft2d.hpp:11,14; fft2d.cpp uses FFTW3, which is
// absent here).  TEST INFRASTRUCTURE ONLY: linked into oracle/_ref so the
// reference's own solver.cpp / pipelines.cpp run unmodified.  Same contract
// as fft2d.hpp:8-14: h x (w/2+1) half spectrum, forward exp(-i), inverse
// scaled by 1/(h*w), spectrum clobbered by the inverse.
#include <complex>
#include <vector>

#include "../blfls_oracle.h"

namespace epls::detail {

std::vector<std::complex<double>> rfft2(const double* data, int h, int w)
{
    const int wc = w / 2 + 1;
    std::vector<std::complex<double>> out(static_cast<std::size_t>(h) * wc);
    orc_rfft2(data, h, w, reinterpret_cast<double*>(out.data()));
    return out;
}

void irfft2(std::vector<std::complex<double>>& spec, int h, int w, double* out)
{
    orc_irfft2(reinterpret_cast<double*>(spec.data()), h, w, out);
}

} // namespace epls::detail
