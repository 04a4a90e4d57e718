// Explicit instantiations of the FFT launchers: double arithmetic, double2 input.
#include "fft_impl.cuh"

namespace sfft {
template void mags_of<double>(sfft2d_ctx*, const cplx<double>*, long, int, double*, unsigned long long*,
                         cudaStream_t);
template void fft2d_grids<double>(sfft2d_ctx*, cplx<double>*, int, int, const cplx<double>*, int, cplx<double>*,
                             double*, unsigned long long*, cudaStream_t);
template void dense_fft<double, double2>(sfft2d_ctx*, const double2*, cplx<double>*, double*, unsigned long long*, int,
                                 const cplx<double>*, cudaStream_t, unsigned*);
template cplx<double>* dense_fft_front<double, double2>(sfft2d_ctx*, const double2*, int, const cplx<double>*,
                                                 cudaStream_t, unsigned*);
template void dense_fft_xhat<double>(sfft2d_ctx*, cplx<double>*, int, const cplx<double>*, cudaStream_t);
template void dense_fft_mags<double>(sfft2d_ctx*, double*, unsigned long long*, int, const cplx<double>*,
                                  cudaStream_t);
}  // namespace sfft
