// Explicit instantiations of the FFT launchers: float arithmetic, double2 input.
#include "fft_impl.cuh"

namespace sfft {
template void dense_fft<float, double2>(sfft2d_ctx*, const double2*, cplx<float>*, float*, unsigned long long*, int,
                                 const cplx<float>*, cudaStream_t, unsigned*);
template cplx<float>* dense_fft_front<float, double2>(sfft2d_ctx*, const double2*, int, const cplx<float>*,
                                                 cudaStream_t, unsigned*);
}  // namespace sfft
