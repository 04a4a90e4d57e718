// Explicit instantiations of the FFT launchers: double arithmetic, float2 input.
#include "fft_impl.cuh"

namespace sfft {
template void dense_fft<double, float2>(sfft2d_ctx*, const float2*, cplx<double>*, double*, unsigned long long*, int,
                                 const cplx<double>*, cudaStream_t, unsigned*);
template cplx<double>* dense_fft_front<double, float2>(sfft2d_ctx*, const float2*, int, const cplx<double>*,
                                                 cudaStream_t, unsigned*);
}  // namespace sfft
