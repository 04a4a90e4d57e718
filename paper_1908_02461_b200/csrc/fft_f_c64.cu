// Explicit instantiations of the FFT launchers: float arithmetic, float2 input.
#include "fft_impl.cuh"

namespace sfft {
template void mags_of<float>(sfft2d_ctx*, const cplx<float>*, long, int, float*, unsigned long long*,
                         cudaStream_t);
template void fft2d_grids<float>(sfft2d_ctx*, cplx<float>*, int, int, const cplx<float>*, int, cplx<float>*,
                             float*, unsigned long long*, cudaStream_t);
template void dense_fft<float, float2>(sfft2d_ctx*, const float2*, cplx<float>*, float*, unsigned long long*, int,
                                 const cplx<float>*, cudaStream_t, unsigned*);
}  // namespace sfft
