// Explicit instantiations of the FFT launchers: float arithmetic, float2 input.
#include "fft_impl.cuh"

namespace sfft {
template void mags_of<float>(sfft2d_ctx*, const cplx<float>*, long, int, float*, unsigned long long*,
                         cudaStream_t);
template void fft2d_grids<float>(sfft2d_ctx*, cplx<float>*, int, int, const cplx<float>*, int, cplx<float>*,
                             float*, unsigned long long*, cudaStream_t);
template void dense_fft<float, float2>(sfft2d_ctx*, const float2*, cplx<float>*, float*, unsigned long long*, int,
                                 const cplx<float>*, cudaStream_t, unsigned*);
template cplx<float>* dense_fft_front<float, float2>(sfft2d_ctx*, const float2*, int, const cplx<float>*,
                                                 cudaStream_t, unsigned*);
template void dense_fft_xhat<float>(sfft2d_ctx*, cplx<float>*, int, const cplx<float>*, cudaStream_t);
template void dense_fft_mags<float>(sfft2d_ctx*, float*, unsigned long long*, int, const cplx<float>*,
                                  cudaStream_t);
// fp64 only: skipping the complex128 x_hat write saves ~70 us per 4096^2
// transform; in fp32 pass B gains only ~6 us while the per-candidate strided
// DFT reads cost ~13 us more (8.4K candidates x 64 scattered sectors).  The
// tuner overrides this for N <= 4096, where a stored x_hat lets the B = N/2
// passes run through k_pass_conv_band (run_ats: conv_possible), so the factored
// form is what fp64 uses at N = 8192 and 16384.
bool dense_factored(int lgN, int precision) {
  if (precision != SFFT2D_FP64) return false;
  const FftPlan2D pl = plan_fft2d<double>(lgN);
  return pl.four_step && !pl.col1;
}
void dense_split(int lgN, int precision, int* lgL1, int* lgL2) {
  const FftPlan2D pl = precision == SFFT2D_FP64 ? plan_fft2d<double>(lgN) : plan_fft2d<float>(lgN);
  *lgL1 = pl.lgL1;
  *lgL2 = pl.lgL2;
}
}  // namespace sfft
