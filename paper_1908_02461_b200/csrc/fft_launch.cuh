// Host launchers of the 2D FFT kernels (definitions in fft_impl.cuh, compiled
// in the fft_*.cu translation units; explicit instantiations for float and
// double there).
#pragma once
#include <cuda_runtime.h>

#include "../../include/sfft2d_b200.h"
#include "common.cuh"

namespace sfft {

// |Z| per element + a per-segment peak key (atomicMax; peaks zeroed by caller)
template <typename T>
void mags_of(sfft2d_ctx* c, const cplx<T>* spec, long seglen, int nseg, T* mags,
             unsigned long long* peaks, cudaStream_t st);

// 2D FFT of `ngrids` contiguous B x B grids held in `grids` (overwritten).
// out (optional): complex spectra (may equal `grids`); mags/peaks (optional):
// |Z| and a per-grid peak key (peaks zeroed by the caller).
template <typename T>
void fft2d_grids(sfft2d_ctx* c, cplx<T>* grids, int lgB, int ngrids, const cplx<T>* tw, int lgN,
                 cplx<T>* out, T* mags, unsigned long long* peaks, cudaStream_t st);

// Dense forward 2D FFT of the N x N input image: complex x_hat into `out`,
// optional |x_hat| + peak; nonfinite (optional) is set if x holds NaN/Inf.
template <typename T, typename Tin>
void dense_fft(sfft2d_ctx* c, const Tin* x, cplx<T>* out, T* mags, unsigned long long* peak,
               int lgN, const cplx<T>* tw, cudaStream_t st, unsigned* nonfinite);

// Factored dense FFT (sides >= 2048, four-step columns): dense_fft_front runs
// the row pass and four-step pass A into the context's "fft_scratch" buffer
// (returns it; nonfinite as in dense_fft); dense_fft_mags then runs pass B
// writing only |x_hat| + peak.  x_hat itself is never written: its entries are
// L2-point DFTs of scratch columns (k_estimate_dense_fs).
bool dense_factored(int lgN, int precision);
void dense_split(int lgN, int precision, int* lgL1, int* lgL2);
template <typename T, typename Tin>
cplx<T>* dense_fft_front(sfft2d_ctx* c, const Tin* x, int lgN, const cplx<T>* tw, cudaStream_t st,
                         unsigned* nonfinite);
template <typename T>
void dense_fft_xhat(sfft2d_ctx* c, cplx<T>* out, int lgN, const cplx<T>* tw, cudaStream_t st);
template <typename T>
void dense_fft_mags(sfft2d_ctx* c, T* mags, unsigned long long* peak, int lgN, const cplx<T>* tw,
                    cudaStream_t st);

}  // namespace sfft
