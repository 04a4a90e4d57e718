// Definitions of the 2D FFT host launchers (fft_launch.cuh).  Every length
// between 16 and 16384 is dispatched to kernels compiled for that length
// (fft2.cuh with_lg), so each launch runs only the Stockham passes it needs.
#pragma once
#include <algorithm>
#include <type_traits>

#include "fft.cuh"
#include "fft2.cuh"
#include "fft_launch.cuh"
#include "host.cuh"
#include "mags.cuh"

namespace sfft {

template <typename T>
void mags_of(sfft2d_ctx* c, const cplx<T>* spec, long seglen, int nseg, T* mags,
             unsigned long long* peaks, cudaStream_t st) {
  pre(c, st);
  kl(k_mags<T>, dim3(grid_for(seglen, 256, kNumSMs * 8 / std::max(1, nseg) + 1), nseg), 256, 0, st,
     spec, seglen, mags, peaks);
  post(c, "k_mags", st, (double)seglen * nseg * (sizeof(cplx<T>) + sizeof(T)));
}

// Row pass: `nrows` rows of length L = 2^lgL from src to dst (may alias).
template <typename T, typename Tin>
void fft_rows(sfft2d_ctx* c, const FftPlan2D& pl, long nrows, const Tin* src, cplx<T>* dst,
              const cplx<T>* tw, int lgN, unsigned* nonfinite, const char* name, double bytes,
              cudaStream_t st) {
  if (pl.smem_row > kMaxDynSmem) {
    // fp64 L = 16384: one 2-CTA cluster per row (k_fftr_cl2)
    if (pl.lgL != 14) fail(SFFT2D_ERR_UNSUPPORTED, "row too long for the smem FFT");
    const size_t sm = (size_t)pad_row(1 << 13) * sizeof(cplx<T>);
    pre(c, st);
    klc(k_fftr_cl2<T, Tin, 13>, (unsigned)(2 * nrows), 512, sm, st, 2, src, dst, tw, lgN, nonfinite);
    post(c, "k_fftr_cl2", st, bytes);
    return;
  }
  const unsigned grid = (unsigned)(nrows / pl.rows_per_cta);
  pre(c, st);
  with_lg<4, 14>(pl.lgL, [&](auto LGc) {
    constexpr int LG = decltype(LGc)::value;
    if constexpr (LG == 14 || LG == 0) {
      if (pl.row_ipt == 2) {
        kl(k_fftr<T, Tin, true, false, 2, LG>, grid, pl.row_threads, pl.smem_row, st, src, dst,
           (T*)nullptr, (unsigned long long*)nullptr, pl.lgL, 2 * pl.lgL, tw, lgN, nonfinite);
        return;
      }
    }
    kl(k_fftr<T, Tin, true, false, 1, LG>, grid, pl.row_threads, pl.smem_row, st, src, dst,
       (T*)nullptr, (unsigned long long*)nullptr, pl.lgL, 2 * pl.lgL, tw, lgN, nonfinite);
  });
  post(c, name, st, bytes);
}

// Column pass of `ngrids` row-transformed grids in `src`: complex result to
// `out` (WC) and/or |Z| + per-grid peak (WM).  Four-step A runs in place on src.
template <typename T, bool WC, bool WM>
void fft_cols(sfft2d_ctx* c, const FftPlan2D& pl, int ngrids, cplx<T>* src, cplx<T>* out,
              T* mags, unsigned long long* peaks, const cplx<T>* tw, int lgN, double gb,
              double wbytes, cudaStream_t st) {
  const int L = 1 << pl.lgL;
  if (pl.col1) {
    pre(c, st);
    kl(k_fftc1<T, WC, WM, 1, 10>, dim3(L >> pl.lgcc1, ngrids), pl.thr1, pl.smem_1, st, src, out,
       mags, peaks, pl.lgL, pl.lgcc1, tw, lgN);
    post(c, "k_fftc1", st, gb + wbytes);
  } else if (pl.four_step) {
    pre(c, st);
    with_lg<6, 7>(pl.lgL1, [&](auto LGc) {
      constexpr int LG1 = decltype(LGc)::value;
      kl(k_fftcA<T, LG1>, dim3(L >> pl.lgccA, 1 << pl.lgL2, ngrids), pl.thrA, pl.smem_A, st, src,
         pl.lgL1, pl.lgL2, pl.lgccA, tw, lgN);
    });
    post(c, "k_fftcA", st, 2 * gb);
    pre(c, st);
    with_lg<5, 7>(pl.lgL2, [&](auto LGc) {
      constexpr int LG2 = decltype(LGc)::value;
      kl(k_fftcB<T, WC, WM, LG2>, dim3(L >> pl.lgccB, 1 << pl.lgL1, ngrids), pl.thrB, pl.smem_B,
         st, (const cplx<T>*)src, out, mags, peaks, pl.lgL1, pl.lgL2, pl.lgccB, tw, lgN);
    });
    post(c, "k_fftcB", st, gb + wbytes);
  } else {
    pre(c, st);
    with_lg<4, 9>(pl.lgL, [&](auto LGc) {
      constexpr int LG = decltype(LGc)::value;
      kl(k_fftc<T, WC, WM, LG>, dim3(L >> pl.lgccB, ngrids), pl.thrB, pl.smem_B, st,
         (const cplx<T>*)src, out, mags, peaks, pl.lgL, pl.lgccB, tw, lgN);
    });
    post(c, "k_fftc", st, gb + wbytes);
  }
}

template <typename T>
void fft2d_grids(sfft2d_ctx* c, cplx<T>* grids, int lgB, int ngrids, const cplx<T>* tw, int lgN,
                 cplx<T>* out, T* mags, unsigned long long* peaks, cudaStream_t st) {
  using C = cplx<T>;
  const int B = 1 << lgB;
  const size_t BB = (size_t)B * B;
  const double gb = (double)BB * ngrids * sizeof(C);
  const bool wc = out != nullptr, wm = mags != nullptr;
  if (BB * sizeof(C) <= (size_t)kSmall2DBytes) {
    const int threads = B * B / 4 >= 256 ? 256 : (B * B / 4 >= 32 ? B * B / 4 : 32);
    pre(c, st);
    kl(k_fft2d_small<T>, ngrids, threads, ((size_t)B * (B + 1) + B) * sizeof(C), st, grids, lgB, tw, lgN);
    post(c, "k_fft2d_small", st, 2 * gb);
    if (wc && out != grids)
      ck(cudaMemcpyAsync(out, grids, BB * ngrids * sizeof(C), cudaMemcpyDeviceToDevice, st), "copy");
    if (wm) mags_of<T>(c, wc ? out : grids, (long)BB, ngrids, mags, peaks, st);
    return;
  }
  const FftPlan2D pl = plan_fft2d<T>(lgB);
  if ((pl.smem_row > kMaxDynSmem && pl.lgL != 14) || pl.row_threads > 512)
    fail(SFFT2D_ERR_UNSUPPORTED, "grid too large for the smem FFT");
  fft_rows<T, C>(c, pl, (long)ngrids * B, grids, grids, tw, lgN, nullptr, "k_fftr", 2 * gb, st);
  const double wbytes = (wc ? gb : 0) + (wm ? (double)BB * ngrids * sizeof(T) : 0);
  C* final_out = out;
  // four-step B cannot run in place (k_fftc / k_fftc1 can: a CTA reads all of
  // its columns before writing)
  if (pl.four_step && !pl.col1 && wc && out == grids)
    out = (C*)ws(c, "fft_tmp", (size_t)BB * ngrids * sizeof(C));
  if (wc && wm) fft_cols<T, true, true>(c, pl, ngrids, grids, out, mags, peaks, tw, lgN, gb, wbytes, st);
  else if (wc) fft_cols<T, true, false>(c, pl, ngrids, grids, out, nullptr, nullptr, tw, lgN, gb, wbytes, st);
  else fft_cols<T, false, true>(c, pl, ngrids, grids, nullptr, mags, peaks, tw, lgN, gb, wbytes, st);
  if (final_out != out)
    ck(cudaMemcpyAsync(final_out, out, BB * ngrids * sizeof(C), cudaMemcpyDeviceToDevice, st), "copy");
}

template <typename T, typename Tin>
void dense_fft(sfft2d_ctx* c, const Tin* x, cplx<T>* out, T* mags, unsigned long long* peak,
               int lgN, const cplx<T>* tw, cudaStream_t st, unsigned* nonfinite) {
  using C = cplx<T>;
  const int N = 1 << lgN;
  const FftPlan2D pl = plan_fft2d<T>(lgN);
  if ((pl.smem_row > kMaxDynSmem && pl.lgL != 14) || pl.row_threads > 512)
    fail(SFFT2D_ERR_UNSUPPORTED, "image side too large for the smem FFT");
  const double nn = (double)N * N;
  C* scratch = (C*)ws(c, "fft_scratch", (size_t)N * N * sizeof(C));
  fft_rows<T, Tin>(c, pl, N, x, scratch, tw, lgN, nonfinite, "k_fftr_dense",
                   nn * (sizeof(Tin) + sizeof(C)), st);
  const double gb = nn * sizeof(C);
  const double wb = nn * sizeof(C) + (mags ? nn * sizeof(T) : 0);
  if (mags) fft_cols<T, true, true>(c, pl, 1, scratch, out, mags, peak, tw, lgN, gb, wb, st);
  else fft_cols<T, true, false>(c, pl, 1, scratch, out, nullptr, nullptr, tw, lgN, gb, wb, st);
}

template <typename T, typename Tin>
cplx<T>* dense_fft_front(sfft2d_ctx* c, const Tin* x, int lgN, const cplx<T>* tw, cudaStream_t st,
                         unsigned* nonfinite) {
  using C = cplx<T>;
  const int N = 1 << lgN;
  const FftPlan2D pl = plan_fft2d<T>(lgN);
  if (!pl.four_step || pl.col1) fail(SFFT2D_ERR_STATE, "factored dense FFT needs four-step columns");
  if ((pl.smem_row > kMaxDynSmem && pl.lgL != 14) || pl.row_threads > 512)
    fail(SFFT2D_ERR_UNSUPPORTED, "image side too large for the smem FFT");
  const double nn = (double)N * N;
  C* scratch = (C*)ws(c, "fft_scratch", (size_t)N * N * sizeof(C));
  fft_rows<T, Tin>(c, pl, N, x, scratch, tw, lgN, nonfinite, "k_fftr_dense",
                   nn * (sizeof(Tin) + sizeof(C)), st);
  pre(c, st);
  with_lg<6, 7>(pl.lgL1, [&](auto LGc) {
    constexpr int LG1 = decltype(LGc)::value;
    kl(k_fftcA<T, LG1>, dim3(N >> pl.lgccA, 1 << pl.lgL2, 1), pl.thrA, pl.smem_A, st, scratch,
       pl.lgL1, pl.lgL2, pl.lgccA, tw, lgN);
  });
  post(c, "k_fftcA", st, 2 * nn * sizeof(C));
  return scratch;
}

template <typename T>
void dense_fft_xhat(sfft2d_ctx* c, cplx<T>* out, int lgN, const cplx<T>* tw, cudaStream_t st) {
  using C = cplx<T>;
  const int N = 1 << lgN;
  const FftPlan2D pl = plan_fft2d<T>(lgN);
  const double nn = (double)N * N;
  C* scratch = (C*)ws(c, "fft_scratch", (size_t)N * N * sizeof(C));
  pre(c, st);
  with_lg<5, 7>(pl.lgL2, [&](auto LGc) {
    constexpr int LG2 = decltype(LGc)::value;
    kl(k_fftcB<T, true, false, LG2>, dim3(N >> pl.lgccB, 1 << pl.lgL1, 1), pl.thrB, pl.smem_B, st,
       (const C*)scratch, out, (T*)nullptr, (unsigned long long*)nullptr, pl.lgL1, pl.lgL2, pl.lgccB,
       tw, lgN);
  });
  post(c, "k_fftcB", st, 2 * nn * sizeof(C));
}

template <typename T>
void dense_fft_mags(sfft2d_ctx* c, T* mags, unsigned long long* peak, int lgN, const cplx<T>* tw,
                    cudaStream_t st) {
  using C = cplx<T>;
  const int N = 1 << lgN;
  const FftPlan2D pl = plan_fft2d<T>(lgN);
  const double nn = (double)N * N;
  C* scratch = (C*)ws(c, "fft_scratch", (size_t)N * N * sizeof(C));
  pre(c, st);
  with_lg<5, 7>(pl.lgL2, [&](auto LGc) {
    constexpr int LG2 = decltype(LGc)::value;
    kl(k_fftcB<T, false, true, LG2>, dim3(N >> pl.lgccB, 1 << pl.lgL1, 1), pl.thrB, pl.smem_B, st,
       (const C*)scratch, (C*)nullptr, mags, peak, pl.lgL1, pl.lgL2, pl.lgccB, tw, lgN);
  });
  post(c, "k_fftcB", st, nn * (sizeof(C) + sizeof(T)));
}

}  // namespace sfft
