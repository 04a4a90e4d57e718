// |Z| with a per-segment peak (atomicMax on an order-preserving integer key:
// exact and independent of the reduction order).
#pragma once
#include "common.cuh"

namespace sfft {

template <typename T>
__global__ void k_mags(const cplx<T>* __restrict__ spec, long seglen, T* __restrict__ mags,
                       unsigned long long* __restrict__ peak) {
  pdl_wait();
  const int seg = blockIdx.y;
  const cplx<T>* s = spec + (size_t)seg * seglen;
  T* m = mags + (size_t)seg * seglen;
  unsigned long long best = 0ull;
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < seglen;
       e += (long)gridDim.x * blockDim.x) {
    const T v = cabs_(s[e]);
    m[e] = v;
    const unsigned long long k = fkey(v);
    best = k > best ? k : best;
  }
  if (peak) {
    for (int o = 16; o > 0; o >>= 1) {
      unsigned long long t = __shfl_xor_sync(0xffffffffu, best, o);
      best = t > best ? t : best;
    }
    if ((threadIdx.x & 31) == 0) atomicMax(peak + seg, best);
  }
}

}  // namespace sfft
