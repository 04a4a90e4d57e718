// Shared device helpers for the sm_100a sparse-FFT kernels.
//
// Complex numbers are stored as float2 / double2 (interleaved re, im) — the
// same byte layout as numpy complex64 / complex128, so images cross the C-ABI
// without repacking.  "T" is the arithmetic type of a kernel (float or double);
// "Tin" is the element type of the input image (float2 or double2).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace sfft {

constexpr int kNumSMs = 148;  // B200

template <typename T> struct CT;
template <> struct CT<float>  { using type = float2; };
template <> struct CT<double> { using type = double2; };
template <typename T> using cplx = typename CT<T>::type;

template <typename T> __host__ __device__ __forceinline__ cplx<T> mk(T re, T im) {
  cplx<T> z; z.x = re; z.y = im; return z;
}
template <typename C> __host__ __device__ __forceinline__ C cadd(C a, C b) {
  C z; z.x = a.x + b.x; z.y = a.y + b.y; return z;
}
template <typename C> __host__ __device__ __forceinline__ C csub(C a, C b) {
  C z; z.x = a.x - b.x; z.y = a.y - b.y; return z;
}
template <typename C> __host__ __device__ __forceinline__ C cmul(C a, C b) {
  C z; z.x = a.x * b.x - a.y * b.y; z.y = a.x * b.y + a.y * b.x; return z;
}
template <typename C, typename T> __host__ __device__ __forceinline__ C cscale(C a, T s) {
  C z; z.x = a.x * s; z.y = a.y * s; return z;
}

// widen / narrow an input element to the arithmetic type
template <typename T, typename Tin> __device__ __forceinline__ cplx<T> load_c(const Tin* p) {
  Tin v = *p;
  return mk<T>((T)v.x, (T)v.y);
}

// |z| the way numpy's np.abs(complex) computes it (hypot, no overflow)
__device__ __forceinline__ double cabs_(double2 z) { return hypot(z.x, z.y); }
__device__ __forceinline__ float  cabs_(float2 z)  { return hypotf(z.x, z.y); }
// |z| of the tuner's spectrum magnitudes (FFT epilogues): fp64 keeps numpy's
// hypot bit for bit; fp32 (a tolerance-checked mode, values O(1e-8..1e6))
// takes the cheaper sqrt(x^2 + y^2), ~10 fewer instructions per bin
__device__ __forceinline__ double mag_(double2 z) { return hypot(z.x, z.y); }
__device__ __forceinline__ float  mag_(float2 z)  { return sqrtf(fmaf(z.x, z.x, z.y * z.y)); }

// order-preserving unsigned key of a non-negative (or any) floating value:
// a < b  <=>  key(a) < key(b)   (NaN-free inputs)
__device__ __forceinline__ uint64_t fkey(double v) {
  uint64_t u = (uint64_t)__double_as_longlong(v);
  return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ uint64_t fkey(float v) { return fkey((double)v); }
__device__ __forceinline__ double fkey_inv(uint64_t k) {
  uint64_t u = (k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)u);
}

__device__ __forceinline__ unsigned bitrev(unsigned v, int bits) {
  return bits ? (__brev(v) >> (32 - bits)) : 0u;
}

// Programmatic dependent launch: kernels are launched with programmatic stream
// serialisation so a kernel's CTAs can be scheduled while its predecessor in
// the stream drains; every kernel waits here, before its first global memory
// access, until the predecessor has completed and its writes are visible.
__device__ __forceinline__ void pdl_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

// 16-byte global -> shared asynchronous copy (LDGSTS), no register staging
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

// ---- mbarrier + 1D bulk copy (TMA engine, no tensor map): one thread moves
// a contiguous global range into shared memory; the barrier's transaction
// count completes when the bytes have landed.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Publish a final per-launch count to mapped (zero-copy) host memory: every
// CTA calls this once after its contribution to *count is done; the CTA that
// takes ticket `target - 1` of the monotonic `done` counter is the last one and
// writes (seq, count) as one 8-byte word into slot[0..1], so the host can spin
// on seq without a stream synchronisation.
__device__ __forceinline__ void publish_count(unsigned* count, unsigned* done, unsigned target,
                                              volatile unsigned* slot, unsigned seq,
                                              unsigned* count2 = nullptr) {
  __threadfence();
  const unsigned t = atomicAdd(done, 1u);
  if (t + 1u == target) {
    __threadfence();
    const unsigned v = atomicAdd(count, 0u);
    if (count2) {   // optional second count: must land before the (seq, count) word
      slot[2] = atomicAdd(count2, 0u);
      __threadfence_system();
    }
    // (seq, count) in ONE aligned 8-byte store: the host sees both or neither,
    // so no system-scope fence (a ~2 us PCIe round trip each) is needed
    *reinterpret_cast<volatile unsigned long long*>(slot) =
        ((unsigned long long)v << 32) | (unsigned long long)seq;
    // the ticket counter is this publication's own (one per seq slot): reset
    // it for the slot's next use (every CTA of this launch has taken its ticket)
    atomicExch(done, 0u);
  }
}

struct Publish {
  unsigned* done;
  unsigned target;
  volatile unsigned* slot;
  unsigned seq;
};

// one permutation as the kernels consume it (see hashing.py:45-80)
struct Perm {
  uint32_t s1, s2, t1, t2, s1i, s2i;
};

// up to kMaxFoldLoops permutations passed by value to a fold launch
constexpr int kMaxFoldLoops = 8;
struct PermPack {
  Perm p[kMaxFoldLoops];
};

// block-wide inclusive scan helper over 32-bit counts (blockDim <= 1024)
__device__ __forceinline__ unsigned warp_incl_scan(unsigned v) {
  const unsigned lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    unsigned t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= (unsigned)o) v += t;
  }
  return v;
}

}  // namespace sfft
