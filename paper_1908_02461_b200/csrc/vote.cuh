// K5 — reverse hashing and voting.
// Replaces _unhash_axis/_unhash_grid (hashing.py:368-386) plus
//   * SFFT per-loop dedup + vote (engine.py:141-160): a coordinate counts once
//     per loop -> a per-coordinate bitmask byte, bit l = "loop l hit it";
//   * tuner votes with multiplicity (tuner.py:175-179, 228-240) -> a per-
//     coordinate byte counter (a strict local maximum's expanded 3x3 preimage
//     can overlap at most 4 others at w = 1 and none at w >= 2, so tallies are
//     bounded by 4 * passes; when that bound exceeds 255 the counters are 32 bit).
// Bytes are packed four to a 32-bit word and updated with atomicOr / atomicAdd
// on the containing word (no carry can cross a byte: bounded above).
//
// Preimage of bin c along one axis with w = N/B and expand e:
//   t in [c*w - floor(w/2) - e, c*w + ceil(w/2) + e)  (length min(w + 2e, N)),
//   coordinate = sigma^-1 * t mod N.
#pragma once
#include "common.cuh"
#include "select.cuh"

namespace sfft {

enum VoteMode { kVoteOrBit = 0, kVoteAdd8 = 1, kVoteAdd32 = 2 };

// bins: flat bin indices (bi*B + bj) per segment, `counts[seg]` valid entries
// (or uniform `count` when counts == nullptr); one permutation per segment.
// budget > 0: skip the whole segment when nb * len^2 > budget (the tuner's
// vote budget, tuner.py:165,175, evaluated on the device so the vote can be
// queued before the host learns the count).
__global__ void k_vote(const int32_t* __restrict__ bins, long seg_stride, const unsigned* counts,
                       long count, const Perm* __restrict__ perms, int lgN, int lgB, int expand,
                       int mode, int bit0, uint32_t* __restrict__ hist, long long budget = 0,
                       Perm pval = Perm{0, 0, 0, 0, 0, 0}) {
  pdl_wait();
  const int seg = blockIdx.y;
  const long nb = counts ? (long)counts[seg] : count;
  const int N = 1 << lgN;
  const unsigned maskN = (unsigned)N - 1u;
  const int w = N >> lgB;
  int len, shiftlo;
  if (w == 1 && expand == 0) {
    len = 1;
    shiftlo = 0;
  } else {
    len = min(w + 2 * expand, N);
    shiftlo = w / 2 + expand;
  }
  const long per = (long)len * len;
  const long total = nb * per;
  if (budget > 0 && total > budget) return;
  const Perm p = perms ? perms[seg] : pval;   // by value for single-segment tuner votes
  const int32_t* sb = bins + seg * seg_stride;
  const unsigned bitv = 1u << ((bit0 + seg) & 7);
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < total;
       e += (long)gridDim.x * blockDim.x) {
    const long q = e / per;
    const int rem = (int)(e - q * per);
    const int a = rem / len, b = rem - a * len;
    const unsigned bin = (unsigned)sb[q];
    const unsigned bi = bin >> lgB, bj = bin & ((1u << lgB) - 1u);
    const unsigned ti = (unsigned)((int)(bi * w) - shiftlo + a) & maskN;
    const unsigned tj = (unsigned)((int)(bj * w) - shiftlo + b) & maskN;
    const unsigned ii = (p.s1i * ti) & maskN, jj = (p.s2i * tj) & maskN;
    const size_t key = ((size_t)ii << lgN) | jj;
    if (mode == kVoteAdd32) {
      atomicAdd(hist + key, 1u);
    } else {
      const unsigned sh = (unsigned)(key & 3u) * 8u;
      if (mode == kVoteAdd8) atomicAdd(hist + (key >> 2), 1u << sh);
      else atomicOr(hist + (key >> 2), bitv << sh);
    }
  }
}

// Fold one group's loop-bit masks into per-coordinate loop counts (L > 8).
__global__ void k_mask_to_counts(uint32_t* __restrict__ masks, uint32_t* __restrict__ counts,
                                 long nwords) {
  pdl_wait();
  for (long w = blockIdx.x * (long)blockDim.x + threadIdx.x; w < nwords;
       w += (long)gridDim.x * blockDim.x) {
    const uint32_t m = masks[w];
    if (!m) continue;
    uint32_t add = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) add |= (uint32_t)__popc((m >> (8 * b)) & 255u) << (8 * b);
    counts[w] += add;
    masks[w] = 0;
  }
}

// value of coordinate `key` in a histogram of the given mode
__device__ __forceinline__ unsigned hist_value(const uint32_t* hist, size_t key, int mode) {
  if (mode == kVoteAdd32) return hist[key];
  const unsigned byte = (hist[key >> 2] >> ((key & 3u) * 8u)) & 255u;
  return mode == kVoteOrBit ? (unsigned)__popc(byte) : byte;
}

// bitmask of coordinates with value >= thr (block = 8192 coordinates)
__global__ void k_hist_bits(const uint32_t* __restrict__ hist, long nkeys, int mode, unsigned thr,
                            uint32_t* __restrict__ bits, unsigned* __restrict__ blk_counts) {
  pdl_wait();
  __shared__ unsigned s_warp[32];
  const long w = (long)blockIdx.x * kCmpWords + threadIdx.x;
  const long wps = words_for(nkeys);
  uint32_t word = 0;
  if (w < wps) {
    const long k0 = w * 32;
    if (mode == kVoteAdd32) {
      for (int b = 0; b < 32; ++b)
        if (k0 + b < nkeys && hist[k0 + b] >= thr) word |= 1u << b;
    } else {
      // 32 keys = 8 packed words = two 16-byte loads
      const uint4* h4 = reinterpret_cast<const uint4*>(hist + k0 / 4);
      const uint4 u0 = h4[0], u1 = h4[1];
      const uint32_t hw[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (!hw[i]) continue;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          unsigned v = (hw[i] >> (8 * b)) & 255u;
          if (mode == kVoteOrBit) v = __popc(v);
          if (v >= thr) word |= 1u << (i * 4 + b);
        }
      }
    }
    bits[w] = word;
  }
  const unsigned pre = block_excl_scan256(__popc(word), s_warp);
  if (threadIdx.x == kCmpThreads - 1) blk_counts[blockIdx.x] = pre + __popc(word);
}

// tallies of compacted keys
__global__ void k_gather_tallies(const uint32_t* __restrict__ hist, int mode,
                                 const int32_t* __restrict__ keys, const unsigned* __restrict__ m,
                                 int32_t* __restrict__ tallies) {
  pdl_wait();
  const long n = *m;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n;
       i += (long)gridDim.x * blockDim.x)
    tallies[i] = (int32_t)hist_value(hist, (size_t)(uint32_t)keys[i], mode);
}

}  // namespace sfft
