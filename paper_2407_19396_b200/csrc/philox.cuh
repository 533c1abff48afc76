// philox.cuh — device Philox4x32-10 and the draw streams of DESIGN.md R#20/R#21.
//
// Salmon et al., SC'11.  Counter (c0, c1, c2, c3) = (global env index,
// episode, domain << 16 | step, block); key = (seed lo, seed hi).  Draw k of a
// stream is word k mod 4 of block k / 4.  Integer in [0, n): (u * n) >> 32.
#pragma once
#include <cstdint>

namespace navix {

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

__device__ __forceinline__ uint32_t bounded(uint32_t u, uint32_t n) { return __umulhi(u, n); }

// Sequential draws from one counter stream (level generation).
struct DrawStream {
  uint32_t c0, c1, c2, k0, k1;
  uint32_t blk;   // block index of `buf`
  uint32_t pos;   // next draw index
  uint4 buf;
  __device__ DrawStream(uint32_t env, uint32_t episode, uint32_t c2_, uint32_t key_lo, uint32_t key_hi)
      : c0(env), c1(episode), c2(c2_), k0(key_lo), k1(key_hi), blk(0xffffffffu), pos(0) {}
  __device__ __forceinline__ uint32_t next() {
    const uint32_t b = pos >> 2;
    if (b != blk) {
      buf = philox4x32_10(make_uint4(c0, c1, c2, b), k0, k1);
      blk = b;
    }
    const uint32_t w = pos & 3;
    ++pos;
    return w == 0 ? buf.x : w == 1 ? buf.y : w == 2 ? buf.z : buf.w;
  }
  __device__ __forceinline__ uint32_t next_bounded(uint32_t n) { return bounded(next(), n); }
};

}  // namespace navix
