// philox.cuh — Philox4x32-10 counter RNG on the device (NS "counter-based Philox RNG";
// D2 in DESIGN.md §3).  Salmon et al., SC'11: ten rounds of two 32x32->64 multiplies,
// key bumped by the Weyl constants between rounds.
#pragma once
#include <stdint.h>

namespace dk {

__host__ __device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r > 0) { k.x += 0x9E3779B9u; k.y += 0xBB67AE85u; }
#ifdef __CUDA_ARCH__
        const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
#else
        const uint64_t p0 = (uint64_t)0xD2511F53u * c.x, p1 = (uint64_t)0xCD9E8D57u * c.z;
        const uint32_t lo0 = (uint32_t)p0, hi0 = (uint32_t)(p0 >> 32);
        const uint32_t lo1 = (uint32_t)p1, hi1 = (uint32_t)(p1 >> 32);
#endif
        c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    }
    return c;
}

// Block `blk` of a stream: counter = (blk, purpose << 24 | slot, generation, run).
__device__ __forceinline__ uint4 stream_block(uint2 key, uint32_t purpose, uint32_t slot,
                                              uint32_t gen, uint32_t run, uint32_t blk) {
    return philox4x32_10(make_uint4(blk, (purpose << 24) | slot, gen, run), key);
}

__device__ __forceinline__ uint32_t lane_of(uint4 v, uint32_t i) {
    return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w));
}

// Word m of a stream = lane (m & 3) of block m >> 2.
__device__ __forceinline__ uint32_t stream_word(uint2 key, uint32_t purpose, uint32_t slot,
                                                uint32_t gen, uint32_t run, uint32_t m) {
    return lane_of(stream_block(key, purpose, slot, gen, run, m >> 2), m & 3);
}

// u01(w) = (w >> 8) * 2^-24 (exact in float); below(w, n) = floor(w * n / 2^32).
__device__ __forceinline__ float u01(uint32_t w) { return (float)(w >> 8) * (1.0f / 16777216.0f); }
__device__ __forceinline__ uint32_t below(uint32_t w, uint32_t n) { return __umulhi(w, n); }

}  // namespace dk
