// q4_unpack.cuh -- in-register unpacking of q4f16 codes (device only).
//
// Storage format (readings 1-4): eight unsigned 4-bit codes per
// little-endian uint32 along K, element k at bits 4*(k mod 8); one fp16 scale
// per 32 consecutive k; W = fp16_RNE((q - 7) * s)  ("int4 weights,
// float16 activations"; the dequant producer fused into the matmul consumer,
// P:471-494).
//
// Both unpackers use the fp16 "magic number" trick: OR-ing a nibble into the
// mantissa of 0x6400 (= 1024.0, whose ulp is 1) gives the exact value
// 1024 + q; a nibble in mantissa bits 4..7 gives 1024 + 16 q.  One fused
// HFMA2 then yields q - 7 exactly (small integers are exact in binary16, and
// the fused multiply-add rounds once, so it is the integer itself).
#pragma once
#include <cstdint>
#include <cuda_fp16.h>
#include "ptx.cuh"

namespace rq4 {

// (1024 + q, 1024 + 16 q') * (1, 1/16) + (-1031, -71) = (q - 7, q' - 7).
__device__ __forceinline__ __half2 magic_to_centered(uint32_t h) {
    const __half2 mul = __halves2half2(__ushort_as_half(0x3C00), __ushort_as_half(0x2C00));   // 1, 1/16
    const __half2 add = __halves2half2(__ushort_as_half(0xE407), __ushort_as_half(0xD470));   // -1031, -71
    return __hfma2(u32_as_h2(h), mul, add);
}

// GEMV unpack: q - 7 for the 8 codes of one word, as 4 half2 in the
// interleaved order the FHFMA selectors consume directly:
//   c[0] = (k0, k4)   c[1] = (k1, k5)   c[2] = (k2, k6)   c[3] = (k3, k7)
// Cost: 1 SHF + 4 LOP3 (ALU) + 4 HFMA2.
__device__ __forceinline__ void unpack_centered_interleaved(uint32_t v, __half2 (&c)[4]) {
    const uint32_t v8 = v >> 8;
    const __half2 mul_lo = __half2half2(__ushort_as_half(0x3C00));           // 1
    const __half2 add_lo = __half2half2(__ushort_as_half(0xE407));           // -1031
    const __half2 mul_hi = __half2half2(__ushort_as_half(0x2C00));           // 1/16
    const __half2 add_hi = __half2half2(__ushort_as_half(0xD470));           // -71
    c[0] = __hfma2(u32_as_h2(lop3_and_or(v,  0x000F000Fu, 0x64006400u)), mul_lo, add_lo);
    c[1] = __hfma2(u32_as_h2(lop3_and_or(v,  0x00F000F0u, 0x64006400u)), mul_hi, add_hi);
    c[2] = __hfma2(u32_as_h2(lop3_and_or(v8, 0x000F000Fu, 0x64006400u)), mul_lo, add_lo);
    c[3] = __hfma2(u32_as_h2(lop3_and_or(v8, 0x00F000F0u, 0x64006400u)), mul_hi, add_hi);
}

// Tensor-core unpack: W = fp16_RNE((q - 7) * s) for the 8 codes of one word,
// bit-exact, as 4 half2 in natural pair order out[p] = (W[2p], W[2p+1]) (the
// K-packing of an fp16 operand in TMEM/SMEM).  Byte b of the word holds codes
// (2b, 2b+1); PRMT copies byte b to bytes 0 and 2, the mask keeps code 2b in
// bits 0..3 and code 2b+1 in bits 20..23.
// Cost: 4 PRMT + 4 LOP3 (ALU) + 4 HFMA2 + 4 HMUL2.
__device__ __forceinline__ void dequant_word_natural(uint32_t v, __half2 s2, uint32_t (&out)[4]) {
#pragma unroll
    for (int b = 0; b < 4; ++b) {
        const uint32_t sel = static_cast<uint32_t>(b) | (4u << 4) | (static_cast<uint32_t>(b) << 8) | (4u << 12);
        const uint32_t t = prmt(v, 0u, sel);
        const __half2 qc = magic_to_centered(lop3_and_or(t, 0x00F0000Fu, 0x64006400u));
        out[b] = h2_as_u32(__hmul2(qc, s2));           // one RNE rounding of the exact product
    }
}

// Tensor-core unpack without byte permutes: W for the 8 codes of one word,
// bit-exact, as 4 half2 in the interleaved order (W0,W4) (W1,W5) (W2,W6)
// (W3,W7) -- the TMEM A columns then hold k in the order 0,4,1,5,2,6,3,7 of
// every 8, and the B operand (x) is written with the same permutation.
// Cost: 1 SHF + 4 LOP3 (ALU) + 4 HFMA2 + 4 HMUL2.
__device__ __forceinline__ void dequant_word_interleaved(uint32_t v, __half2 s2, uint32_t (&out)[4]) {
    __half2 c[4];
    unpack_centered_interleaved(v, c);
#pragma unroll
    for (int i = 0; i < 4; ++i) out[i] = h2_as_u32(__hmul2(c[i], s2));
}

// x permutation matching dequant_word_interleaved: 8 fp16 (k0..k7 as 4 half2
// words w0=(k0,k1) w1=(k2,k3) w2=(k4,k5) w3=(k6,k7)) -> (k0,k4)(k1,k5)(k2,k6)(k3,k7).
__device__ __forceinline__ uint4 permute_x8(uint4 v) {
    return make_uint4(prmt(v.x, v.z, 0x5410u), prmt(v.x, v.z, 0x7632u),
                      prmt(v.y, v.w, 0x5410u), prmt(v.y, v.w, 0x7632u));
}

}  // namespace rq4
