// fusion.cuh -- element-wise neighbours fused into the matmul epilogue
// (include/relax_q4.h RELAX_OP_*).  Device only.
//
// Fusion keeps the semantics of the unfused fp16 program: every
// value is rounded to fp16 where the unfused chain would store a tensor.
#pragma once
#include <cstdint>
#include <cuda_fp16.h>
#include "relax_q4.h"

namespace rq4 {

// SiLU-mul of one (gate, up) pair of fp32 sums: both rounded to fp16 first
// (the unfused matmul's output tensor), silu in fp32, one RNE rounding.
__device__ __forceinline__ uint16_t silu_mul_value(float sg, float su) {
    const float g = __half2float(__float2half_rn(sg));
    const float u = __half2float(__float2half_rn(su));
    const float sl = g / (1.0f + expf(-g));
    return __half_as_ushort(__float2half_rn(sl * u));
}

// Residual add on the fp16 output value v: fp16(v + r) (r = the residual's
// fp16 bits; ignored without RELAX_OP_RESIDUAL).
__device__ __forceinline__ uint16_t residual_add(uint16_t v, uint32_t ops, uint16_t r) {
    if (!(ops & RELAX_OP_RESIDUAL)) return v;
    const float f = __half2float(__ushort_as_half(v)) + __half2float(__ushort_as_half(r));
    return __half_as_ushort(__float2half_rn(f));
}

__device__ __forceinline__ uint16_t epilogue_value(uint16_t v, uint32_t ops, const uint16_t* res, int64_t idx) {
    return residual_add(v, ops, (ops & RELAX_OP_RESIDUAL) ? res[idx] : uint16_t(0));
}

}  // namespace rq4
