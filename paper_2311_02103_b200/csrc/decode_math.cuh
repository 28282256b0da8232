// decode_math.cuh -- the per-lane arithmetic of the streamed decode kernels
// (gemv_stream.cu: one matrix per launch; decode_chain.cu: a whole chain of
// matrices in one persistent launch).  DESIGN.md §5.2.
#pragma once
#include <cstdint>
#include <cuda_fp16.h>
#include "ptx.cuh"

namespace rq4 {

// Transposed butterfly: acc[0..R) per lane -> every lane holds, in acc[0],
// the full 32-lane sum of row rsel(lane) = sum_s bit(lane, 4-s) * R >> (s+1).
template <int R>
__device__ __forceinline__ float reduce_rows(float (&acc)[R], int lane) {
    int cnt = R;
    int off = 16;
#pragma unroll
    for (int step = 0; (R >> step) > 1; ++step) {
        const int half = cnt >> 1;
        const bool upper = (lane & off) != 0;
#pragma unroll
        for (int j = 0; j < R / 2; ++j) {
            if (j < half) {
                const float send = upper ? acc[j] : acc[j + half];
                const float keep = upper ? acc[j + half] : acc[j];
                acc[j] = keep + __shfl_xor_sync(0xffffffffu, send, off);
            }
        }
        cnt = half;
        off >>= 1;
    }
#pragma unroll
    for (; off > 0; off >>= 1) acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], off);
    return acc[0];
}

template <int R>
__device__ __forceinline__ int reduce_row_of_lane(int lane) {
    int row = 0, off = 16;
#pragma unroll
    for (int step = 0; (R >> step) > 1; ++step) {
        if (lane & off) row += R >> (step + 1);
        off >>= 1;
    }
    return row;
}

// ZPF = 2 (default): integer dot products.  x of the lane's 32-code group is
// converted once per kernel to 16-bit fixed point with the group's own power
// of two (x_int = rint(x * 2^e), e chosen so max |x_int| is in [2^14, 2^15):
// exact for every x within 2^4 of the group's largest, within 2^-15 of it
// otherwise), and the codes stay bytes: per 8 codes 1 SHF + 2 LOP3 and four
// dp2a (int16 x int8 pairs -> int32, exact).  Per group
//   v = sum q x_int - 7 sum x_int      (int32, exact; |v| < 2^24)
// and out = float(v) * s * 2^-e.  An all-7 group gives v = 0 exactly; one-hot
// and integer x are exact (reading 6).  dp2a issues at
// 2 warp-instr/clk/SM and co-issues with the ALU (profiles/r02/ubench_idp_r02.txt):
// ~2.7x the FHFMA loop's math rate.
__device__ __forceinline__ int dp2a_lo(uint32_t a16x2, uint32_t b8x4, int c) {
    int d;
    asm("dp2a.lo.s32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a16x2), "r"(b8x4), "r"(c));
    return d;
}
__device__ __forceinline__ int dp2a_hi(uint32_t a16x2, uint32_t b8x4, int c) {
    int d;
    asm("dp2a.hi.s32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a16x2), "r"(b8x4), "r"(c));
    return d;
}
__device__ __forceinline__ uint32_t pack16(int lo, int hi) {
    return (static_cast<uint32_t>(lo) & 0xFFFFu) | (static_cast<uint32_t>(hi) << 16);
}

// x (4 uint4 = 32 fp16 of one group) -> int16 pairs in the dp2a order
// (x0,x2) (x4,x6) (x1,x3) (x5,x7) per 8 k, 7 * sum x_int, and 2^-e.
__device__ __forceinline__ void x_to_fixed(const uint4 (&xr)[4], uint32_t (&xi)[4][4], int& sx7, float& inv) {
    float f[32];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const uint32_t w4[4] = {xr[q].x, xr[q].y, xr[q].z, xr[q].w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const float2 v = __half22float2(u32_as_h2(w4[u]));
            f[q * 8 + 2 * u] = v.x;
            f[q * 8 + 2 * u + 1] = v.y;
        }
    }
    float m = 0.f;
#pragma unroll
    for (int i = 0; i < 32; ++i) m = fmaxf(m, fabsf(f[i]));
    int e = 0;                                       // scale 2^e with max|x| * 2^e in [2^14, 2^15)
    if (m > 0.f) e = 14 - (((__float_as_int(m) >> 23) & 0xFF) - 127);
    const float up = __int_as_float((127 + e) << 23);
    inv = __int_as_float((127 - e) << 23);
    int xi_[32];
    int sx = 0;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
        xi_[i] = __float2int_rn(f[i] * up);
        sx += xi_[i];
    }
    sx7 = 7 * sx;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int* v = xi_ + q * 8;
        xi[q][0] = pack16(v[0], v[2]);
        xi[q][1] = pack16(v[4], v[6]);
        xi[q][2] = pack16(v[1], v[3]);
        xi[q][3] = pack16(v[5], v[7]);
    }
}

template <int NT>
__device__ __forceinline__ void row_dot_idp(const uint4& cw, uint16_t sbits, const uint32_t (&xi)[NT][4][4],
                                            const int (&sx7)[NT], const float (&inv)[NT], float (&out)[NT]) {
    const uint32_t words[4] = {cw.x, cw.y, cw.z, cw.w};
    int acc_e[NT], acc_o[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) { acc_e[t] = 0; acc_o[t] = 0; }
#pragma unroll
    for (int wi = 0; wi < 4; ++wi) {
        const uint32_t ev = words[wi] & 0x0F0F0F0Fu;            // bytes q0 q2 q4 q6
        const uint32_t od = (words[wi] >> 4) & 0x0F0F0F0Fu;     // bytes q1 q3 q5 q7
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            acc_e[t] = dp2a_lo(xi[t][wi][0], ev, acc_e[t]);
            acc_e[t] = dp2a_hi(xi[t][wi][1], ev, acc_e[t]);
            acc_o[t] = dp2a_lo(xi[t][wi][2], od, acc_o[t]);
            acc_o[t] = dp2a_hi(xi[t][wi][3], od, acc_o[t]);
        }
    }
    const float sc = __half2float(__ushort_as_half(sbits));
#pragma unroll
    for (int t = 0; t < NT; ++t) out[t] = __int2float_rn(acc_e[t] + acc_o[t] - sx7[t]) * (sc * inv[t]);
}

}  // namespace rq4
