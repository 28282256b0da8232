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

// x (4 uint4 = 32 fp16 of one group) -> int16 pairs in the dp2a order
// (x0,x2) (x4,x6) (x1,x3) (x5,x7) per 8 k, 7 * sum x_int, and 2^-e.
__device__ __forceinline__ void x_to_fixed(const uint4 (&xr)[4], uint32_t (&xi)[4][4], int& sx7, float& inv) {
    // On the critical path of every decode kernel (right after
    // griddepcontrol.wait), so written without conversion instructions
    // (F2I is quarter rate): wait -> x in registers 1.05 -> 0.8 us (load
    // included), the same bits.
    const uint32_t w[16] = {xr[0].x, xr[0].y, xr[0].z, xr[0].w, xr[1].x, xr[1].y, xr[1].z, xr[1].w,
                            xr[2].x, xr[2].y, xr[2].z, xr[2].w, xr[3].x, xr[3].y, xr[3].z, xr[3].w};
    // max |x| of the group: a half2 tree (exact)
    __half2 mx[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) mx[i] = __hmax2(__habs2(u32_as_h2(w[2 * i])), __habs2(u32_as_h2(w[2 * i + 1])));
#pragma unroll
    for (int i = 0; i < 4; ++i) mx[i] = __hmax2(mx[i], mx[i + 4]);
    mx[0] = __hmax2(__hmax2(mx[0], mx[2]), __hmax2(mx[1], mx[3]));
    const float m = fmaxf(__low2float(mx[0]), __high2float(mx[0]));
    int e = 0;                                       // scale 2^e with max|x| * 2^e in [2^14, 2^15)
    if (m > 0.f) e = 14 - (((__float_as_int(m) >> 23) & 0xFF) - 127);
    const float up = __int_as_float((127 + e) << 23);
    inv = __int_as_float((127 - e) << 23);
    // x_int = rint(x * 2^e) through the 1.5 * 2^23 magic number: fma(x, 2^e,
    // magic) is magic + rint(x * 2^e) exactly (|x * 2^e| < 2^15 < 2^22, one RNE
    // rounding of an exact product), so its bits are 0x4B400000 + x_int and
    // their low 16 bits are x_int's
    constexpr float kMagic = 12582912.0f;
    uint32_t b[32];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        const float2 f = __half22float2(u32_as_h2(w[i]));
        b[2 * i] = __float_as_uint(fmaf(f.x, up, kMagic));
        b[2 * i + 1] = __float_as_uint(fmaf(f.y, up, kMagic));
    }
    uint32_t s4[4] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int i = 0; i < 32; ++i) s4[i & 3] += b[i];
    const uint32_t sum = (s4[0] + s4[1]) + (s4[2] + s4[3]) - 32u * 0x4B400000u;   // mod 2^32: |sum| < 2^20
    sx7 = 7 * static_cast<int>(sum);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const uint32_t* v = b + q * 8;
        xi[q][0] = __byte_perm(v[0], v[2], 0x5410);   // (x0, x2) as int16 pairs
        xi[q][1] = __byte_perm(v[4], v[6], 0x5410);
        xi[q][2] = __byte_perm(v[1], v[3], 0x5410);
        xi[q][3] = __byte_perm(v[5], v[7], 0x5410);
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
