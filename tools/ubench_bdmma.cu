// ubench_bdmma.cu -- math-rate probe for the "block-diagonal" warp-MMA decode
// GEMV (DESIGN.md §5.2, §10 item 1) against the FHFMA inner loop it would
// replace, both on shared-memory-resident codes (no HBM, no barriers):
//
//   fhfma: per lane one 32-code group of 4 rows per step (LDS.128 + LDS.U16 per
//          row, 1 SHF + 4 LOP3 + 8 FHFMA per word, scale FMAs), as in
//          gemv_stream.cu;
//   bdmma: per warp 16 rows x 8 groups per step: lane (g, t) loads word t of
//          group i for rows g and g + 8, masks them into fp16-subnormal pairs,
//          and 16 chained mma.sync m16n8k16 accumulate column i <- group i
//          (B zero outside the lane's own group column), then 4 FFMA apply the
//          per-(row, group) scales.
//
// Reports weights per clock per SM with 16 warps per CTA, one CTA per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_bdmma tools/ubench_bdmma.cu
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

constexpr int STEPS = 2048;
#ifndef WARPS_N
#define WARPS_N 16
#endif
constexpr int WARPS = WARPS_N;

__device__ __forceinline__ float fhfma(uint16_t a, uint16_t b, float c) {
    float d;
    asm volatile("fma.rn.f32.f16 %0, %1, %2, %3;" : "=f"(d) : "h"(a), "h"(b), "f"(c));
    return d;
}

__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// FHFMA loop: 4 rows x 32 codes per lane per step = 128 weights/lane/step.
__global__ void __launch_bounds__(WARPS * 32, 2) k_fhfma(float* out, long long* cyc, uint32_t seed) {
    __shared__ __align__(16) uint8_t sm[4 * 2048 + 4 * 256 + 256];     // 4 rows of K = 4096 codes + scales (+ step jitter)
    for (int i = threadIdx.x; i < (int)sizeof(sm) / 4; i += blockDim.x)
        reinterpret_cast<uint32_t*>(sm)[i] = seed * 2654435761u + i;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = (warp & 3) * 32 + lane;                          // group of this lane (K = 4096: 128 groups)
    uint32_t x[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = 0x3c003c00u ^ (seed + i);
    float acc = 0.f;
    long long t0 = clock64();
    for (int st = 0; st < STEPS; ++st) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int jit = (st & 7) * 16;      // defeats loop-invariant hoisting
            const uint4 cw = *reinterpret_cast<const uint4*>(sm + jit + r * 2048 + g * 16);
            const uint16_t sb = *reinterpret_cast<const uint16_t*>(sm + jit + 8192 + r * 256 + g * 2);
            const uint32_t w[4] = {cw.x, cw.y, cw.z, cw.w};
            float e = 0.f, o = 0.f;
#pragma unroll
            for (int wi = 0; wi < 4; ++wi) {
                const uint32_t v8 = w[wi] >> 8;
                const uint32_t c0 = w[wi] & 0x000F000Fu, c1 = w[wi] & 0x00F000F0u;
                const uint32_t c2 = v8 & 0x000F000Fu, c3 = v8 & 0x00F000F0u;
                const uint32_t X0 = x[wi * 4], X1 = x[wi * 4 + 1], X2 = x[wi * 4 + 2], X3 = x[wi * 4 + 3];
                e = fhfma((uint16_t)c0, (uint16_t)X0, e);  o = fhfma((uint16_t)c1, (uint16_t)(X0 >> 16), o);
                e = fhfma((uint16_t)c2, (uint16_t)X1, e);  o = fhfma((uint16_t)c3, (uint16_t)(X1 >> 16), o);
                e = fhfma((uint16_t)(c0 >> 16), (uint16_t)X2, e);  o = fhfma((uint16_t)(c1 >> 16), (uint16_t)(X2 >> 16), o);
                e = fhfma((uint16_t)(c2 >> 16), (uint16_t)X3, e);  o = fhfma((uint16_t)(c3 >> 16), (uint16_t)(X3 >> 16), o);
            }
            acc = fmaf(__half2float(__ushort_as_half(sb)), fmaf(o, 0.0625f, e), acc);
        }
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// Block-diagonal MMA loop: 16 rows x 8 groups (4096 weights) per warp per step.
// V adds the real kernel's per-step overheads one at a time:
//   V >= 1: the 128-B-swizzled stage addressing of gemv_mma.cu (jj ^ g)
//   V >= 2: quad-shuffle row reduction + partial-sum read-modify-write in SMEM
//   V >= 3: an mbarrier try_wait (already complete) + arrive per step
template <int V>
__global__ void __launch_bounds__(WARPS * 32, 2) k_bdmma(float* out, long long* cyc, uint32_t seed) {
    // 16 rows x 8 groups x 16 B codes, padded row stride 144 B (conflict-free), + scales
    __shared__ __align__(16) uint8_t sm[16 * 144 + 16 * 16 + 128];
    __shared__ float part[16 * WARPS];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"((uint32_t)__cvta_generic_to_shared(&bar)), "r"((1 << 20) - 1));
    }
    for (int i = threadIdx.x; i < (int)sizeof(sm) / 4; i += blockDim.x)
        reinterpret_cast<uint32_t*>(sm)[i] = seed * 2654435761u + i;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const uint32_t xa = 0x3c003c00u ^ seed, xb = 0x3c003c00u ^ (seed * 3);
    float y0 = 0.f, y1 = 0.f;
    long long t0 = clock64();
    for (int st = 0; st < STEPS; ++st) {
        float dd[4][4] = {};                                      // 4 independent MMA chains
        const int jit = (st & 7) * 16;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int off = V >= 1 ? (((i ^ g) & 7) * 16) : i * 16;
            const uint32_t wa = *reinterpret_cast<const uint32_t*>(sm + jit + g * 144 + off + t * 4);
            const uint32_t wb = *reinterpret_cast<const uint32_t*>(sm + jit + (g + 8) * 144 + off + t * 4);
            const uint32_t wa8 = wa >> 8, wb8 = wb >> 8;
            const uint32_t a1[4] = {wa & 0x000F000Fu, wb & 0x000F000Fu, wa8 & 0x000F000Fu, wb8 & 0x000F000Fu};
            const uint32_t a2[4] = {wa & 0x00F000F0u, wb & 0x00F000F0u, wa8 & 0x00F000F0u, wb8 & 0x00F000F0u};
            const bool mine = g == i;                                 // this lane's B column is group i
            mma16816(dd[(2 * i) & 3], a1, mine ? xa : 0u, mine ? xb : 0u);
            mma16816(dd[(2 * i + 1) & 3], a2, mine ? xb : 0u, mine ? xa : 0u);
        }
        float d[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) d[q] = (dd[0][q] + dd[1][q]) + (dd[2][q] + dd[3][q]);
        const uint32_t sa = *reinterpret_cast<const uint32_t*>(sm + jit + 16 * 144 + g * 16 + t * 4);
        const uint32_t sb = *reinterpret_cast<const uint32_t*>(sm + jit + 16 * 144 + (g + 8) * 16 + t * 4);
        const float2 fa = __half22float2(*reinterpret_cast<const __half2*>(&sa));
        const float2 fb = __half22float2(*reinterpret_cast<const __half2*>(&sb));
        float r0 = fa.x * d[0] + fa.y * d[1], r1 = fb.x * d[2] + fb.y * d[3];
        if (V >= 2) {
            r0 += __shfl_xor_sync(0xffffffffu, r0, 1); r0 += __shfl_xor_sync(0xffffffffu, r0, 2);
            r1 += __shfl_xor_sync(0xffffffffu, r1, 1); r1 += __shfl_xor_sync(0xffffffffu, r1, 2);
            if (t == 0) {
                float* p = &part[(threadIdx.x >> 5) * 16 + g];
                *p = (st & 1) ? *p + r0 : r0;
                p[8] = (st & 1) ? p[8] + r1 : r1;
            }
        }
        if (V >= 3) {
            const uint32_t ba = (uint32_t)__cvta_generic_to_shared(&bar);
            uint32_t ok;
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                         : "=r"(ok) : "r"(ba), "r"(1u) : "memory");
            __syncwarp();
            if (lane == 0) asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" :: "r"(ba) : "memory");
            y0 += (float)ok;
        }
        y0 += r0;
        y1 += r1;
    }
    y0 += __shfl_xor_sync(0xffffffffu, y0, 1);
    y0 += __shfl_xor_sync(0xffffffffu, y0, 2);
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = y0 + y1;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// All overheads, but two 8-group windows (8192 weights) per warp step and
// precomputed stage offsets: the amortised design.
__global__ void __launch_bounds__(WARPS * 32, 2) k_bdmma2(float* out, long long* cyc, uint32_t seed) {
    __shared__ __align__(16) uint8_t sm[16 * 272 + 16 * 32 + 128];
    __shared__ float part[16 * WARPS];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"((uint32_t)__cvta_generic_to_shared(&bar)), "r"((1 << 20) - 1));
    }
    for (int i = threadIdx.x; i < (int)sizeof(sm) / 4; i += blockDim.x)
        reinterpret_cast<uint32_t*>(sm)[i] = seed * 2654435761u + i;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const uint32_t xa = 0x3c003c00u ^ seed, xb = 0x3c003c00u ^ (seed * 3);
    int offs[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) offs[i] = g * 272 + (((i & 7) ^ g) + (i >> 3) * 8) * 16 + t * 4;   // precomputed
    float y0 = 0.f, y1 = 0.f;
    long long t0 = clock64();
    for (int st = 0; st < STEPS; ++st) {
        const int jit = (st & 7) * 16;
        float r0 = 0.f, r1 = 0.f;
#pragma unroll
        for (int w = 0; w < 2; ++w) {
            float dd[4][4] = {};
#pragma unroll
            for (int ii = 0; ii < 8; ++ii) {
                const int i = w * 8 + ii;
                const uint32_t wa = *reinterpret_cast<const uint32_t*>(sm + jit + offs[i]);
                const uint32_t wb = *reinterpret_cast<const uint32_t*>(sm + jit + offs[i] + 8 * 272);
                const uint32_t wa8 = wa >> 8, wb8 = wb >> 8;
                const uint32_t a1[4] = {wa & 0x000F000Fu, wb & 0x000F000Fu, wa8 & 0x000F000Fu, wb8 & 0x000F000Fu};
                const uint32_t a2[4] = {wa & 0x00F000F0u, wb & 0x00F000F0u, wa8 & 0x00F000F0u, wb8 & 0x00F000F0u};
                const bool mine = g == ii;
                mma16816(dd[(2 * ii) & 3], a1, mine ? xa : 0u, mine ? xb : 0u);
                mma16816(dd[(2 * ii + 1) & 3], a2, mine ? xb : 0u, mine ? xa : 0u);
            }
            float d[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) d[q] = (dd[0][q] + dd[1][q]) + (dd[2][q] + dd[3][q]);
            const uint32_t sa = *reinterpret_cast<const uint32_t*>(sm + jit + 16 * 272 + g * 32 + w * 16 + t * 4);
            const uint32_t sb = *reinterpret_cast<const uint32_t*>(sm + jit + 16 * 272 + (g + 8) * 32 + w * 16 + t * 4);
            const float2 fa = __half22float2(*reinterpret_cast<const __half2*>(&sa));
            const float2 fb = __half22float2(*reinterpret_cast<const __half2*>(&sb));
            r0 = fmaf(fa.x, d[0], fmaf(fa.y, d[1], r0));
            r1 = fmaf(fb.x, d[2], fmaf(fb.y, d[3], r1));
        }
        r0 += __shfl_xor_sync(0xffffffffu, r0, 1); r0 += __shfl_xor_sync(0xffffffffu, r0, 2);
        r1 += __shfl_xor_sync(0xffffffffu, r1, 1); r1 += __shfl_xor_sync(0xffffffffu, r1, 2);
        if (t == 0) {
            float* p = &part[(threadIdx.x >> 5) * 16 + g];
            *p = (st & 1) ? *p + r0 : r0;
            p[8] = (st & 1) ? p[8] + r1 : r1;
        }
        const uint32_t ba = (uint32_t)__cvta_generic_to_shared(&bar);
        uint32_t ok;
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(ok) : "r"(ba), "r"(1u) : "memory");
        __syncwarp();
        if (lane == 0) asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" :: "r"(ba) : "memory");
        y0 += r0 + (float)ok;
        y1 += r1;
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = y0 + y1;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
    float* out;
    long long* cyc;
    cudaMalloc(&out, 148 * 1024 * 4);
    cudaMalloc(&cyc, 148 * 8);
    long long c[148];
    const char* names[] = {"fhfma (gemv_stream loop)", "bdmma", "bdmma + swizzled addressing",
                           "bdmma + swizzle + quad reduce + partial RMW", "bdmma + all + mbarrier wait/arrive", "bdmma, all overheads, 2 windows/step + precomputed offsets"};
    for (int v = 0; v < 6; ++v) {
        for (int rep = 0; rep < 2; ++rep) {
            if (v == 0) k_fhfma<<<148, WARPS * 32>>>(out, cyc, 7);
            else if (v == 1) k_bdmma<0><<<148, WARPS * 32>>>(out, cyc, 7);
            else if (v == 2) k_bdmma<1><<<148, WARPS * 32>>>(out, cyc, 7);
            else if (v == 3) k_bdmma<2><<<148, WARPS * 32>>>(out, cyc, 7);
            else if (v == 4) k_bdmma<3><<<148, WARPS * 32>>>(out, cyc, 7);
            else k_bdmma2<<<148, WARPS * 32>>>(out, cyc, 7);
            cudaDeviceSynchronize();
        }
        cudaMemcpy(c, cyc, sizeof c, cudaMemcpyDeviceToHost);
        long long mx = 0;
        for (int i = 0; i < 148; ++i) mx = c[i] > mx ? c[i] : mx;
        const double w = v == 0 ? (double)STEPS * 4 * 32 * 32 * WARPS      // 4 rows x 32 codes x 32 lanes per warp-step
                        : v == 5 ? (double)STEPS * 16 * 512 * WARPS         // 16 rows x 512 codes per warp-step
                                 : (double)STEPS * 16 * 256 * WARPS;        // 16 rows x 256 codes per warp-step
        printf("%s: %.1f weights/clk/SM (%s)\n", names[v],
               w / mx, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
