// ubench_mma.cu -- (1) warp-level mma.sync m16n8k16 f16 x f16 -> f32 issue
// throughput per SM on sm_100a, alone and mixed with the LOP3 unpack it would
// need in a decode GEMV; (2) exactness of fp16 SUBNORMAL A operands
// (codes q * 2^-24, the factored-zero-point encoding) through the tensor
// core: D must equal sum_k q_k 2^-24 x_k up to fp32 accumulation rounding.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_mma tools/ubench_mma.cu
#include <cmath>
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

constexpr int ITERS = 2048;

__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

// OP 0: MMA only (8 independent accumulators); OP k>0: MMA + k LOP3.
template <int OP>
__global__ void kern(float* out, uint32_t seed, long long* cycles) {
    float d[8][4];
    uint32_t a[4], b[2], u[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) { d[i][0] = d[i][1] = d[i][2] = d[i][3] = 0.f; u[i] = seed * (i + 3) + threadIdx.x; }
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = 0x00050003u + i;
    b[0] = 0x3c003c00u; b[1] = 0x3c003c00u ^ seed;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            mma16816(d[i], a, b);
#pragma unroll
            for (int j = 0; j < OP; ++j)
                asm volatile("lop3.b32 %0, %0, %1, %2, 0xea;" : "+r"(u[(i + j) & 7]) : "r"(seed), "r"(b[1]));
        }
    }
    long long t1 = clock64();
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += d[i][0] + d[i][1] + d[i][2] + d[i][3] + (float)u[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

__global__ void exact_kern(const uint16_t* A, const uint16_t* B, float* D) {
    // A [16][16] row-major, B [16 k][8 n], D [16][8]
    const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
    auto pk = [](uint16_t lo, uint16_t hi) { return (uint32_t)lo | ((uint32_t)hi << 16); };
    uint32_t a[4] = {pk(A[g * 16 + 2 * t], A[g * 16 + 2 * t + 1]), pk(A[(g + 8) * 16 + 2 * t], A[(g + 8) * 16 + 2 * t + 1]),
                     pk(A[g * 16 + 2 * t + 8], A[g * 16 + 2 * t + 9]), pk(A[(g + 8) * 16 + 2 * t + 8], A[(g + 8) * 16 + 2 * t + 9])};
    uint32_t b[2] = {pk(B[(2 * t) * 8 + g], B[(2 * t + 1) * 8 + g]), pk(B[(2 * t + 8) * 8 + g], B[(2 * t + 9) * 8 + g])};
    float d[4] = {0.f, 0.f, 0.f, 0.f};
    mma16816(d, a, b);
    D[g * 8 + 2 * t] = d[0]; D[g * 8 + 2 * t + 1] = d[1];
    D[(g + 8) * 8 + 2 * t] = d[2]; D[(g + 8) * 8 + 2 * t + 1] = d[3];
}

static double h2d(uint16_t h) { __half_raw r; r.x = h; return (double)__half2float(__half(r)); }

int main() {
    float* out;
    long long* cyc;
    cudaMalloc(&out, 148 * 1024 * 4);
    cudaMalloc(&cyc, 148 * 8);
    for (int op : {0, 2, 4, 5, 6, 8}) {
        for (int threads : {256, 512}) {
            auto launch = [&] {
                switch (op) {
                    case 0: kern<0><<<148, threads>>>(out, 7, cyc); break;
                    case 2: kern<2><<<148, threads>>>(out, 7, cyc); break;
                    case 4: kern<4><<<148, threads>>>(out, 7, cyc); break;
                    case 5: kern<5><<<148, threads>>>(out, 7, cyc); break;
                    case 6: kern<6><<<148, threads>>>(out, 7, cyc); break;
                    default: kern<8><<<148, threads>>>(out, 7, cyc); break;
                }
            };
            launch(); cudaDeviceSynchronize();
            launch(); cudaDeviceSynchronize();
            long long c[148];
            cudaMemcpy(c, cyc, sizeof c, cudaMemcpyDeviceToHost);
            long long mx = 0;
            for (int i = 0; i < 148; ++i) mx = c[i] > mx ? c[i] : mx;
            const double nmma = (double)ITERS * 8 * threads / 32;
            printf("MMA + %d LOP3  threads=%4d  mma/clk/SM = %.3f  (dense f16 FMA/clk/SM = %.0f)  total warp-inst/clk/SM = %.2f\n",
                   op, threads, nmma / mx, nmma * 2048 / mx, nmma * (1 + op) / mx);
        }
    }
    // exactness with subnormal A
    uint16_t hA[256], hB[128];
    uint32_t st = 12345;
    auto rnd = [&] { st = st * 1664525u + 1013904223u; return st >> 8; };
    double maxrel = 0, maxabs_ulp = 0;
    int zero_hits = 0;
    uint16_t *dA, *dB;
    float* dD;
    cudaMalloc(&dA, sizeof hA); cudaMalloc(&dB, sizeof hB); cudaMalloc(&dD, 128 * 4);
    for (int trial = 0; trial < 200; ++trial) {
        for (int i = 0; i < 256; ++i) hA[i] = (uint16_t)(rnd() & 15u) << ((trial & 1) ? 4 : 0);   // q*2^-24 or q*2^-20
        for (int i = 0; i < 128; ++i) {
            float v = ((int)(rnd() % 20001) - 10000) / 997.0f;
            __half hv = __float2half_rn(v);
            std::memcpy(&hB[i], &hv, 2);
        }
        cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice);
        cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
        exact_kern<<<1, 32>>>(dA, dB, dD);
        float hD[128];
        cudaMemcpy(hD, dD, sizeof hD, cudaMemcpyDeviceToHost);
        for (int m = 0; m < 16; ++m)
            for (int n = 0; n < 8; ++n) {
                double e = 0, mag = 0;
                for (int k = 0; k < 16; ++k) {
                    const double p = h2d(hA[m * 16 + k]) * h2d(hB[k * 8 + n]);
                    e += p; mag += std::fabs(p);
                }
                const double err = std::fabs((double)hD[m * 8 + n] - e);
                if (mag > 0) maxrel = std::fmax(maxrel, err / mag);
                if (mag > 0 && hD[m * 8 + n] == 0.f && e != 0) ++zero_hits;
                (void)maxabs_ulp;
            }
    }
    printf("subnormal-A exactness: max |D - exact| / sum|products| = %.3g (fp32 ulp 2^-23 = %.3g); flushed-to-zero results: %d\n",
           maxrel, std::ldexp(1.0, -23), zero_hits);
    return 0;
}
