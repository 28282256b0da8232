// ubench_mma_sync.cu -- legacy warp-level MMA on sm_100a: latency (one
// dependent chain per warp) and throughput (8 independent chains per warp, 16
// warps per SM) of
//   HMMA  mma.sync.m16n8k16.f32.f16.f16.f32   (4096 MAC)
//   IMMA  mma.sync.m16n8k32.s32.u8.s8.s32     (8192 MAC)
// -- whether an integer small-batch kernel (codes as u8, 16-bit x split into
// two byte MMAs, zero point exact in integers) could replace the fp16 one.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubm tools/ubench_mma_sync.cu && /tmp/ubm
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int CH>
__global__ void hmma_k(float* out, int iters) {
    uint32_t a[4] = {threadIdx.x, threadIdx.x * 3u, threadIdx.x * 5u, threadIdx.x * 7u};
    uint32_t b0 = threadIdx.x * 11u, b1 = threadIdx.x * 13u;
    float d[CH][4] = {};
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < CH; ++c)
            asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                         "{%0,%1,%2,%3};"
                         : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
                         : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
    }
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int CH>
__global__ void imma_k(int* out, int iters) {
    uint32_t a[4] = {threadIdx.x, threadIdx.x * 3u, threadIdx.x * 5u, threadIdx.x * 7u};
    uint32_t b0 = threadIdx.x * 11u, b1 = threadIdx.x * 13u;
    int d[CH][4] = {};
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < CH; ++c)
            asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                         "{%0,%1,%2,%3};"
                         : "+r"(d[c][0]), "+r"(d[c][1]), "+r"(d[c][2]), "+r"(d[c][3])
                         : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
    }
    int s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename K, typename T>
static void run(const char* name, K kern, T* out, int blocks, int threads, int iters, int chains, double macs) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    kern<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e0);
    kern<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    int dev = 0, clk = 0, sms = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const double n_mma = static_cast<double>(blocks) * (threads / 32) * iters * chains;
    const double cyc = ms * 1e-3 * clk * 1e3;
    printf("%-34s %8.3f ms  %7.2f clk per MMA per warp-chain  %8.1f TOPS (dense MAC*2)  %6.1f MMA/clk/SM\n", name, ms,
           cyc / (iters), 2.0 * macs * n_mma / (ms * 1e-3) / 1e12, n_mma / cyc / (blocks < sms ? blocks : sms));
}

int main() {
    float* of;
    int* oi;
    cudaMalloc(&of, 1 << 24);
    cudaMalloc(&oi, 1 << 24);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int it = 4096;
    run("HMMA 16816 latency (1 warp, 1 chain)", hmma_k<1>, of, 1, 32, it, 1, 4096.0);
    run("IMMA 16832 latency (1 warp, 1 chain)", imma_k<1>, oi, 1, 32, it, 1, 8192.0);
    run("HMMA 16816 throughput (16 w x 8 ch)", hmma_k<8>, of, sms, 512, it, 8, 4096.0);
    run("IMMA 16832 throughput (16 w x 8 ch)", imma_k<8>, oi, sms, 512, it, 8, 8192.0);
    cudaError_t e = cudaDeviceSynchronize();
    printf("status: %s\n", cudaGetErrorString(e));
    return 0;
}
