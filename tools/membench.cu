// membench.cu -- read-bandwidth ceilings on this B200 for the access patterns
// the GEMV uses (not part of the product library).
//   ldg     : grid-stride LDG.128 (ld.global.nc.L1::no_allocate), U loads in
//             flight per thread, XOR-reduced so the loads are not dead
//   bulk    : one CTA per SM, one producer thread streaming contiguous chunks
//             through an SMEM ring with cp.async.bulk; consumers only touch
//             one word per stage (pure transport ceiling)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/membench tools/membench.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint4 ldnc(const uint4* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}

template <int U>
__global__ void ldg_kernel(const uint4* __restrict__ src, size_t n16, uint32_t* out) {
    uint32_t acc = 0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + (U - 1) * stride < n16; i += U * stride) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = ldnc(src + i + u * stride);
#pragma unroll
        for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
    }
    for (; i < n16; i += stride) { uint4 v = ldnc(src + i); acc ^= v.x ^ v.y ^ v.z ^ v.w; }
    if (acc == 0x12345678u) out[0] = acc;
}

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void bulk_kernel(const uint8_t* __restrict__ src, size_t bytes, int stage_bytes, int NS, uint32_t* out) {
    extern __shared__ __align__(128) uint8_t sm[];
    uint64_t* full = (uint64_t*)sm;
    uint64_t* empty = full + NS;
    uint8_t* ring = sm + 128;
    const size_t per = (bytes / gridDim.x) / stage_bytes * stage_bytes;
    const uint8_t* base = src + per * blockIdx.x;
    const int nst = (int)(per / stage_bytes);
    const int nwc = (blockDim.x / 32) - 1;
    if (threadIdx.x == 0) {
        for (int i = 0; i < NS; ++i) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(su32(&full[i])), "r"(1));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(su32(&empty[i])), "r"(nwc));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
    auto wait = [](uint64_t* b, uint32_t ph) {
        uint32_t d = 0;
        while (!d) asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}" : "=r"(d) : "r"(su32(b)), "r"(ph) : "memory");
    };
    if (warp == nwc) {
        if (lane == 0) {
            uint64_t pol;
            asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
            for (int s = 0; s < nst; ++s) {
                int slot = s % NS;
                wait(&empty[slot], ((s / NS) & 1) ^ 1);
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su32(&full[slot])), "r"(stage_bytes) : "memory");
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                             :: "r"(su32(ring + (size_t)slot * stage_bytes)), "l"(base + (size_t)s * stage_bytes), "r"(stage_bytes), "r"(su32(&full[slot])), "l"(pol) : "memory");
            }
        }
    } else {
        uint32_t acc = 0;
        for (int s = 0; s < nst; ++s) {
            int slot = s % NS;
            wait(&full[slot], (s / NS) & 1);
            acc ^= ((const uint32_t*)(ring + (size_t)slot * stage_bytes))[threadIdx.x];
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(su32(&empty[slot])) : "memory");
        }
        if (acc == 0x12345678u) out[0] = acc;
    }
}

int main(int argc, char** argv) {
    const size_t bytes = (size_t)2 << 30;   // 2 GiB >> L2
    uint8_t* buf;
    uint32_t* out;
    CK(cudaMalloc(&buf, bytes));
    CK(cudaMalloc(&out, 64));
    CK(cudaMemset(buf, 1, bytes));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto timeit = [&](auto launch, const char* name) {
        for (int i = 0; i < 3; ++i) launch();
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        const int reps = 10;
        for (int i = 0; i < reps; ++i) launch();
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("%-40s %8.1f GB/s\n", name, bytes * (double)reps / (ms * 1e-3) / 1e9);
    };
    const size_t n16 = bytes / 16;
    for (int blocksPerSM : {4}) {
        for (int threads : {512}) {
            char nm[128];
            snprintf(nm, sizeof nm, "ldg U=8 grid=148x%d thr=%d", blocksPerSM, threads);
            timeit([&] { ldg_kernel<8><<<148 * blocksPerSM, threads>>>((const uint4*)buf, n16, out); }, nm);
        }
    }
    timeit([&] { ldg_kernel<16><<<148 * 4, 256>>>((const uint4*)buf, n16, out); }, "ldg U=16 grid=148x4 thr=256");
    for (int sb : {8192, 16384, 32768, 65536}) {
        for (int ns : {2, 4, 8}) {
            size_t smem = 128 + (size_t)sb * ns;
            if (smem > 227 * 1024) continue;
            CK(cudaFuncSetAttribute(bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
            char nm[128];
            snprintf(nm, sizeof nm, "bulk stage=%dK NS=%d ring=%zuK", sb / 1024, ns, (size_t)sb * ns / 1024);
            timeit([&] { bulk_kernel<<<148, 256, smem>>>(buf, bytes, sb, ns, out); }, nm);
        }
    }
    for (int cps : {2}) {
        size_t sb = 16384; int ns = 6;
        size_t smem = 128 + sb * ns;
        char nm[128];
        snprintf(nm, sizeof nm, "bulk 2 CTA/SM stage=16K NS=6");
        timeit([&] { bulk_kernel<<<148 * cps, 256, smem>>>(buf, bytes, (int)sb, ns, out); }, nm);
    }
    return 0;
}
