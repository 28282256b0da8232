// dispatch_cost.cpp -- host cost of one C-ABI call (validation, dispatch on n,
// tensor-map lookup, launch), measured from C++ so no Python is in the loop
// ("must be << kernel time").  Calls are made while the
// stream is being captured into a CUDA graph, so nothing executes on the GPU
// and the number is pure host time per call; a second pass times the same
// calls launched eagerly (each call then also pays the driver's launch path).
//
// g++ -O2 -std=c++17 -I include -I /usr/local/cuda/include tools/dispatch_cost.cpp \
//     -L paper_2311_02103_b200 -lrelax_q4 -L /usr/local/cuda/lib64 -lcudart -Wl,-rpath,$PWD/paper_2311_02103_b200 \
//     -o tools/dispatch_cost
#include <chrono>
#include <cstdio>
#include <vector>

#include <cuda_runtime.h>

#include "relax_q4.h"

static double now_us() {
    using namespace std::chrono;
    return duration<double, std::micro>(steady_clock::now().time_since_epoch()).count();
}

int main() {
    struct Shape { int64_t n, K, N; const char* what; };
    const Shape shapes[] = {{1, 4096, 4096, "decode GEMV"}, {1, 4096, 11008, "decode GEMV"},
                            {8, 4096, 4096, "small-n TC (cluster split)"}, {512, 4096, 11008, "prefill TC"},
                            {4096, 4096, 4096, "prefill TC"}};
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    for (const Shape& s : shapes) {
        void *x, *w, *sc, *y;
        cudaMalloc(&x, s.n * s.K * 2);
        cudaMalloc(&w, s.N * s.K / 2);
        cudaMalloc(&sc, s.N * (s.K / 32) * 2);
        cudaMalloc(&y, s.n * s.N * 2);
        cudaMemset(w, 0x77, s.N * s.K / 2);
        cudaMemset(sc, 0, s.N * (s.K / 32) * 2);
        cudaMemset(x, 0, s.n * s.K * 2);
        // warm-up: first-call attribute setup and tensor-map cache fill
        int rc = relax_q4_matmul(x, s.n, s.K, s.N, static_cast<const uint32_t*>(w), sc, y, st);
        cudaStreamSynchronize(st);
        if (rc) { printf("rc=%d\n", rc); return 1; }
        const int calls = 2000;
        cudaGraph_t g;
        cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
        const double t0 = now_us();
        for (int i = 0; i < calls; ++i) relax_q4_matmul(x, s.n, s.K, s.N, static_cast<const uint32_t*>(w), sc, y, st);
        const double t1 = now_us();
        cudaStreamEndCapture(st, &g);
        cudaGraphDestroy(g);
        // eager: launches queue on the GPU (bounded batch so the queue does not fill)
        const int eager = 200;
        const double t2 = now_us();
        for (int i = 0; i < eager; ++i) relax_q4_matmul(x, s.n, s.K, s.N, static_cast<const uint32_t*>(w), sc, y, st);
        const double t3 = now_us();
        cudaStreamSynchronize(st);
        printf("n=%-5lld K=%-5lld N=%-6lld %-28s host per call: %.2f us (captured), %.2f us (eager enqueue)\n",
               (long long)s.n, (long long)s.K, (long long)s.N, s.what, (t1 - t0) / calls, (t3 - t2) / eager);
        cudaFree(x); cudaFree(w); cudaFree(sc); cudaFree(y);
    }
    return 0;
}
