// repack.cu -- one-time conversion of a stored int4 weight into the
// kernel-native format ("lift out quantization and layout
// transforms in tensor programs to enable pre-computation").
//
// Source formats (include/relax_q4.h RELAX_LAYOUT_*, readings 19-20):
//   NK: packed [N][K/8], scales [N][K/G]      KN: packed [K/8][N], scales [K/G][N]
//   NK3 (3-bit, zero point 3): packed [N][3 K/32] (32 codes per 96 bits), scales [N][K/G]
// with G in {32, 64, 128}; a word always holds the codes of 8 consecutive k of
// one output column, low nibble first.  Native: NK with G = 32.  The codes
// move unchanged and every 32-group takes the scale of the G-group holding
// it, so the repacked weight dequantizes to the same W bit for bit.
// Memory-bound and run once per weight: 32x32 shared-memory tiles keep both
// sides of the KN transposes coalesced.
#include "internal.h"

namespace rq4 {

constexpr int kTile = 32;

// out[j][c] = in[c][j] for a [R][C] -> [C][R] transpose of 32- or 16-bit
// elements; `rep` > 1 (scales) writes each input column c to output columns
// c*rep .. c*rep+rep-1 (group-size expansion).
template <typename T>
__global__ void __launch_bounds__(kTile * 8) transpose_rep_kernel(const T* __restrict__ in, int64_t R, int64_t C,
                                                                  int rep, T* __restrict__ out) {
    __shared__ T tile[kTile][kTile + 1];
    const int64_t c0 = static_cast<int64_t>(blockIdx.x) * kTile;
    const int64_t r0 = static_cast<int64_t>(blockIdx.y) * kTile;
    for (int i = threadIdx.y; i < kTile; i += blockDim.y) {
        const int64_t r = r0 + i, c = c0 + threadIdx.x;
        if (r < R && c < C) tile[i][threadIdx.x] = in[r * C + c];
    }
    __syncthreads();
    const int64_t ocols = R * rep;                          // output row length
    for (int i = threadIdx.y; i < kTile; i += blockDim.y) {
        const int64_t oc = c0 + i;                          // output row = input column
        const int64_t orr = r0 + threadIdx.x;               // input row
        if (oc < C && orr < R) {
            const T v = tile[threadIdx.x][i];
            for (int u = 0; u < rep; ++u) out[oc * ocols + orr * rep + u] = v;
        }
    }
}

// NK scales: out[j][c*rep + u] = in[j][c]
__global__ void __launch_bounds__(256) expand_rows_kernel(const uint16_t* __restrict__ in, int64_t rows, int64_t cols,
                                                          int rep, uint16_t* __restrict__ out) {
    const int64_t total = rows * cols * rep;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = i / (cols * rep);
        const int64_t c = (i - r * cols * rep) / rep;
        out[i] = in[r * cols + c];
    }
}

// 3-bit source (RELAX_LAYOUT_NK3): per (row, 32-group) three words hold the
// codes at bits 3 i .. 3 i + 2 of their 96 bits; the native word w (codes
// 8 w .. 8 w + 7) gets q4 = q3 + 4 (q4 - 7 == q3 - 3: the same W).
__global__ void __launch_bounds__(256) repack_q3_kernel(const uint32_t* __restrict__ in, int64_t groups,
                                                        uint32_t* __restrict__ out) {
    for (int64_t gi = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; gi < groups;
         gi += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const uint64_t lo = static_cast<uint64_t>(in[3 * gi]) | (static_cast<uint64_t>(in[3 * gi + 1]) << 32);
        const uint32_t hi = in[3 * gi + 2];
        uint32_t o[4];
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            uint32_t v = 0;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int bit = 3 * (8 * w + i);
                uint32_t q;
                if (bit + 3 <= 64) q = static_cast<uint32_t>(lo >> bit) & 7u;
                else if (bit >= 64) q = (hi >> (bit - 64)) & 7u;
                else q = (static_cast<uint32_t>(lo >> bit) | (hi << (64 - bit))) & 7u;   // straddles words 1 and 2
                v |= (q + 4u) << (4 * i);
            }
            o[w] = v;
        }
        reinterpret_cast<uint4*>(out)[gi] = make_uint4(o[0], o[1], o[2], o[3]);
    }
}

template <typename T>
static int launch_transpose(const T* in, int64_t R, int64_t C, int rep, T* out, cudaStream_t st) {
    const dim3 grid(static_cast<unsigned>((C + kTile - 1) / kTile), static_cast<unsigned>((R + kTile - 1) / kTile));
    transpose_rep_kernel<T><<<grid, dim3(kTile, 8), 0, st>>>(in, R, C, rep, out);
    return static_cast<int>(cudaGetLastError());
}

int launch_repack(const uint32_t* src_w, const uint16_t* src_s, int64_t K, int64_t N, int layout, int group,
                  uint32_t* w, uint16_t* s, cudaStream_t st) {
    const int rep = group / kGroup;
    int e;
    if (layout == 2) {                                   // 3-bit NK
        const int64_t groups = N * (K / kGroup);
        int64_t blocks = (groups + 255) / 256;
        const int64_t bmax = 8 * static_cast<int64_t>(num_sms());
        if (blocks > bmax) blocks = bmax;
        repack_q3_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(src_w, groups, w);
        e = static_cast<int>(cudaGetLastError());
        if (e) return e;
        const int64_t total = N * (K / kGroup);
        int64_t sblocks = (total + 255) / 256;
        if (sblocks > bmax) sblocks = bmax;
        expand_rows_kernel<<<static_cast<unsigned>(sblocks), 256, 0, st>>>(src_s, N, K / group, rep, s);
        return static_cast<int>(cudaGetLastError());
    }
    if (layout == 0) {
        e = static_cast<int>(cudaMemcpyAsync(w, src_w, static_cast<size_t>(N) * (K / 8) * 4, cudaMemcpyDeviceToDevice, st));
        if (e) return e;
        const int64_t total = N * (K / kGroup);
        int64_t blocks = (total + 255) / 256;
        const int64_t bmax = 8 * static_cast<int64_t>(num_sms());
        if (blocks > bmax) blocks = bmax;
        expand_rows_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(src_s, N, K / group, rep, s);
        return static_cast<int>(cudaGetLastError());
    }
    e = launch_transpose<uint32_t>(src_w, K / 8, N, 1, w, st);       // [K/8][N] -> [N][K/8]
    if (e) return e;
    return launch_transpose<uint16_t>(src_s, K / group, N, rep, s, st);   // [K/G][N] -> [N][K/32]
}

}  // namespace rq4
