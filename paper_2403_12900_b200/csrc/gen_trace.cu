// gen_trace.cu -- HARNESS ONLY (not part of the method): the synthetic
// Llama2-shaped request trace, generated in place on the device from global
// request indices (so a shard never moves data).  Same integer recipe as
// synth.gen_tokens (numpy): one Philox4x32-10 call per request on stream 1,
// counter = (g lo32, g hi32, 1, 0); L0 tokens from a 4096-entry quantile
// table, level i >= 1 = max(1, (tok0 * ratio_i[byte]) >> 16); class and
// opted-out flag from word 3.
#include "sprout_device.cuh"
#include "sprout_kernels.cuh"

namespace sprout {

template <int N>
__global__ void __launch_bounds__(256) gen_kernel(GenArgs a) {
    const int64_t groups = a.pitch / 8;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < groups; v += (int64_t)gridDim.x * blockDim.x) {
        uint32_t tw[N][4];
        uint32_t fw[2] = {0u, 0u};
#pragma unroll
        for (int i = 0; i < N; ++i)
#pragma unroll
            for (int q = 0; q < 4; ++q) tw[i][q] = 0u;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int64_t r = v * 8 + k;
            if (r >= a.n_requests) continue;
            const uint64_t g = a.first_request + (uint64_t)r;
            const Philox4 w = philox4x32_10((uint32_t)g, (uint32_t)(g >> 32), 1u, 0u, (uint32_t)a.gen_seed,
                                            (uint32_t)(a.gen_seed >> 32));
            const uint32_t cls = (uint32_t)(((uint64_t)(w.v[3] >> 16) * (uint32_t)a.NC) >> 16);
            const uint32_t tok0 = a.q0_table[cls * 4096u + (w.v[0] >> 20)];
            const int sh = 16 * (k & 1);
            tw[0][k >> 1] |= tok0 << sh;
#pragma unroll
            for (int i = 1; i < N; ++i) {
                const uint32_t src = i <= 4 ? w.v[1] : w.v[2];
                const uint32_t byte = (src >> (8 * (i <= 4 ? i - 1 : i - 5))) & 0xFFu;
                uint32_t t = (tok0 * (uint32_t)a.ratio_table[i * 256 + byte]) >> 16;
                t = t < 1u ? 1u : t;
                tw[i][k >> 1] |= t << sh;
            }
            const uint32_t pinned = (w.v[3] & 0xFFFFFFu) < a.pin_thresh ? 1u : 0u;
            fw[k >> 2] |= (pinned | (cls << 1)) << (8 * (k & 3));
        }
#pragma unroll
        for (int i = 0; i < N; ++i)
            reinterpret_cast<uint4 *>(a.tokens + (size_t)i * a.pitch)[v] = make_uint4(tw[i][0], tw[i][1], tw[i][2], tw[i][3]);
        if (a.flags) reinterpret_cast<uint2 *>(a.flags)[v] = make_uint2(fw[0], fw[1]);
    }
}

cudaError_t launch_generate(const GenArgs &a, cudaStream_t stream, int *launches) {
    const int64_t groups = a.pitch / 8;
    if (groups == 0) return cudaSuccess;
    int64_t blocks = (groups + 255) / 256;
    if (blocks > 148 * 32) blocks = 148 * 32;
    switch (a.n) {
#define GEN_CASE(NN) case NN: gen_kernel<NN><<<(unsigned)blocks, 256, 0, stream>>>(a); break;
        GEN_CASE(1) GEN_CASE(2) GEN_CASE(3) GEN_CASE(4) GEN_CASE(5) GEN_CASE(6) GEN_CASE(7) GEN_CASE(8)
#undef GEN_CASE
        default: return cudaErrorInvalidValue;
    }
    ++*launches;
    return cudaGetLastError();
}

}  // namespace sprout
