// Memory-only ceiling for the dequantize access pattern (read N bytes, write 4N):
// same loads/stores as k_dequant_blocks with the arithmetic replaced by a copy.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <bool STREAM>
__global__ void __launch_bounds__(256) k_rw(const uint32_t* __restrict__ in, float4* __restrict__ out, size_t nblocks) {
    for (size_t b = blockIdx.x; b < nblocks; b += gridDim.x) {
        uint32_t w[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) w[k] = STREAM ? __ldcs(in + b * 1024 + threadIdx.x + k * 256) : in[b * 1024 + threadIdx.x + k * 256];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            float4 v = make_float4(__uint_as_float(w[k]), __uint_as_float(w[k] ^ 1u), __uint_as_float(w[k] ^ 2u), __uint_as_float(w[k] ^ 3u));
            if (STREAM) __stcs(out + b * 1024 + threadIdx.x + k * 256, v);
            else out[b * 1024 + threadIdx.x + k * 256] = v;
        }
    }
}

int main() {
    const size_t N = 1ull << 28, nb = N / 4096;
    uint32_t* in; float4* out;
    cudaMalloc(&in, N); cudaMalloc(&out, 4 * N);
    cudaMemset(in, 1, N);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int stream = 0; stream < 2; ++stream)
    for (int mult : {4, 6, 8, 16, 64}) {
        unsigned g = sms * mult;
        for (int i = 0; i < 3; ++i) stream ? k_rw<true><<<g, 256>>>(in, out, nb) : k_rw<false><<<g, 256>>>(in, out, nb);
        cudaEventRecord(a);
        for (int i = 0; i < 20; ++i) stream ? k_rw<true><<<g, 256>>>(in, out, nb) : k_rw<false><<<g, 256>>>(in, out, nb);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); ms /= 20;
        printf("stream=%d grid=%dx%d: %.1f us %.0f GB/s\n", stream, sms, mult, ms * 1e3, 5.0 * N / (ms * 1e-3) / 1e9);
    }
    return 0;
}
