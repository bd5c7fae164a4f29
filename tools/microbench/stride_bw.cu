// stride_bw.cu — HBM read+write bandwidth of the column-pass access pattern.
// Each CTA walks `rows` chunks of W bytes spaced `stride` bytes apart (the
// quad-layout column pair at 4096^2: W = 32 B, stride = 64 KiB), reading them
// and writing them back, as the fused column pass does.  Compared with a
// contiguous stream of the same total bytes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stride_bw stride_bw.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int W>
__global__ void k_strided(const char* __restrict__ in, char* __restrict__ out, size_t stride, int rows,
                          int chunks_per_row) {
    // CTA -> (target, chunk index within the row); threads walk rows
    constexpr int V = W / 16;  // float4 per chunk
    const size_t cta = blockIdx.x;
    const size_t target = cta / chunks_per_row, ch = cta % chunks_per_row;
    const char* base = in + target * stride * rows + ch * W;
    char* obase = out + target * stride * rows + ch * W;
    for (int i = threadIdx.x; i < rows * V; i += blockDim.x) {
        const int r = i / V, v = i % V;
        float4 x = *reinterpret_cast<const float4*>(base + r * stride + v * 16);
        x.x += 1.f;
        *reinterpret_cast<float4*>(obase + r * stride + v * 16) = x;
    }
}

__global__ void k_stream(const float4* __restrict__ in, float4* __restrict__ out, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        float4 x = in[i];
        x.x += 1.f;
        out[i] = x;
    }
}

int main() {
    const size_t row_bytes = 4096ull * 2 * 8;  // one quad row of a 4096^2 complex64 field: 64 KiB
    const int rows = 2048, targets = 16;
    const size_t bytes = row_bytes * rows * targets;  // 2 GiB
    char *a, *b;
    cudaMalloc(&a, bytes);
    cudaMalloc(&b, bytes);
    cudaMemset(a, 0, bytes);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto time = [&](auto f) {
        f();
        cudaEventRecord(e0);
        for (int r = 0; r < 5; ++r) f();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        return ms / 5;
    };
    float ms = time([&] { k_stream<<<148 * 8, 512>>>((float4*)a, (float4*)b, bytes / 16); });
    printf("contiguous stream          : %7.1f GB/s (R+W)\n", 2.0 * bytes / ms / 1e6);
    float m32 = time([&] { k_strided<32><<<targets * (row_bytes / 32), 256>>>(a, b, row_bytes, rows, row_bytes / 32); });
    printf("32 B chunks @ 64 KiB stride: %7.1f GB/s\n", 2.0 * bytes / m32 / 1e6);
    float m64 = time([&] { k_strided<64><<<targets * (row_bytes / 64), 256>>>(a, b, row_bytes, rows, row_bytes / 64); });
    printf("64 B chunks @ 64 KiB stride: %7.1f GB/s\n", 2.0 * bytes / m64 / 1e6);
    float m128 = time([&] { k_strided<128><<<targets * (row_bytes / 128), 256>>>(a, b, row_bytes, rows, row_bytes / 128); });
    printf("128B chunks @ 64 KiB stride: %7.1f GB/s\n", 2.0 * bytes / m128 / 1e6);
    float m256 = time([&] { k_strided<256><<<targets * (row_bytes / 256), 256>>>(a, b, row_bytes, rows, row_bytes / 256); });
    printf("256B chunks @ 64 KiB stride: %7.1f GB/s\n", 2.0 * bytes / m256 / 1e6);
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
