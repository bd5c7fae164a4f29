// Throughput of scalar vs packed FP32 (FADD/FFMA vs FADD2/FFMA2) on sm_100a.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 f32x2_tput.cu -o f32x2_tput
// Each thread runs 8 independent chains; prints lane-ops per clock per SM.
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 4096
typedef unsigned long long u64;

__device__ __forceinline__ u64 pk(float a, float b) {
    u64 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}

__global__ void k_fadd(float* out, float s) {
    float a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i;
    float b = s, c = s * 0.5f;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = a[i] + ((i & 1) ? b : c);
    }
    float r = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) r += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
__global__ void k_ffma(float* out, float s) {
    float a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i;
    float b = s, c = s * 0.5f;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], b, c);
    }
    float r = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) r += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
__global__ void k_fadd2(float* out, float s) {
    u64 a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = pk(threadIdx.x * 1e-3f + i, i * 2.f);
    u64 b = pk(s, s * 0.25f);
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(a[i]) : "l"(b));
    }
    float r = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        float x, y;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(a[i]));
        r += x + y;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
__global__ void k_ffma2(float* out, float s) {
    u64 a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = pk(threadIdx.x * 1e-3f + i, i * 2.f);
    u64 b = pk(s, s * 0.25f), c = pk(s * 0.5f, s * 0.125f);
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[i]) : "l"(b), "l"(c));
    }
    float r = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        float x, y;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(a[i]));
        r += x + y;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
// mixed: 4 FADD2 + 4 IADD-ish ALU ops interleaved (does ALU co-issue with packed FP?)
__global__ void k_fadd2_alu(float* out, float s) {
    u64 a[4];
    unsigned k[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) { a[i] = pk(threadIdx.x * 1e-3f + i, i * 2.f); k[i] = threadIdx.x * (i + 1); }
    u64 b = pk(s, s * 0.25f);
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(a[i]) : "l"(b));
            asm volatile("xor.b32 %0, %0, %1;" : "+r"(k[i]) : "r"(it));
        }
    }
    float r = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        float x, y;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(a[i]));
        r += x + y + k[i];
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

int main() {
    int sms, clk;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    float* out;
    const int threads = 512, blocks = sms * 4;
    cudaMalloc(&out, sizeof(float) * threads * blocks);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    struct K { const char* name; void (*f)(float*, float); double lane_ops; double instrs; };
    K ks[] = {{"FADD", k_fadd, 8, 8}, {"FFMA", k_ffma, 8, 8}, {"FADD2", k_fadd2, 16, 8}, {"FFMA2", k_ffma2, 16, 8},
              {"FADD2+LOP", k_fadd2_alu, 8, 8}};
    for (auto& k : ks) {
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(e0);
            k.f<<<blocks, threads>>>(out, 1.0001f);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
        }
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double cycles = ms * 1e-3 * clk * 1e3;  // at the nominal max clock
        double warps = (double)blocks * threads / 32;
        double winstr = warps * ITERS * k.instrs;
        printf("%-10s %.3f ms  warp-instr/clk/SM %.2f  lane-ops/clk/SM %.1f\n", k.name, ms, winstr / cycles / sms,
               winstr * 32 * (k.lane_ops / k.instrs) / cycles / sms);
    }
    printf("(clock %d kHz nominal, %d SMs; err %s)\n", clk, sms, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
