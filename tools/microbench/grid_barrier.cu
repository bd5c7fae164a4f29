// grid_barrier.cu — what a pass boundary costs on B200: (a) a chain of
// dependent empty kernels inside one CUDA graph, (b) a software grid barrier
// (arrive counter + generation flag, release/acquire at gpu scope) inside one
// persistent launch of G co-resident CTAs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gb grid_barrier.cu && /tmp/gb
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_empty(int* p) {
    if (p && threadIdx.x == 0 && blockIdx.x == 0) atomicAdd(p, 0);
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void grid_sync(unsigned* count, unsigned* gen, unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned g = ld_acquire(gen);
        unsigned old;
        asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(count) : "memory");
        if (old == nblocks - 1) {
            *count = 0;
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(gen), "r"(g + 1) : "memory");
        } else {
            while (ld_acquire(gen) == g) {
            }
        }
    }
    __syncthreads();
}

__global__ void k_barriers(unsigned* count, unsigned* gen, int reps) {
    for (int i = 0; i < reps; ++i) grid_sync(count, gen, gridDim.x);
}

int main() {
    cudaStream_t st;
    cudaStreamCreate(&st);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int* dummy;
    cudaMalloc(&dummy, 4);
    for (int grid : {148, 256, 512}) {
        for (int threads : {64, 128, 256}) {
            const int n = 200;
            cudaGraph_t g;
            cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
            for (int i = 0; i < n; ++i) k_empty<<<grid, threads, 0, st>>>(dummy);
            cudaStreamEndCapture(st, &g);
            cudaGraphExec_t ge;
            cudaGraphInstantiate(&ge, g, 0);
            cudaGraphLaunch(ge, st);
            cudaEventRecord(e0, st);
            for (int r = 0; r < 5; ++r) cudaGraphLaunch(ge, st);
            cudaEventRecord(e1, st);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("graph chain   grid %4d x %4d: %.3f us per kernel\n", grid, threads, 1e3 * ms / (5 * n));
            cudaGraphExecDestroy(ge);
            cudaGraphDestroy(g);
        }
    }
    unsigned* cnt;
    cudaMalloc(&cnt, 8);
    for (int grid : {148, 256, 296, 512}) {
        for (int threads : {64, 128, 256}) {
            cudaMemset(cnt, 0, 8);
            const int reps = 2000;
            k_barriers<<<grid, threads, 0, st>>>(cnt, cnt + 1, 10);
            cudaEventRecord(e0, st);
            k_barriers<<<grid, threads, 0, st>>>(cnt, cnt + 1, reps);
            cudaEventRecord(e1, st);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("grid barrier  grid %4d x %4d: %.3f us per barrier (%s)\n", grid, threads, 1e3 * ms / reps,
                   cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
