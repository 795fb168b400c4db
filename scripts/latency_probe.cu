// latency_probe.cu — fixed costs that bound the small (L2-resident) configs on this B200:
//   (a) dependent kernel-to-kernel time inside a CUDA graph (empty kernels, 1 and 296 CTAs);
//   (b) one grid-wide barrier (atomic arrive + spin on a generation word) in a cooperative
//       launch of 148 / 296 CTAs;
//   (c) an arrival counter + "last CTA" handoff (no spin), as used by a fused block kernel.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/latency_probe scripts/latency_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void empty_k(int* p) {
    if (p && threadIdx.x == 0 && blockIdx.x == 0) p[0] += 1;
}

__device__ __forceinline__ void grid_barrier(unsigned* count, volatile unsigned* gen, unsigned nb) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned g = *gen;
        __threadfence();
        if (atomicAdd(count, 1u) == nb - 1) {
            *count = 0;
            __threadfence();
            atomicAdd((unsigned*)gen, 1u);
        } else {
            while (*gen == g) {
            }
        }
        __threadfence();
    }
    __syncthreads();
}

__global__ void barrier_k(unsigned* count, unsigned* gen, int iters) {
    for (int i = 0; i < iters; ++i) grid_barrier(count, gen, gridDim.x);
}

__global__ void coop_k(int iters) {
    namespace cg = cooperative_groups;
    cg::grid_group g = cg::this_grid();
    for (int i = 0; i < iters; ++i) g.sync();
}

__global__ void lastcta_k(unsigned* count, double* out) {
    __shared__ bool last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(count, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
        *count = 0;
        out[0] += 1.0;
    }
}

int main() {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    int* d;
    unsigned *cnt, *gen;
    double* out;
    cudaMalloc(&d, 64);
    cudaMalloc(&cnt, 64);
    cudaMalloc(&gen, 64);
    cudaMalloc(&out, 64);
    cudaMemset(d, 0, 64);
    cudaMemset(cnt, 0, 64);
    cudaMemset(gen, 0, 64);
    cudaMemset(out, 0, 64);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int NK = 200;
    for (int grid : {1, nsm, 2 * nsm, 4 * nsm}) {
        for (int kind = 0; kind < 2; ++kind) {
            cudaGraph_t g;
            cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
            for (int k = 0; k < NK; ++k) {
                if (kind == 0) empty_k<<<grid, 256, 0, s>>>(d);
                else lastcta_k<<<grid, 256, 0, s>>>(cnt, out);
            }
            cudaStreamEndCapture(s, &g);
            cudaGraphExec_t ge;
            cudaGraphInstantiate(&ge, g, 0);
            for (int w = 0; w < 3; ++w) cudaGraphLaunch(ge, s);
            cudaEventRecord(e0, s);
            for (int r = 0; r < 10; ++r) cudaGraphLaunch(ge, s);
            cudaEventRecord(e1, s);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("graph chain %-12s grid %4d: %.2f us per kernel\n", kind ? "lastcta" : "empty", grid,
                   1e3 * ms / (10 * NK));
            cudaGraphExecDestroy(ge);
            cudaGraphDestroy(g);
        }
    }
    const int IT = 2000;
    for (int grid : {nsm, 2 * nsm, 4 * nsm}) {
        void* args[] = {&cnt, &gen, (void*)&IT};
        cudaLaunchCooperativeKernel((void*)barrier_k, grid, 256, args, 0, s);
        cudaEventRecord(e0, s);
        cudaLaunchCooperativeKernel((void*)barrier_k, grid, 256, args, 0, s);
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("atomic grid barrier grid %4d: %.3f us per barrier (%s)\n", grid, 1e3 * ms / IT,
               cudaGetErrorString(cudaGetLastError()));
        void* a2[] = {(void*)&IT};
        cudaLaunchCooperativeKernel((void*)coop_k, grid, 256, a2, 0, s);
        cudaEventRecord(e0, s);
        cudaLaunchCooperativeKernel((void*)coop_k, grid, 256, a2, 0, s);
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("cg grid.sync    grid %4d: %.3f us per barrier (%s)\n", grid, 1e3 * ms / IT,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
