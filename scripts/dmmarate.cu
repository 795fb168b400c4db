// dmmarate.cu — fp64 tensor-core (mma.sync m8n8k4 f64, SASS DMMA) issue-rate microbenchmark
// (diagnostic): CH independent accumulator chains per warp, 8 warps per CTA, one wave of CTAs.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int CH>
__global__ void chains(double* out, int iters, double a, double b) {
    double x[CH][2];
#pragma unroll
    for (int k = 0; k < CH; ++k) x[k][0] = x[k][1] = (double)(threadIdx.x + k);
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int k = 0; k < CH; ++k) dmma(x[k][0], x[k][1], a, b);
    double s = 0;
#pragma unroll
    for (int k = 0; k < CH; ++k) s += x[k][0] + x[k][1];
    if (s == 123.456) out[0] = s;
}
template <int CH>
void bench(int nsm, double* o) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 4096;
    for (int bps : {1, 2, 4}) {
        chains<CH><<<nsm * bps, 256>>>(o, iters, 0.999, 0.001);
        cudaEventRecord(e0);
        chains<CH><<<nsm * bps, 256>>>(o, iters, 0.999, 0.001);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double fma = (double)nsm * bps * 8 * iters * CH * 256;
        printf("DMMA m8n8k4 %2d chains/warp %d CTA/SM: %.3f ms  %.2f TFLOP/s\n", CH, bps, ms, 2 * fma / (ms * 1e-3) / 1e12);
    }
}
int main() {
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    double* o;
    cudaMalloc(&o, 64);
    bench<1>(nsm, o);
    bench<4>(nsm, o);
    bench<16>(nsm, o);
    return 0;
}
