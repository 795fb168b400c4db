// fp64rate.cu — DFMA / FFMA issue-rate microbenchmark (diagnostic): 16 independent chains
// per thread, 8 warps per CTA, one wave of CTAs.
#include <cstdio>
#include <cuda_runtime.h>
template <typename T>
__global__ void chains(T* out, int iters, T a, T b) {
    T x[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) x[k] = (T)(threadIdx.x + k);
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int k = 0; k < 16; ++k) x[k] = x[k] * a + b;
    T s = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) s += x[k];
    if (s == (T)123.456) out[0] = s;
}
int main() {
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    double* o;
    cudaMalloc(&o, 64);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 4096;
    for (int bps : {1, 4, 8}) {
        for (int dbl = 0; dbl < 2; ++dbl) {
            auto run = [&] {
                if (dbl) chains<double><<<nsm * bps, 256>>>(o, iters, 0.999, 0.001);
                else chains<float><<<nsm * bps, 256>>>((float*)o, iters, 0.999f, 0.001f);
            };
            run();
            cudaEventRecord(e0);
            run();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double fma = (double)nsm * bps * 256 * iters * 16;
            printf("%s %d CTA/SM: %.3f ms  %.2f TFLOP/s\n", dbl ? "DFMA" : "FFMA", bps, ms, 2 * fma / (ms * 1e-3) / 1e12);
        }
    }
    return 0;
}
