// gram_mma_bench.cu — the k-loop and warp-order reduction of big_gram_mma (solve.cuh) in
// isolation (diagnostic): R = 36, I_i = 256, one CTA of 256 threads per column, 256 columns.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
constexpr int R = 36, NA = 256, LDA = 37, NRT = 5, NTILE = 15, TPR = 4;
template <int MODE>  // 0 all, 1 no reduction, 2 no DMMA, 3 no loads (register operands), 4 scratch reduction
__global__ void __launch_bounds__(256) k(const double* g, const double* w, double* out, long long* clk) {
    extern __shared__ double sm[];
    double* gs = sm;
    double* A = gs + NA * R + 40;
    double* om = A + 40 * LDA;
    double* be = om + NA;
    double* rhs = be + NA;
    double* scr = rhs + 40;  // MODE 4: 8 warps x TPR tiles x 64
    const int tid = threadIdx.x, lane = tid & 31, wi = tid >> 5, lk = lane & 3, lq = lane >> 2;
    for (int e = tid; e < NA * R + 40; e += 256) gs[e] = e < NA * R ? g[e] : 0.0;
    for (int a = tid; a < NA; a += 256) { om[a] = w[a]; be[a] = w[NA + a]; }
    __syncthreads();
    long long t0 = clock64();
    double acc[NTILE][2];
#pragma unroll
    for (int t = 0; t < NTILE; ++t) acc[t][0] = acc[t][1] = 0.0;
    for (int ks = wi; 4 * ks < NA; ks += 8) {
        const int a = 4 * ks + lk;
        const double ww = om[a], b = be[a];
        const double* gr = gs + a * R + lq;
        double fa[NRT], fb[NRT];
#pragma unroll
        for (int t = 0; t < NRT; ++t) fa[t] = MODE == 3 ? ww + t : gr[8 * t];
#pragma unroll
        for (int t = 0; t < NRT; ++t) {
            const int s = 8 * t + lq;
            fb[t] = (t + 1 < NRT || s < R) ? ww * fa[t] : (s == R ? b : 0.0);
        }
        int t = 0;
#pragma unroll
        for (int tr = 0; tr < NRT; ++tr)
#pragma unroll
            for (int tc = tr; tc < NRT; ++tc, ++t) {
                if (MODE == 2) { acc[t][0] += fa[tr]; acc[t][1] += fb[tc]; }
                else dmma884(acc[t][0], acc[t][1], fa[tr], fb[tc]);
            }
    }
    long long t1 = clock64();
    if (MODE == 4) {
        // rounds of TPR tiles: every warp writes its partial tiles, then one thread per entry
        // sums the 8 partials in warp order
        constexpr int NQ = (NTILE + TPR - 1) / TPR;
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            if (q) __syncthreads();
#pragma unroll
            for (int tt = 0; tt < TPR; ++tt)
                if (q * TPR + tt < NTILE)
                    *reinterpret_cast<double2*>(scr + (wi * TPR + tt) * 64 + 2 * lane) =
                        make_double2(acc[q * TPR + tt][0], acc[q * TPR + tt][1]);
            __syncthreads();
            const int tt = tid >> 6, idx = tid & 63, t = q * TPR + tt;
            if (t < NTILE) {
                double v[8];
#pragma unroll
                for (int w8 = 0; w8 < 8; ++w8) v[w8] = scr[(w8 * TPR + tt) * 64 + idx];
                double sum = v[0];
#pragma unroll
                for (int w8 = 1; w8 < 8; ++w8) sum += v[w8];
                int tr = 0, rem = t;
                while (rem >= NRT - tr) { rem -= NRT - tr; ++tr; }
                const int r = 8 * tr + (idx >> 3), sc = 8 * (tr + rem) + (idx & 7);
                if (r < R && sc <= R && r <= sc) *(sc < R ? A + r * LDA + sc : rhs + r) = sum;
            }
        }
    } else if (MODE != 1) {
        for (int h = 0; h < 8; ++h) {
            __syncthreads();
        if (wi == h) {  // every load of the warp's entries in flight before the first store
            double old[NTILE][2];
            int t = 0;
#pragma unroll
            for (int tr = 0; tr < NRT; ++tr)
#pragma unroll
                for (int tc = tr; tc < NRT; ++tc, ++t) {
                    const int r = 8 * tr + lq;
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int s = 8 * tc + 2 * lk + e;
                        const bool on = r < R && s <= R && r <= s;
                        const double* d = s < R ? A + r * LDA + s : rhs + r;
                        old[t][e] = (on && h) ? *d : 0.0;
                    }
                }
            t = 0;
#pragma unroll
            for (int tr = 0; tr < NRT; ++tr)
#pragma unroll
                for (int tc = tr; tc < NRT; ++tc, ++t) {
                    const int r = 8 * tr + lq;
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int s = 8 * tc + 2 * lk + e;
                        double* d = s < R ? A + r * LDA + s : rhs + r;
                        if (r < R && s <= R && r <= s) *d = old[t][e] + acc[t][e];
                    }
                }
        }
        }
    } else {
        double s = 0;
#pragma unroll
        for (int t = 0; t < NTILE; ++t) s += acc[t][0] + acc[t][1];
        if (s == 1.2345) A[tid] = s;
    }
    __syncthreads();
    long long t2 = clock64();
    if (tid < R) out[blockIdx.x * R + tid] = A[tid * LDA + tid] + rhs[tid];
    if (blockIdx.x == 0 && (tid & 31) == 0) { clk[2 * wi] = t1 - t0; clk[2 * wi + 1] = t2 - t1; }
}
template <int MODE>
void run(const double* g, const double* w, double* out, long long* clk, const char* name) {
    const size_t smem = sizeof(double) * (NA * R + 40 + 40 * LDA + 2 * NA + 40 + 8 * TPR * 64);
    cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k<MODE><<<256, 256, smem>>>(g, w, out, clk);
    cudaEventRecord(e0);
    k<MODE><<<256, 256, smem>>>(g, w, out, clk);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long h[16];
    cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost);
    printf("%-12s %.1f us  CTA 0 per warp [k-loop | reduce] cycles:", name, ms * 1e3);
    for (int w8 = 0; w8 < 8; ++w8) printf(" %lld|%lld", h[2 * w8], h[2 * w8 + 1]);
    printf("  (%s)\n", cudaGetErrorString(cudaGetLastError()));
}
int main() {
    double *g, *w, *out;
    long long* clk;
    cudaMalloc(&g, sizeof(double) * NA * R);
    cudaMalloc(&w, sizeof(double) * 2 * NA);
    cudaMalloc(&out, sizeof(double) * 256 * R);
    cudaMalloc(&clk, sizeof(long long) * 16);
    double hg[NA * R], hw[2 * NA];
    for (int i = 0; i < NA * R; ++i) hg[i] = 0.001 * ((i * 7919) % 1000) - 0.5;
    for (int i = 0; i < 2 * NA; ++i) hw[i] = 0.01 * (i % 97);
    cudaMemcpy(g, hg, sizeof(hg), cudaMemcpyHostToDevice);
    cudaMemcpy(w, hw, sizeof(hw), cudaMemcpyHostToDevice);
    run<0>(g, w, out, clk, "all");
    run<1>(g, w, out, clk, "no reduce");
    run<2>(g, w, out, clk, "no DMMA");
    run<3>(g, w, out, clk, "no g loads");
    run<4>(g, w, out, clk, "scratch red");
    cudaMemcpy(hw, out, sizeof(double) * 8, cudaMemcpyDeviceToHost);
    printf("scratch out %.12g %.12g\n", hw[0], hw[7]);
    run<0>(g, w, out, clk, "all");
    cudaMemcpy(hw, out, sizeof(double) * 8, cudaMemcpyDeviceToHost);
    printf("serial  out %.12g %.12g\n", hw[0], hw[7]);
    return 0;
}
