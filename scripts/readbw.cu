// readbw.cu — B200 read-bandwidth ceilings for the a2 pass design (diagnostic, not product):
//   (1) LDG.128 grid-stride sum, (2) per-warp TMA cp.async.bulk ring of 2 KB stages into
//   shared memory with an mbarrier per stage (the fiber_pass data movement with no math).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o readbw scripts/readbw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) ldg_sum(const float4* __restrict__ x, size_t n4, float* out) {
    float acc = 0.f;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll 4
    for (; i < n4; i += stride) {
        float4 v;
        asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(x + i));
        acc += v.x + v.y + v.z + v.w;
    }
    if (acc == 123456.f) out[0] = acc;
}

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// PERM = 8: logical stage L of the warp stream maps to physical stage (L mod FR)·8 + L / FR
// (FR = stages / 8), i.e. a warp's consecutive stages are 8 stages (16 KB) apart — the access
// pattern of the tiled a2 pass (8 v-blocks of 2 KB per 16 KB).
template <int D, int STAGE_BYTES, int PERM = 1>
__global__ void __launch_bounds__(256) tma_ring(const char* __restrict__ x, size_t nbytes, float* out) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm) + warp * D;
    unsigned char* ring = sm + 8 * D * nw + (size_t)warp * D * STAGE_BYTES;
    if (lane == 0)
        for (int s = 0; s < D; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    __syncwarp();
    const size_t nst = nbytes / STAGE_BYTES;
    const size_t gw = (size_t)blockIdx.x * nw + warp, tw = (size_t)gridDim.x * nw;
    const size_t per = (nst + tw - 1) / tw;
    const size_t FR = nst / PERM;
    auto phys = [&](size_t L) { return PERM == 1 ? L : (L % FR) * PERM + L / FR; };
    const size_t s0 = gw * per, s1 = s0 + per < nst ? s0 + per : nst;
    auto issue = [&](size_t st, int n) {
        const int s = n % D;
        const uint32_t bar = su32(&bars[s]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(STAGE_BYTES));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(su32(ring + s * STAGE_BYTES)), "l"(x + phys(st) * STAGE_BYTES), "r"(STAGE_BYTES), "r"(bar) : "memory");
    };
    int pn = 0;
    if (lane == 0)
        for (int d = 0; d < D && s0 + d < s1; ++d) issue(s0 + d, pn++);
    float acc = 0.f;
    int cn = 0;
    for (size_t st = s0; st < s1; ++st, ++cn) {
        const int s = cn % D;
        uint32_t done = 0;
        do {
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                         : "=r"(done) : "r"(su32(&bars[s])), "r"((uint32_t)((cn / D) & 1)) : "memory");
        } while (!done);
        const float4 v = reinterpret_cast<const float4*>(ring + s * STAGE_BYTES)[lane];
        acc += v.x + v.y + v.z + v.w;
        __syncwarp();
        if (lane == 0 && st + D < s1) {
            asm volatile("fence.proxy.async.shared::cta;");
            issue(st + D, pn++);
        }
    }
    if (acc == 123456.f) out[0] = acc;
}

template <int D, int SB, int PERM>
void run_ring(const char* x, size_t nbytes, float* out, int nsm, int bps, int threads,
              cudaEvent_t a, cudaEvent_t b) {
    const size_t smem = 8 * D * (threads / 32) + (size_t)(threads / 32) * D * SB;
    cudaFuncSetAttribute(tma_ring<D, SB, PERM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    auto fn = [&] { tma_ring<D, SB, PERM><<<nsm * bps, threads, smem>>>(x, nbytes, out); };
    for (int w = 0; w < 3; ++w) fn();
    cudaEventRecord(a);
    const int reps = 10;
    for (int r = 0; r < reps; ++r) fn();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("tma ring D%d %5dB perm%d %d CTA/SM x %2d warps (%3zu KB smem, %3d KB in flight/SM) %7.1f us %7.1f GB/s\n",
           D, SB, PERM, bps, threads / 32, smem / 1024, bps * (threads / 32) * D * SB / 1024,
           1e3 * ms / reps, nbytes / (ms / reps / 1e3) / 1e9);
}

int main(int argc, char** argv) {
    const size_t nbytes = 2147483648ull;
    char* x;
    float* out;
    cudaMalloc(&x, nbytes);
    cudaMalloc(&out, 4);
    cudaMemset(x, 0, nbytes);
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int rep = 0; rep < 2; ++rep) {
        for (int bps : {1, 2}) {
            for (int th : {256, 512}) {
                if (bps * th > 1024) continue;
                run_ring<2, 2048, 8>(x, nbytes, out, nsm, bps, th, a, b);
                run_ring<4, 2048, 8>(x, nbytes, out, nsm, bps, th, a, b);
                run_ring<4, 1024, 8>(x, nbytes, out, nsm, bps, th, a, b);
                run_ring<8, 1024, 8>(x, nbytes, out, nsm, bps, th, a, b);
                run_ring<3, 2048, 8>(x, nbytes, out, nsm, bps, th, a, b);
                run_ring<2, 4096, 8>(x, nbytes, out, nsm, bps, th, a, b);
                if (th == 256) run_ring<4, 4096, 8>(x, nbytes, out, nsm, bps, th, a, b);
            }
        }
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
