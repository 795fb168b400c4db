// masks.cu — on-device RM / FM sampling-set generators (include/ifctn.h
// ifctn_mask_uniform / ifctn_mask_fibres).
//
// The paper evaluates under random missingness (RM) and fibre-wise missingness (FM)
// (P:L423); reading R12 fixes the protocol: an exact count, drawn uniformly
// without replacement, as the k smallest of n i.i.d. keys.  Here the keys are the
// counter-based splitmix64 stream, key(u) = fmix64(seed + (u+1)·γ): a bijection of u, so all
// keys are distinct and "the k smallest" is unique (no tie rule needed).  The k-th smallest
// key is found by an 8-digit (8-bit) MSD radix select, entirely stream-ordered: per digit one
// histogram pass over the candidates that share the resolved prefix, then one 256-thread
// scan kernel that fixes the digit and the remaining rank in device memory (no host sync).
// A final pass writes mask[u] = key(u) ≤ T (RM: observed; FM: the fibre of u is missing).
#include <cstdint>

#include <cuda_runtime.h>

#include "../../include/ifctn.h"

namespace {

constexpr unsigned long long kGamma = 0x9E3779B97F4A7C15ull;

__host__ __device__ __forceinline__ unsigned long long fmix64(unsigned long long z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ unsigned long long key_of(unsigned long long seed, unsigned long long u) {
    return fmix64(seed + (u + 1ull) * kGamma);
}

// device-resident select state
struct SelectState {
    unsigned long long prefix;   // resolved high digits of the threshold key
    unsigned long long rank;     // 1-based rank of the threshold among keys with that prefix
    unsigned long long hist[256];
};

// Histogram of digit `d` (0 = most significant byte) over the keys whose higher digits equal
// the resolved prefix.  Shared-memory bins, one global atomic per bin per CTA.
__global__ void __launch_bounds__(256) select_hist(SelectState* st, unsigned long long seed,
                                                   long long n, int d) {
    __shared__ unsigned int h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    const int shift = 56 - 8 * d;
    const unsigned long long pre = st->prefix;
    const unsigned long long hi_mask = d == 0 ? 0ull : (~0ull << (64 - 8 * d));
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long u = (long long)blockIdx.x * blockDim.x + threadIdx.x; u < n; u += stride) {
        const unsigned long long k = key_of(seed, (unsigned long long)u);
        if ((k & hi_mask) == pre) atomicAdd(&h[(k >> shift) & 0xFF], 1u);
    }
    __syncthreads();
    if (h[threadIdx.x]) atomicAdd(&st->hist[threadIdx.x], (unsigned long long)h[threadIdx.x]);
}

// Fix digit d: the bin holding the rank-th smallest candidate; clear the histogram.
__global__ void __launch_bounds__(256) select_digit(SelectState* st, int d) {
    __shared__ unsigned long long c[256];
    const int t = threadIdx.x;
    c[t] = st->hist[t];
    __syncthreads();
    // inclusive scan (Hillis–Steele; 256 entries)
    for (int off = 1; off < 256; off <<= 1) {
        const unsigned long long v = t >= off ? c[t - off] : 0ull;
        __syncthreads();
        c[t] += v;
        __syncthreads();
    }
    const unsigned long long r = st->rank;
    const unsigned long long below = t ? c[t - 1] : 0ull;
    __syncthreads();
    if (below < r && r <= c[t]) {
        st->prefix |= (unsigned long long)t << (56 - 8 * d);
        st->rank = r - below;
    }
    st->hist[t] = 0ull;
}

__global__ void __launch_bounds__(256) init_state(SelectState* st, unsigned long long k) {
    st->hist[threadIdx.x] = 0ull;
    if (threadIdx.x == 0) {
        st->prefix = 0ull;
        st->rank = k;
    }
}

// 16 mask bytes from registers: one 16-byte store where whole and aligned, else bytewise.
__device__ __forceinline__ void store16(uint8_t* mask, long long u0, long long n, const uint8_t (&b)[16]) {
    if (u0 + 16 <= n && ((reinterpret_cast<uintptr_t>(mask + u0) & 15) == 0)) {
        unsigned int w[4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
            w[q] = (unsigned)b[4 * q] | ((unsigned)b[4 * q + 1] << 8) | ((unsigned)b[4 * q + 2] << 16) |
                   ((unsigned)b[4 * q + 3] << 24);
        *reinterpret_cast<uint4*>(mask + u0) = make_uint4(w[0], w[1], w[2], w[3]);
    } else {
#pragma unroll
        for (int j = 0; j < 16; ++j)
            if (u0 + j < n) mask[u0 + j] = b[j];
    }
}

// RM: mask[u] = 1 iff key(u) ≤ T.  16 entries per thread, one 16-byte store where aligned.
__global__ void __launch_bounds__(256) write_uniform(uint8_t* __restrict__ mask, const SelectState* st,
                                                     unsigned long long seed, long long n, int all) {
    const unsigned long long T = st->prefix;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g * 16 < n; g += stride) {
        const long long u0 = g * 16;
        uint8_t b[16];
#pragma unroll
        for (int j = 0; j < 16; ++j)
            b[j] = (all || key_of(seed, (unsigned long long)(u0 + j)) <= T) ? 1 : 0;
        store16(mask, u0, n, b);
    }
}

// FM: entry u lies on fibre f(u) = lo + inner·hi (u = lo + inner·(i_m + I_m·hi)); the fibre is
// missing iff key(f) ≤ T.  `none` = no fibre missing, `every` = all missing.
__global__ void __launch_bounds__(256) write_fibres(uint8_t* __restrict__ mask, const SelectState* st,
                                                    unsigned long long seed, long long n,
                                                    long long inner, long long Im, int none, int every) {
    const unsigned long long T = st->prefix;
    const long long stride = (long long)gridDim.x * blockDim.x;
    const long long span = inner * Im;
    for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g * 16 < n; g += stride) {
        const long long u0 = g * 16;
        uint8_t b[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const long long u = u0 + j;
            const long long f = u % inner + inner * (u / span);
            const bool miss = every || (!none && key_of(seed, (unsigned long long)f) <= T);
            b[j] = miss ? 0 : 1;
        }
        store16(mask, u0, n, b);
    }
}

int grid_for(long long work) {
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const long long want = (work + 255) / 256;
    const long long cap = (long long)sms * 8;  // 8 resident 256-thread CTAs per SM
    return (int)(want < 1 ? 1 : (want < cap ? want : cap));
}

// Radix-select the k-th smallest of key(0..n-1) into st->prefix (1 ≤ k ≤ n).
cudaError_t select_kth(SelectState* st, unsigned long long seed, long long n, long long k, cudaStream_t s) {
    init_state<<<1, 256, 0, s>>>(st, (unsigned long long)k);
    const int g = grid_for(n);
    for (int d = 0; d < 8; ++d) {
        select_hist<<<g, 256, 0, s>>>(st, seed, n, d);
        select_digit<<<1, 256, 0, s>>>(st, d);
    }
    return cudaGetLastError();
}

bool is_device_ptr(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

}  // namespace

extern "C" ifctn_status ifctn_mask_uniform(uint8_t* mask, int64_t n, int64_t observed, uint64_t seed,
                                           void* stream_) {
    cudaStream_t stream = static_cast<cudaStream_t>(stream_);
    if (n < 0 || observed < 0 || observed > n || (n > 0 && !mask)) return IFCTN_E_ARG;
    if (n == 0) return IFCTN_OK;
    if (!is_device_ptr(mask)) return IFCTN_E_ARG;
    SelectState* st = nullptr;
    if (cudaMallocAsync(reinterpret_cast<void**>(&st), sizeof(SelectState), stream) != cudaSuccess)
        return IFCTN_E_CUDA;
    const int all = observed == n;
    if (observed > 0 && !all) {
        if (select_kth(st, seed, n, observed, stream) != cudaSuccess) return IFCTN_E_CUDA;
    } else {
        init_state<<<1, 256, 0, stream>>>(st, 0ull);  // T unused: all observed, or memset below
    }
    if (observed == 0) {
        if (cudaMemsetAsync(mask, 0, (size_t)n, stream) != cudaSuccess) return IFCTN_E_CUDA;
    } else {
        write_uniform<<<grid_for((n + 15) / 16), 256, 0, stream>>>(mask, st, seed, n, all);
    }
    if (cudaFreeAsync(st, stream) != cudaSuccess) return IFCTN_E_CUDA;
    return cudaGetLastError() == cudaSuccess ? IFCTN_OK : IFCTN_E_CUDA;
}

extern "C" ifctn_status ifctn_mask_fibres(uint8_t* mask, int order, const int64_t* dims, int mode,
                                          int64_t missing_fibres, uint64_t seed, void* stream_) {
    cudaStream_t stream = static_cast<cudaStream_t>(stream_);
    if (order < 1 || !dims || mode < 0 || mode >= order || missing_fibres < 0) return IFCTN_E_ARG;
    long long n = 1, inner = 1;
    for (int m = 0; m < order; ++m) {
        if (dims[m] < 1) return IFCTN_E_SHAPE;
        n *= dims[m];
        if (m < mode) inner *= dims[m];
    }
    const long long Im = dims[mode];
    const long long nf = n / Im;
    if (missing_fibres > nf || !mask) return IFCTN_E_ARG;
    if (!is_device_ptr(mask)) return IFCTN_E_ARG;
    SelectState* st = nullptr;
    if (cudaMallocAsync(reinterpret_cast<void**>(&st), sizeof(SelectState), stream) != cudaSuccess)
        return IFCTN_E_CUDA;
    const int none = missing_fibres == 0, every = missing_fibres == nf;
    if (!none && !every) {
        if (select_kth(st, seed, nf, missing_fibres, stream) != cudaSuccess) return IFCTN_E_CUDA;
    } else {
        init_state<<<1, 256, 0, stream>>>(st, 0ull);  // T unused (none / every flag)
    }
    write_fibres<<<grid_for((n + 15) / 16), 256, 0, stream>>>(mask, st, seed, n, inner, Im, none, every);
    if (cudaFreeAsync(st, stream) != cudaSuccess) return IFCTN_E_CUDA;
    return cudaGetLastError() == cudaSuccess ? IFCTN_OK : IFCTN_E_CUDA;
}
