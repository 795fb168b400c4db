// masks.cu — on-device RM / FM sampling-set generators (include/ifctn.h
// ifctn_mask_uniform / ifctn_mask_fibres).
//
// The paper evaluates under random missingness (RM) and fibre-wise missingness (FM)
// (P:L423); reading R12 fixes the protocol: an exact count, drawn uniformly
// without replacement, as the k smallest of n i.i.d. keys.  Here the keys are the
// counter-based splitmix64 stream, key(u) = fmix64(seed + (u+1)·γ): a bijection of u, so all
// keys are distinct and "the k smallest" is unique (no tie rule needed).  The k-th smallest
// key is found by an MSD radix select, entirely stream-ordered (no host sync): two 12-bit
// digits, each one histogram pass over the keys sharing the resolved prefix plus one scan
// kernel that fixes the digit and the remaining rank in device memory; then the ≈ n/2^24
// keys left are collected and ranked in one CTA (8-bit full passes only on overflow).
// A final pass writes mask[u] = key(u) ≤ T (RM: observed; FM: the fibre of u is missing).
#include <cstdint>
#include <cstdlib>

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
constexpr int kBins = 4096;   // widest digit (12 bits)
constexpr int kCand = 4096;   // candidate buffer after the two 12-bit digits

struct SelectState {
    unsigned long long prefix;   // resolved high digits of the threshold key (the full key at the end)
    unsigned long long rank;     // 1-based rank of the threshold among keys with that prefix
    unsigned long long count;    // candidates matching the 24-bit prefix
    int overflow;                // 1: more than kCand candidates -> finish with 8-bit full passes
    int pad;
    unsigned long long hist[kBins];
    unsigned long long cand[kCand];
};

// Histogram of the `width`-bit digit at `shift` over the keys whose bits above the digit equal
// the resolved prefix.  Shared-memory bins, one global atomic per non-empty bin per CTA.
// `fallback`: run only when the candidate buffer overflowed (else return at once).
__global__ void __launch_bounds__(256) select_hist(SelectState* st, unsigned long long seed,
                                                   long long n, int shift, int width, int fallback) {
    if (fallback && !st->overflow) return;
    __shared__ unsigned int h[kBins];
    const int bins = 1 << width;
    for (int b = threadIdx.x; b < bins; b += blockDim.x) h[b] = 0;
    __syncthreads();
    const unsigned long long pre = st->prefix;
    const unsigned long long hi_mask = shift + width >= 64 ? 0ull : (~0ull << (shift + width));
    const unsigned int dmask = bins - 1;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long u = (long long)blockIdx.x * blockDim.x + threadIdx.x; u < n; u += stride) {
        const unsigned long long k = key_of(seed, (unsigned long long)u);
        if ((k & hi_mask) == pre) atomicAdd(&h[(unsigned)(k >> shift) & dmask], 1u);
    }
    __syncthreads();
    for (int b = threadIdx.x; b < bins; b += blockDim.x)
        if (h[b]) atomicAdd(&st->hist[b], (unsigned long long)h[b]);
}

// Fix the digit at `shift`: the bin holding the rank-th smallest candidate; clear the
// histogram.  1024 threads, each owning bins/1024 consecutive bins (≥ 1 when width ≥ 10,
// else threads past `bins` own none).
__global__ void __launch_bounds__(1024) select_digit(SelectState* st, int shift, int width, int fallback) {
    if (fallback && !st->overflow) return;
    __shared__ unsigned long long c[1024];
    const int t = threadIdx.x;
    const int bins = 1 << width;
    const int per = bins >= 1024 ? bins / 1024 : 1;
    const int b0 = t * per;
    unsigned long long own = 0;
    for (int q = 0; q < per && b0 + q < bins; ++q) own += st->hist[b0 + q];
    c[t] = own;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {   // inclusive scan (Hillis–Steele)
        const unsigned long long v = t >= off ? c[t - off] : 0ull;
        __syncthreads();
        c[t] += v;
        __syncthreads();
    }
    const unsigned long long r = st->rank;
    unsigned long long below = t ? c[t - 1] : 0ull;
    __syncthreads();
    if (below < r && r <= c[t]) {
        for (int q = 0; q < per; ++q) {
            const unsigned long long h = st->hist[b0 + q];
            if (r <= below + h) {
                st->prefix |= (unsigned long long)(b0 + q) << shift;
                st->rank = r - below;
                break;
            }
            below += h;
        }
    }
    __syncthreads();
    for (int q = 0; q < per && b0 + q < bins; ++q) st->hist[b0 + q] = 0ull;
}

// Append every key matching the resolved prefix (bits ≥ `shift`) to the candidate buffer.
__global__ void __launch_bounds__(256) select_collect(SelectState* st, unsigned long long seed, long long n,
                                                     int shift, unsigned long long cap) {
    const unsigned long long pre = st->prefix;
    const unsigned long long hi_mask = ~0ull << shift;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long u = (long long)blockIdx.x * blockDim.x + threadIdx.x; u < n; u += stride) {
        const unsigned long long k = key_of(seed, (unsigned long long)u);
        if ((k & hi_mask) == pre) {
            const unsigned long long slot = atomicAdd(&st->count, 1ull);
            if (slot < cap) st->cand[slot] = k;
        }
    }
}

// The rank-th smallest candidate (keys are distinct): for each candidate, count the smaller
// ones.  Sets prefix = T, or flags overflow for the 8-bit fallback passes.
__global__ void __launch_bounds__(1024) select_resolve(SelectState* st, unsigned long long cap) {
    const unsigned long long cnt = st->count;
    if (cnt > cap) {
        if (threadIdx.x == 0) st->overflow = 1;
        return;
    }
    __shared__ unsigned long long c[kCand];
    for (unsigned long long x = threadIdx.x; x < cnt; x += blockDim.x) c[x] = st->cand[x];
    __syncthreads();
    const unsigned long long r = st->rank;
    for (unsigned long long x = threadIdx.x; x < cnt; x += blockDim.x) {
        unsigned long long less = 0;
        for (unsigned long long y = 0; y < cnt; ++y) less += c[y] < c[x];
        if (less + 1 == r) st->prefix = c[x];  // rank is not read after a resolve
    }
}

__global__ void __launch_bounds__(1024) init_state(SelectState* st, unsigned long long k) {
    for (int b = threadIdx.x; b < kBins; b += blockDim.x) st->hist[b] = 0ull;
    if (threadIdx.x == 0) {
        st->prefix = 0ull;
        st->rank = k;
        st->count = 0ull;
        st->overflow = 0;
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
    for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g * 16 < n; g += stride) {
        const long long u0 = g * 16;
        // (lo, mid, hi) of u0 once, then stepped: u = lo + inner·(mid + Im·hi)
        long long lo = u0 % inner, q = u0 / inner;
        long long mid = q % Im, hi = q / Im;
        uint8_t b[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const long long f = lo + inner * hi;
            const bool miss = every || (!none && key_of(seed, (unsigned long long)f) <= T);
            b[j] = miss ? 0 : 1;
            if (++lo == inner) {
                lo = 0;
                if (++mid == Im) {
                    mid = 0;
                    ++hi;
                }
            }
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

// Select the k-th smallest of key(0..n-1) into st->prefix (1 ≤ k ≤ n): two 12-bit digits
// over all keys, then the ~n/2^24 keys left are collected and ranked in one CTA; only if more
// than kCand remain (never expected below n ≈ 2^34) do five 8-bit full passes finish the job.
cudaError_t select_kth(SelectState* st, unsigned long long seed, long long n, long long k, cudaStream_t s) {
    init_state<<<1, 1024, 0, s>>>(st, (unsigned long long)k);
    const int g = grid_for(n);
    for (int shift : {52, 40}) {
        select_hist<<<g, 256, 0, s>>>(st, seed, n, shift, 12, 0);
        select_digit<<<1, 1024, 0, s>>>(st, shift, 12, 0);
    }
    // IFCTN_MASK_CAND_CAP (tests only) lowers the buffer to exercise the fallback passes
    static const long long cap_env = [] {
        const char* e = getenv("IFCTN_MASK_CAND_CAP");
        return e ? atoll(e) : (long long)kCand;
    }();
    const unsigned long long cap = (unsigned long long)(cap_env < 0 ? 0 : (cap_env > kCand ? kCand : cap_env));
    select_collect<<<g, 256, 0, s>>>(st, seed, n, 40, cap);
    select_resolve<<<1, 1024, 0, s>>>(st, cap);
    for (int shift = 32; shift >= 0; shift -= 8) {
        select_hist<<<g, 256, 0, s>>>(st, seed, n, shift, 8, 1);
        select_digit<<<1, 1024, 0, s>>>(st, shift, 8, 1);
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

// Single exit after the scratch allocation: the scratch is always released on the stream,
// whatever failed before (a failed launch leaves the stream usable for the free).
ifctn_status finish(SelectState* st, cudaStream_t stream, cudaError_t e) {
    if (e == cudaSuccess) e = cudaGetLastError();
    const cudaError_t f = cudaFreeAsync(st, stream);
    return (e == cudaSuccess && f == cudaSuccess) ? IFCTN_OK : IFCTN_E_CUDA;
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
    cudaError_t e = cudaSuccess;
    if (observed > 0 && !all) {
        e = select_kth(st, seed, n, observed, stream);
    } else {
        init_state<<<1, 1024, 0, stream>>>(st, 0ull);  // T unused: all observed, or memset below
    }
    if (e == cudaSuccess) {
        if (observed == 0) e = cudaMemsetAsync(mask, 0, (size_t)n, stream);
        else write_uniform<<<grid_for((n + 15) / 16), 256, 0, stream>>>(mask, st, seed, n, all);
    }
    return finish(st, stream, e);
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
    cudaError_t e = cudaSuccess;
    if (!none && !every) {
        e = select_kth(st, seed, nf, missing_fibres, stream);
    } else {
        init_state<<<1, 1024, 0, stream>>>(st, 0ull);  // T unused (none / every flag)
    }
    if (e == cudaSuccess)
        write_fibres<<<grid_for((n + 15) / 16), 256, 0, stream>>>(mask, st, seed, n, inner, Im, none, every);
    return finish(st, stream, e);
}
