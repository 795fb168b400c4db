// peer.cuh — device-side exchange of the per-block Gram/RHS partials over peer memory
// (SURVEY §8(e) exchange step, §8(f4) "device-side allreduce"; BASELINE.json: "NCCL allreduce
// over NVLink of the small per-mode Gram/RHS partials").
//
// Every rank owns one exchange buffer (cudaMalloc'd by the library, exported with a CUDA IPC
// handle and opened by every peer of the node, so each rank holds W device pointers):
//     [ flag: last published epoch (u64) | pad to 128 B | slot 0 | slot 1 ]   (slots: doubles)
// Exchange number e (1, 2, … — the same sequence on every rank) uses slot e & 1:
//   1. the producer of this rank's partial (the SOLVE_PROJECT kernel, or peer_allreduce)
//      writes it into its own slot e & 1;
//   2. the consumer kernel publishes flag = e (system-scope release after a system fence),
//      then waits until every peer's flag ≥ e (system-scope acquire), and sums slot e & 1 of
//      all W ranks in rank order 0..W−1 — the same sum, bit for bit, on every rank;
//   3. the last CTA of the consumer kernel to finish advances this rank's epoch counter to e.
// Two slots suffice: a rank writes slot e & 1 again only in exchange e + 2, after it has seen
// every peer publish e + 1, which each peer does only after finishing exchange e.  A rank
// reaches the wait only after its own partial is complete (kernel boundary), and every CTA
// publishes before it waits, so no CTA can spin on a flag that only a not-yet-resident CTA of
// the same kernel would set.
//
// The consumer for the block partials is the solve itself (block_solve / block_solve_big with
// SOLVE_FROM_PROJ and a PeerCtx): the collective and the Cholesky solves are one kernel, no
// host-issued collective, nothing for the CPU to do inside the sweep graph.
#pragma once

#include <cstdint>

namespace ifctn {

constexpr int kPeerMax = 16;        // ranks of one node
constexpr int64_t kPeerHeader = 16;  // doubles before slot 0 (flag + pad: 128 B)

struct PeerCtx {
    double* bufs[kPeerMax];  // every rank's exchange buffer (own and peers', device pointers)
    int W, rank;
    int64_t slot_elems;      // doubles per slot
    unsigned long long* epoch;  // this rank's epoch counter (device)
    unsigned* arrive;           // arrival counter of the consumer kernel's CTAs (self-resetting)
};

__device__ __forceinline__ unsigned long long peer_next_epoch(const PeerCtx& X) {
    return *reinterpret_cast<volatile unsigned long long*>(X.epoch) + 1ull;
}

// this rank's slot for the exchange that follows the current epoch (producer side)
__device__ __forceinline__ double* peer_my_slot(const PeerCtx& X) {
    const unsigned long long e = peer_next_epoch(X);
    return X.bufs[X.rank] + kPeerHeader + (int64_t)(e & 1ull) * X.slot_elems;
}

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

constexpr unsigned long long kPeerTimeoutNs = 20ull * 1000ull * 1000ull * 1000ull;  // 20 s

// CTA-wide: publish epoch e, then wait for every rank's flag ≥ e (thread 0 spins).
__device__ __forceinline__ void peer_publish_wait(const PeerCtx& X, unsigned long long e) {
    if (threadIdx.x == 0) {
        __threadfence_system();
        st_release_sys(reinterpret_cast<unsigned long long*>(X.bufs[X.rank]), e);
        for (int r = 0; r < X.W; ++r) {
            const unsigned long long* f = reinterpret_cast<const unsigned long long*>(X.bufs[r]);
            unsigned spins = 0;
            unsigned long long t0 = 0;
            while (ld_acquire_sys(f) < e) {
                // watchdog: a peer that never publishes (a crashed or stuck rank) must not hang
                // this GPU — after kPeerTimeoutNs the kernel traps (a launch failure, reported
                // as IFCTN_E_CUDA by the next call) instead of spinning forever
                if ((++spins & 0x3ffu) == 0) {
                    unsigned long long t;
                    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
                    if (t0 == 0) t0 = t;
                    else if (t - t0 > kPeerTimeoutNs) __trap();
                }
            }
        }
    }
    __syncthreads();
}

// Σ_r slot_r[i], r = 0..W−1 in order (L1-bypassing loads: peers wrote these)
__device__ __forceinline__ double peer_sum(const PeerCtx& X, unsigned long long e, int64_t i) {
    const int64_t o = kPeerHeader + (int64_t)(e & 1ull) * X.slot_elems + i;
    double v = 0.0;
    for (int r = 0; r < X.W; ++r) v += __ldcv(X.bufs[r] + o);
    return v;
}

// CTA-wide, at the end of the consumer kernel: the last CTA advances the epoch counter to e.
__device__ __forceinline__ void peer_retire(const PeerCtx& X, unsigned long long e) {
    __syncthreads();
    if (threadIdx.x == 0) {
        if (atomicAdd(X.arrive, 1u) == gridDim.x - 1) {
            *X.arrive = 0u;
            *reinterpret_cast<volatile unsigned long long*>(X.epoch) = e;
            __threadfence();
        }
    }
}

// All-reduce (sum) of `count` ≤ slot_elems doubles in place, one CTA: the norms of a sweep
// (4 doubles), the RSE sums and the metric sums.
static __global__ void __launch_bounds__(256) peer_allreduce(const __grid_constant__ PeerCtx X, double* buf,
                                                             int64_t count) {
    const unsigned long long e = peer_next_epoch(X);
    double* mine = X.bufs[X.rank] + kPeerHeader + (int64_t)(e & 1ull) * X.slot_elems;
    for (int64_t i = threadIdx.x; i < count; i += blockDim.x) mine[i] = buf[i];
    __syncthreads();
    peer_publish_wait(X, e);
    for (int64_t i = threadIdx.x; i < count; i += blockDim.x) buf[i] = peer_sum(X, e, i);
    peer_retire(X, e);
}

// Protocol self-test: W virtual ranks in ONE cooperative launch on one device (blocks of
// rank r = blockIdx.x mod W; B200_PROFILING.md: ranks that wait on one another must not be
// separate launches on one GPU).  Every round each rank writes value(r, round, i) into its
// slot, publishes, waits, sums in rank order and compares with the closed form; the ranks'
// epoch counters advance like the library's.  errors[0] counts mismatches.
static __global__ void peer_selftest(PeerCtx X0, int rounds, int64_t n, unsigned* errors) {
    const int W = X0.W;
    const int r = blockIdx.x % W;
    PeerCtx X = X0;
    X.rank = r;
    X.epoch = X0.epoch + r;
    X.arrive = X0.arrive + r;
    const unsigned per_rank = gridDim.x / W;
    for (int round = 0; round < rounds; ++round) {
        const unsigned long long e = peer_next_epoch(X);
        // producer phase of rank r: its first CTA writes the slot
        if (blockIdx.x == (unsigned)r) {
            double* mine = X.bufs[r] + kPeerHeader + (int64_t)(e & 1ull) * X.slot_elems;
            for (int64_t i = threadIdx.x; i < n; i += blockDim.x) mine[i] = (double)((r + 1) * (round + 1)) + (double)i;
        }
        // (the library has a kernel boundary here; emulate it with a per-rank barrier)
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            unsigned* bar = X0.arrive + kPeerMax + r;
            const unsigned target = per_rank * (unsigned)(round + 1);
            atomicAdd(bar, 1u);
            while (*reinterpret_cast<volatile unsigned*>(bar) < target) {
            }
        }
        __syncthreads();
        peer_publish_wait(X, e);
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
            const double want = (double)(W * (W + 1) / 2) * (double)(round + 1) + (double)W * (double)i;
            if (peer_sum(X, e, i) != want) atomicAdd(errors, 1u);
        }
        // retire: last CTA of rank r advances its epoch; the others wait for it (the library
        // has the next kernel boundary here)
        __syncthreads();
        if (threadIdx.x == 0) {
            if (atomicAdd(X.arrive, 1u) == per_rank - 1) {
                *X.arrive = 0u;
                __threadfence();
                *reinterpret_cast<volatile unsigned long long*>(X.epoch) = e;
            }
            while (*reinterpret_cast<volatile unsigned long long*>(X.epoch) < e) {
            }
        }
        __syncthreads();
    }
}

}  // namespace ifctn
