// grid.cu — multi-instance driver (include/ifctn.h ifctn_grid_run).
//
// Host-side runtime on top of the public C-ABI: a pool of `concurrency` slots, each with a
// CUDA stream and a reusable workspace; instances are created into free slots wave by wave,
// their sweeps enqueued asynchronously (CUDA graphs on independent streams run
// concurrently), then each slot's results are read back and the contexts destroyed.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/ifctn.h"

namespace {

struct Slot {
    cudaStream_t stream = nullptr;
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    void* ws = nullptr;
    ifctn_ctx* ctx = nullptr;
    int inst = -1;
};

}  // namespace

extern "C" ifctn_status ifctn_grid_run(int order, const int64_t* dims, ifctn_dtype dtype,
                                       const void* observed, const uint8_t* mask, const void* truth,
                                       const ifctn_instance* instances, int count, int t_max,
                                       int concurrency, ifctn_instance_result* results) {
    if (!dims || !observed || !mask || !instances || !results || count < 0 || t_max < 1 || concurrency < 1)
        return IFCTN_E_ARG;
    if (count == 0) return IFCTN_OK;
    for (int q = 0; q < count; ++q) {
        results[q].rse = NAN;
        results[q].objective = NAN;
        results[q].seconds = 0.0;
        results[q].status = IFCTN_OK;
        if (!instances[q].ranks || !instances[q].init_factors) return IFCTN_E_ARG;
    }
    // workspace size: the largest instance
    size_t wmax = 0;
    for (int q = 0; q < count; ++q) {
        size_t b = 0;
        const ifctn_status st = ifctn_workspace_bytes(order, dims, instances[q].ranks, dtype, nullptr, &b);
        if (st != IFCTN_OK) {
            results[q].status = st;
            return st;
        }
        wmax = b > wmax ? b : wmax;
    }
    const int nslot = concurrency < count ? concurrency : count;
    std::vector<Slot> slots(nslot);
    ifctn_status first = IFCTN_OK;
    auto note = [&](int q, ifctn_status st) {
        if (st != IFCTN_OK) {
            if (q >= 0) results[q].status = st;
            if (first == IFCTN_OK) first = st;
        }
    };
    bool ok = true;
    for (Slot& s : slots) {
        ok = ok && cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking) == cudaSuccess;
        ok = ok && cudaEventCreate(&s.t0) == cudaSuccess && cudaEventCreate(&s.t1) == cudaSuccess;
        ok = ok && cudaMalloc(&s.ws, wmax) == cudaSuccess;
    }
    if (ok) {
        for (int base = 0; base < count; base += nslot) {
            // create this wave's contexts and enqueue their sweeps (asynchronous: eps = 0)
            for (int u = 0; u < nslot && base + u < count; ++u) {
                Slot& s = slots[u];
                const int q = base + u;
                s.inst = q;
                const ifctn_instance& in = instances[q];
                ifctn_status st = ifctn_create(&s.ctx, order, dims, in.ranks, dtype, in.rho, observed, mask,
                                               in.init_factors, s.ws, wmax, nullptr, s.stream, 0u);
                if (st == IFCTN_OK) {
                    cudaEventRecord(s.t0, s.stream);
                    st = ifctn_sweep(s.ctx, t_max, 0.0, nullptr, nullptr);
                    cudaEventRecord(s.t1, s.stream);
                }
                note(q, st);
            }
            // collect: device time, objective and RSE per instance, then release the wave
            for (int u = 0; u < nslot && base + u < count; ++u) {
                Slot& s = slots[u];
                const int q = s.inst;
                if (s.ctx && results[q].status == IFCTN_OK) {
                    ifctn_status st = ifctn_sync(s.ctx);
                    if (st == IFCTN_OK) {
                        float ms = 0.f;
                        cudaEventElapsedTime(&ms, s.t0, s.t1);
                        results[q].seconds = 1e-3 * ms;
                        st = ifctn_objective(s.ctx, &results[q].objective);
                    }
                    if (st == IFCTN_OK && truth) st = ifctn_rse(s.ctx, truth, &results[q].rse);
                    note(q, st);
                }
                if (s.ctx) ifctn_destroy(s.ctx);
                s.ctx = nullptr;
                s.inst = -1;
            }
        }
    } else {
        note(-1, IFCTN_E_CUDA);
    }
    for (Slot& s : slots) {
        if (s.ws) cudaFree(s.ws);
        if (s.t0) cudaEventDestroy(s.t0);
        if (s.t1) cudaEventDestroy(s.t1);
        if (s.stream) cudaStreamDestroy(s.stream);
    }
    return first;
}
