// nccl_lite.h — the four NCCL entry points the multi-GPU sweep uses, resolved at run time
// from the process's libnccl.so.2 (the copy torch already loaded when present), so the
// library has no link-time NCCL dependency and never mixes two NCCL builds in one process.
#pragma once

#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstddef>

namespace ifctn {

struct NcclUniqueId {
    char internal[128];
};

struct NcclLite {
    using InitFn = int (*)(void** comm, int nranks, NcclUniqueId id, int rank);
    using AllReduceFn = int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t);
    using DestroyFn = int (*)(void*);
    using ErrFn = const char* (*)(int);
    InitFn init = nullptr;
    AllReduceFn allreduce = nullptr;
    DestroyFn destroy = nullptr;
    ErrFn err = nullptr;

    static NcclLite* get() {
        static NcclLite inst;
        static bool tried = false;
        if (!tried) {
            tried = true;
            void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
            if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
            if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
            if (h) {
                inst.init = (InitFn)dlsym(h, "ncclCommInitRank");
                inst.allreduce = (AllReduceFn)dlsym(h, "ncclAllReduce");
                inst.destroy = (DestroyFn)dlsym(h, "ncclCommDestroy");
                inst.err = (ErrFn)dlsym(h, "ncclGetErrorString");
            }
        }
        if (!inst.init || !inst.allreduce || !inst.destroy) return nullptr;
        return &inst;
    }

    int commInitRank(void** comm, int nranks, const void* id, int rank) {
        NcclUniqueId u;
        const char* c = (const char*)id;
        for (int t = 0; t < 128; ++t) u.internal[t] = c[t];
        return init(comm, nranks, u, rank);
    }
    int allReduce(const void* s, void* r, size_t n, int dt, int op, void* comm, cudaStream_t st) {
        return allreduce(s, r, n, dt, op, comm, st);
    }
    int commDestroy(void* comm) { return destroy(comm); }
    const char* errorString(int r) { return err ? err(r) : "nccl error"; }
};

}  // namespace ifctn
