// launch.cuh -- every kernel of the library is launched through launch_k():
// cudaLaunchKernelEx with Programmatic Dependent Launch (PDL) allowed, so the
// next kernel of the block is scheduled while the previous one drains and its
// prologue (mbarrier init, TMEM alloc, tensor-map prefetch, weight/bias
// staging) overlaps that tail.  Every kernel calls pdl_wait() before its first
// access to memory written by an earlier kernel (griddepcontrol.wait returns
// once the prerequisite grid has completed and its writes are visible), and
// pdl_trigger() once it no longer needs to delay its dependents.
// On by default; LASNET_PDL=0 disables it (see pdl_enabled).
#pragma once
#include <cstdio>
#include <cstdlib>
#include <utility>
#include <cuda_runtime.h>

namespace lasnet {

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// PDL is on by default (LASNET_PDL=0: off): as CUDA-graph replays the LAS-R101 forward
// takes 5.57 instead of 5.72 ms and the configs[1] block 84.0 instead of 88.1 us (round 2;
// round 1 measured it neutral on the block before the kernels' prologues grew).
inline bool pdl_enabled() {
    static const bool on = [] {
        const char *e = getenv("LASNET_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

// LASNET_SYNC_DEBUG=1: synchronise after every launch and name the kernel that failed (debugging only).
inline bool sync_debug() {
    static const bool on = [] {
        const char *e = getenv("LASNET_SYNC_DEBUG");
        return e && e[0] == '1';
    }();
    return on;
}
template <typename K>
inline cudaError_t debug_check(K kern, cudaError_t e, cudaStream_t st) {
    if (!sync_debug()) return e;
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
        const char *name = "?";
        cudaFuncGetName(&name, reinterpret_cast<const void *>(kern));
        fprintf(stderr, "lasnet: kernel %s failed: %s\n", name, cudaGetErrorString(e));
    }
    return e;
}

template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return debug_check(kern, cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...), st);
}

// A cooperative launch (cudaLaunchAttributeCooperative): the runtime guarantees
// that every CTA of the grid is co-resident, or fails the launch (then nothing
// runs) -- required by kernels that spin in a software grid barrier.
template <typename... KArgs, typename... Args>
cudaError_t launch_k_coop(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                          Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    return debug_check(kern, cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...), st);
}

// The same with a 1-D thread-block cluster of `cluster` CTAs (grid.x % cluster == 0).
template <typename... KArgs, typename... Args>
cudaError_t launch_k_cluster(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, int cluster,
                             Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    int na = 0;
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = (unsigned)cluster;
    at[na].val.clusterDim.y = 1;
    at[na].val.clusterDim.z = 1;
    ++na;
    if (pdl_enabled()) {
        at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    return debug_check(kern, cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...), st);
}

}  // namespace lasnet
