// Shared device helpers for the walkjoin B200 kernels (sm_100a).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/walkjoin_b200.h"

namespace wj {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ULL;
constexpr unsigned kFull = 0xffffffffu;

// splitmix64 finalizer: reference _kernels.py:22-27
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// start state of node u's stream: reference _kernels.py:47-50
__host__ __device__ __forceinline__ uint64_t node_stream_state(uint64_t seed, int64_t u) {
    return mix64(seed + kGolden * ((uint64_t)u + 1ULL));
}

// multiply-shift draw of _kernels.py:36-39: ((z >> 32) * deg) >> 32, deg < 2^31
__device__ __forceinline__ uint32_t bounded(uint64_t z, uint32_t deg) {
    return __umulhi((uint32_t)(z >> 32), deg);
}

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ unsigned lanemask_le() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_le;" : "=r"(m));
    return m;
}

// exact q = p / d for p < 2^16, d < 2^16 with magic = floor(2^32 / d) + 1
__host__ __device__ __forceinline__ uint32_t div_magic(uint32_t d) {
    return (uint32_t)((0x100000000ULL / d) + 1ULL);
}
__device__ __forceinline__ uint32_t fast_div16(uint32_t p, uint32_t magic) {
    return __umulhi(p, magic);
}

__host__ __device__ __forceinline__ int bits_for(uint64_t v) {  // bits to hold values in [0, v]
    int b = 0;
    while (b < 64 && (v >> b) != 0) ++b;
    return b == 0 ? 1 : b;
}

// Ampere-style asynchronous global -> shared copies (LDGSTS): a thread issues
// all of its staging copies back to back instead of serialising one L2
// round trip per loop iteration.
__device__ __forceinline__ void cp_async4(void *smem, const void *gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"((uint32_t)__cvta_generic_to_shared(smem)),
                 "l"(gmem));
}
__device__ __forceinline__ void cp_async8(void *smem, const void *gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"((uint32_t)__cvta_generic_to_shared(smem)),
                 "l"(gmem));
}
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((uint32_t)__cvta_generic_to_shared(smem)),
                 "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
// wait until at most one committed group (the most recent) is still in flight
__device__ __forceinline__ void cp_async_wait_group1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

// Programmatic dependent launch (PDL): a kernel launched with
// launch_pdl() may start while its stream predecessor is still running; it
// must pdl_wait() before touching the predecessor's outputs (a no-op when it
// was launched normally).  pdl_trigger() lets this kernel's own dependents
// get scheduled early.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                              Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, args...);
}

// per-thread error string for wj_last_error()
void set_error(const char *fmt, ...);

inline int check_launch(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error("%s: %s", what, cudaGetErrorString(e));
        return WJ_ERR_CUDA;
    }
    return WJ_OK;
}

int sm_count();

}  // namespace wj
