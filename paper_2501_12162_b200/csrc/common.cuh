// common.cuh -- shared device helpers of libadaserve (CUDA path only; the
// CPU oracle under oracle/ shares nothing with this file).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "../../include/adaserve.h"

namespace as {

// Workspace header (first 256 bytes of every workspace).
struct WsHeader {
    int32_t err_code;     // sticky first device error (AS_DEV_*)
    int32_t err_request;  // request index of that error
    uint32_t ticket;      // last-block counter of the select kernel (self-resetting)
    uint32_t pad[61];
};
static_assert(sizeof(WsHeader) == 256, "header size");

constexpr size_t kWsHeaderBytes = 256;
constexpr size_t kAttnTraceBytes = 4096 * 64;  // debug pipeline trace area of the attention workspace

__host__ __device__ inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

__device__ __forceinline__ void set_dev_error(void* ws, int code, int req) {
    WsHeader* h = reinterpret_cast<WsHeader*>(ws);
    if (atomicCAS(&h->err_code, 0, code) == 0) atomicExch(&h->err_request, req);
}

// Programmatic dependent launch (PDL): the hot path's kernels are launched
// with cudaLaunchAttributeProgrammaticStreamSerialization, so each one is
// dispatched while its predecessor is still running; it runs its prologue,
// then waits here for the predecessor's results.  Both are no-ops for a
// normally launched kernel.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Host: launch attributes of the hot path (PDL on unless AS_PDL=0).
int pdl_enabled();
inline int fill_launch_attrs(cudaLaunchAttribute* attr) {
    if (!pdl_enabled()) return 0;
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    return 1;
}

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ unsigned warp_id() { return threadIdx.x >> 5; }

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

}  // namespace as
