// membench.cu -- as_debug_stream_bw: HBM streaming micro-benchmark used to size
// the attention kernel's load path (debug / tuning only, not on the hot path).
//
// Every CTA streams chunks of `chunk_bytes` from `src` (chunk order given by
// `order`, e.g. a random page permutation) into a shared-memory ring of
// `stages` slots and discards them.  mode 0: one thread issues 1-D bulk copies
// (cp.async.bulk, the TMA engine); mode 1: two threads issue alternately;
// mode 2: plain 16-byte vector loads by all 256 threads (LSU path).
#include "common.cuh"
#include "tc_ptx.cuh"

namespace as {

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            ptx::smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(ptx::smem_u32(bar))
        : "memory");
}

// mode 3/4: like 0/1 but each chunk is fetched as a 3-D TENSOR box
// {64 elems, rows, 2 halves} with SWIZZLE_128B from a [rows][128] bf16 view
// (exactly the attention kernel's K/V tile loads); chunk_bytes = rows * 256.
__global__ void __launch_bounds__(256, 1)
    stream_bw_kernel(const unsigned char* __restrict__ src, const int* __restrict__ order, int n_chunks,
                     int chunk_bytes, int stages, int mode, unsigned long long* sink,
                     const __grid_constant__ CUtensorMap tmap) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)stages * chunk_bytes);
    const int tid = threadIdx.x;
    const bool tensor = mode >= 3;
    const int rows_per_chunk = chunk_bytes / 256;
    int nthr_sel = 1;
    if (mode == 1 || mode == 4) nthr_sel = 2;
    if (mode == 5) nthr_sel = 4;
    if (mode == 6) nthr_sel = 8;
    if (tensor) mode = 0;
    else if (mode == 1) mode = 0;
    if (mode <= 1) {
        if (tid == 0) {
            for (int s = 0; s < stages; ++s) ptx::mbar_init(bars + s, 1);
            ptx::fence_mbar_init();
        }
        __syncthreads();
        const int nthr = nthr_sel;
        if (tid < nthr) {
            // thread tid owns stages tid, tid+nthr, ... and chunks k = blockIdx + (tid + j*nthr)*grid
            const int my_stages = (stages - tid + nthr - 1) / nthr;
            const int kstep = nthr * gridDim.x;
            int k = blockIdx.x + tid * gridDim.x;
            int primed = 0;
            for (int j = 0; j < my_stages && k < n_chunks; ++j, k += kstep, ++primed) {
                const int st = tid + j * nthr;
                ptx::mbar_arrive_expect_tx(bars + st, chunk_bytes);
                if (tensor)
                    ptx::tma_load_3d(smem + (size_t)st * chunk_bytes, &tmap, bars + st, 0, order[k] * rows_per_chunk, 0);
                else
                    bulk_g2s(smem + (size_t)st * chunk_bytes, src + (size_t)order[k] * chunk_bytes, chunk_bytes, bars + st);
            }
            uint32_t it = 0;
            for (; k < n_chunks; k += kstep, ++it) {
                const int st = tid + (int)(it % my_stages) * nthr;
                ptx::mbar_wait(bars + st, (it / my_stages) & 1);
                ptx::mbar_arrive_expect_tx(bars + st, chunk_bytes);
                if (tensor)
                    ptx::tma_load_3d(smem + (size_t)st * chunk_bytes, &tmap, bars + st, 0, order[k] * rows_per_chunk, 0);
                else
                    bulk_g2s(smem + (size_t)st * chunk_bytes, src + (size_t)order[k] * chunk_bytes, chunk_bytes, bars + st);
            }
            for (int d = 0; d < primed; ++d, ++it) {
                const int st = tid + (int)(it % my_stages) * nthr;
                ptx::mbar_wait(bars + st, (it / my_stages) & 1);
            }
        }
        __syncthreads();
        if (tid == 0) sink[blockIdx.x] = *reinterpret_cast<unsigned long long*>(smem);
    } else {
        unsigned long long acc = 0;
        const int vec_per_chunk = chunk_bytes / 16;
        for (int k = blockIdx.x; k < n_chunks; k += gridDim.x) {
            const uint4* c = reinterpret_cast<const uint4*>(src + (size_t)order[k] * chunk_bytes);
#pragma unroll 4
            for (int v = tid; v < vec_per_chunk; v += 256) {
                uint4 x = __ldcs(c + v);
                acc ^= x.x ^ x.y ^ x.z ^ x.w;
            }
        }
        if (acc == 0x123456789ull) sink[blockIdx.x] = acc;
    }
}

int launch_stream_bw(const void* src, const int* order, int n_chunks, int chunk_bytes, int stages, int mode,
                     unsigned long long* sink, int grid, const CUtensorMap* tmap, cudaStream_t stream) {
    size_t smem = mode != 2 ? (size_t)stages * chunk_bytes + stages * 8 + 64 + 1024 : 0;
    if (smem > 48 * 1024 &&
        cudaFuncSetAttribute(stream_bw_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return -1;
    stream_bw_kernel<<<grid, 256, smem, stream>>>(reinterpret_cast<const unsigned char*>(src), order, n_chunks,
                                                  chunk_bytes, stages, mode, sink, *tmap);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace as
