// selftest.cu -- as_selftest_umma: one-CTA tcgen05 GEMM that exercises the
// exact building blocks of the bf16 attention kernel (TMA SW128 tiles, K-major
// and MN-major UMMA shared-memory descriptors, the kind::f16 instruction
// descriptor, TMEM alloc / commit / 32x32b loads).  Debug and tests only.
#include "common.cuh"
#include "tc_ptx.cuh"

namespace as {

__global__ void __launch_bounds__(128, 1)
    umma_selftest_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                         float* d, int N, int K, int b_mn, const __nv_bfloat16* a_g, int a_tmem) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    unsigned char* sa = smem;                  // (K/64) chunks of [128 x 64]
    unsigned char* sb = smem + 2 * 128 * 128;  // K-major: (K/64) chunks of [N x 64]; MN-major: (N/64) chunks of [K x 64]
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 4 * 128 * 128);
    uint32_t* holder = reinterpret_cast<uint32_t*>(bar + 2);
    const int warp = warp_id(), lane = lane_id();
    if (threadIdx.x == 0) {
        ptx::mbar_init(bar, 1);
        ptx::mbar_init(bar + 1, 1);
        ptx::fence_mbar_init();
    }
    if (warp == 0) ptx::tmem_alloc(holder, 512);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *holder;
    if (a_tmem) {
        // stage A into TMEM columns [256, 256 + K/2): lane = row, bf16 pairs packed per column
        const int row = warp * 32 + lane;
        for (int c0 = 0; c0 < K / 2; c0 += 32) {
            uint32_t r[32];
            for (int j = 0; j < 32; ++j) {
                const int k = 2 * (c0 + j);
                __nv_bfloat162 h2 = __halves2bfloat162(a_g[(size_t)row * K + k], a_g[(size_t)row * K + k + 1]);
                r[j] = *reinterpret_cast<uint32_t*>(&h2);
            }
            ptx::tmem_st32(tmem + ((uint32_t)(warp * 32) << 16) + 256 + c0, r);
        }
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
        __syncthreads();
        ptx::tc_fence_after();
    }
    if (threadIdx.x == 0) {
        const int kch = K / 64;
        const uint32_t bytes = (uint32_t)(kch * 128 * 128 + K * N * 2);
        ptx::mbar_arrive_expect_tx(bar, bytes);
        for (int c = 0; c < kch; ++c) ptx::tma_load_2d(sa + c * 128 * 128, &tm_a, bar, c * 64, 0);
        if (!b_mn) {
            for (int c = 0; c < kch; ++c) ptx::tma_load_2d(sb + c * N * 128, &tm_b, bar, c * 64, 0);
        } else {
            for (int c = 0; c < N / 64; ++c) ptx::tma_load_2d(sb + c * K * 128, &tm_b, bar, c * 64, 0);
        }
        ptx::mbar_wait(bar, 0);
        ptx::tc_fence_after();
        const uint32_t idesc = ptx::idesc_bf16_f32(128, N, b_mn);
        const uint32_t a0 = ptx::smem_u32(sa), b0 = ptx::smem_u32(sb);
        for (int ks = 0; ks < K / 16; ++ks) {
            const int c = ks >> 2, kk = ks & 3;
            const uint64_t ad = ptx::sw128_desc(a0 + c * 128 * 128 + kk * 32, 0, 1024);
            uint64_t bd;
            if (!b_mn) bd = ptx::sw128_desc(b0 + c * N * 128 + kk * 32, 0, 1024);
            else bd = ptx::sw128_desc(b0 + ks * 16 * 128, K * 128, 1024);
            if (a_tmem) ptx::mma_bf16_ts(tmem, tmem + 256 + ks * 8, bd, idesc, ks > 0 ? 1u : 0u);
            else ptx::mma_bf16_ss(tmem, ad, bd, idesc, ks > 0 ? 1u : 0u);
        }
        ptx::mma_commit(bar + 1);
    }
    __syncwarp();
    ptx::mbar_wait(bar + 1, 0);
    ptx::tc_fence_after();
    const int row = warp * 32 + lane;
    for (int c0 = 0; c0 < N; c0 += 32) {
        uint32_t r[32];
        ptx::tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + c0, r);
        ptx::tmem_ld_wait();
        for (int j = 0; j < 32; ++j) d[(size_t)row * N + c0 + j] = __uint_as_float(r[j]);
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, 512);
    }
}

// CTA-pair variant (cluster of 2): D[256, N] = A[256, K] . B^T with one
// tcgen05.mma.cta_group::2 (M = 256) per 16-wide K step, issued by the leader.
// CTA r holds A rows [128 r, 128 r + 128) and the N half [r N/2, (r+1) N/2) of B
// (K-major B: N/2 rows; MN-major B (N = 128): the 64-column chunk r), loaded
// by 2-SM TMA that signals the leader's barrier; the result rows come back from
// each CTA's own TMEM.  bit 1 of b_mn: A staged in each CTA's TMEM (the P form).
__global__ void __launch_bounds__(128, 1)
    umma2_selftest_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                          float* d, int N, int K, int b_mn, const __nv_bfloat16* a_g, int a_tmem) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    unsigned char* sa = smem;                  // (K/64) chunks of [128 x 64]
    unsigned char* sb = smem + 2 * 128 * 128;  // K-major: (K/64) chunks of [N/2 x 64]; MN-major: [K x 64]
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 4 * 128 * 128);
    uint32_t* holder = reinterpret_cast<uint32_t*>(bar + 2);
    const int warp = warp_id(), lane = lane_id();
    const uint32_t rank = ptx::cluster_ctarank();
    if (threadIdx.x == 0) {
        ptx::mbar_init(bar, 1);
        ptx::mbar_init(bar + 1, 1);
        ptx::fence_mbar_init();
    }
    if (warp == 0) ptx::tmem_alloc_pair(holder, 512);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::cluster_sync();
    ptx::tc_fence_after();
    const uint32_t tmem = *holder;
    const int kch = K / 64;
    if (a_tmem) {
        const int row = warp * 32 + lane;
        const int grow = (int)rank * 128 + row;
        for (int c0 = 0; c0 < K / 2; c0 += 32) {
            uint32_t r[32];
            for (int j = 0; j < 32; ++j) {
                const int k = 2 * (c0 + j);
                __nv_bfloat162 h2 = __halves2bfloat162(a_g[(size_t)grow * K + k], a_g[(size_t)grow * K + k + 1]);
                r[j] = *reinterpret_cast<uint32_t*>(&h2);
            }
            ptx::tmem_st32(tmem + ((uint32_t)(warp * 32) << 16) + 256 + c0, r);
        }
        ptx::tmem_st_wait();
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::cluster_sync();
    ptx::tc_fence_after();
    if (threadIdx.x == 0) {
        const uint32_t lbar = ptx::leader_bar(bar);
        const uint32_t b_half = (uint32_t)(K * N);  // bytes of B per CTA (N/2 x K bf16)
        if (rank == 0) ptx::mbar_arrive_expect_tx(bar, 2u * ((a_tmem ? 0u : (uint32_t)(kch * 128 * 128)) + b_half));
        if (!a_tmem)
            for (int c = 0; c < kch; ++c) ptx::tma_load_2d_pair(sa + c * 128 * 128, &tm_a, lbar, c * 64, (int)rank * 128);
        if (!(b_mn & 1)) {
            for (int c = 0; c < kch; ++c) ptx::tma_load_2d_pair(sb + c * (N / 2) * 128, &tm_b, lbar, c * 64, (int)rank * (N / 2));
        } else {
            ptx::tma_load_2d_pair(sb, &tm_b, lbar, (int)rank * 64, 0);
        }
        if (rank == 0) {
            ptx::mbar_wait(bar, 0);
            ptx::tc_fence_after();
            const uint32_t idesc = ptx::idesc_bf16_f32(256, N, b_mn & 1);
            const uint32_t a0 = ptx::smem_u32(sa), b0 = ptx::smem_u32(sb);
            for (int ks = 0; ks < K / 16; ++ks) {
                const int c = ks >> 2, kk = ks & 3;
                const uint64_t ad = ptx::sw128_desc(a0 + c * 128 * 128 + kk * 32, 0, 1024);
                uint64_t bd;
                if (!(b_mn & 1)) bd = ptx::sw128_desc(b0 + c * (N / 2) * 128 + kk * 32, 0, 1024);
                else bd = ptx::sw128_desc(b0 + ks * 16 * 128, K * 128, 1024);
                if (a_tmem) ptx::mma_bf16_ts_pair(tmem, tmem + 256 + ks * 8, bd, idesc, ks > 0 ? 1u : 0u);
                else ptx::mma_bf16_ss_pair(tmem, ad, bd, idesc, ks > 0 ? 1u : 0u);
            }
            ptx::mma_commit_pair(bar + 1, 0x3);
        }
    }
    __syncwarp();
    ptx::mbar_wait(bar + 1, 0);
    ptx::tc_fence_after();
    const int row = (int)rank * 128 + warp * 32 + lane;
    for (int c0 = 0; c0 < N; c0 += 32) {
        uint32_t r[32];
        ptx::tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + c0, r);
        ptx::tmem_ld_wait();
        for (int j = 0; j < 32; ++j) d[(size_t)row * N + c0 + j] = __uint_as_float(r[j]);
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::cluster_sync();
    if (warp == 0) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc_pair(tmem, 512);
    }
}

int launch_umma2_selftest(const CUtensorMap* ma, const CUtensorMap* mb, float* d, int N, int K, int b_mn,
                          const void* a_g, int a_tmem, cudaStream_t stream) {
    const int smem = 4 * 128 * 128 + 64 + 1024;
    if (cudaFuncSetAttribute(umma2_selftest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
        return -1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, umma2_selftest_kernel, *ma, *mb, d, N, K, b_mn,
                           reinterpret_cast<const __nv_bfloat16*>(a_g), a_tmem) != cudaSuccess)
        return -1;
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int launch_umma_selftest(const CUtensorMap* ma, const CUtensorMap* mb, float* d, int N, int K, int b_mn,
                         const void* a_g, int a_tmem, cudaStream_t stream) {
    const int smem = 4 * 128 * 128 + 64 + 1024;
    if (cudaFuncSetAttribute(umma_selftest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
        return -1;
    umma_selftest_kernel<<<1, 128, smem, stream>>>(*ma, *mb, d, N, K, b_mn,
                                                   reinterpret_cast<const __nv_bfloat16*>(a_g), a_tmem);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace as
