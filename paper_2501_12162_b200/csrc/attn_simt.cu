// attn_simt.cu -- K2f: as_tree_verify_attn for dtype AS_F32 (CUDA cores).
//
// Verification attention with reading R15: node j of request i
// attends to the committed prefix [0, kv_len[i]) (paged) plus its tree
// ancestors-or-self.  This fp32 path exists for the 1e-5 parity configuration
// (BASELINE config 1, a latency-bound single request); the bf16 product path is
// attn_tc.cu (tcgen05/TMEM).
//
// CTA = (request i, kv head g, block of 16 query rows); rows r = node*G + hh;
// 8 warps x 2 rows.  Keys are processed in large chunks (128 keys for d = 64,
// 64 for d = 128) so a whole c1 request is ONE chunk: the chunk's page ids are
// staged first, then its K (rows padded to d+1 floats: conflict-free column
// reads) and V in one sweep of independent loads; per row, every lane scores
// its keys with 4 independent partial sums, the chunk's max / exp / sum run in
// the warp, p goes to shared memory, and each lane accumulates its output dims
// over the chunk's keys (2 independent chains).  Online softmax across chunks
// in fp32 with accurate expf.
#include "params.cuh"

namespace as {

constexpr int kSimtRows = 16;  // 8 warps x 2 rows
constexpr int kRowsPerWarp = 2;

template <int D>
struct SimtCfg {
    static constexpr int KC = D <= 64 ? 128 : 64;  // keys per chunk
    static constexpr int DP = D + 1;
};

template <int D>
__global__ void __launch_bounds__(256) tree_attn_simt_kernel(SimtParams p) {
    constexpr int KC = SimtCfg<D>::KC;
    constexpr int DP = SimtCfg<D>::DP;
    constexpr int DL = D / 32;       // output dims per lane
    constexpr int KL = KC / 32;      // keys per lane in the scoring pass
    extern __shared__ float simt_smem[];
    float* sk = simt_smem;                       // [KC][DP]
    float* sv = sk + KC * DP;                    // [KC][D]
    float* sq = sv + KC * D;                     // [kSimtRows][D]
    float* sp = sq + kSimtRows * D;              // [kSimtRows][KC] probabilities of the chunk
    __shared__ unsigned long long anc[AS_MAX_TREE][AS_MAX_TREE / 64];
    __shared__ int spar[AS_MAX_TREE];
    __shared__ int spage[KC];
    pdl_launch_dependents();
    pdl_wait();

    const int i = blockIdx.x;
    const int g = blockIdx.y;
    const int rb = blockIdx.z;
    const int off = p.tree_offsets[i];
    const int K = p.tree_offsets[i + 1] - off;
    const int G = p.G;
    const int rows = K * G;
    if (rb * kSimtRows >= rows) return;
    if (K > AS_MAX_TREE) {
        if (threadIdx.x == 0 && rb == 0 && g == 0) set_dev_error(p.ws, AS_DEV_TREE_TOO_BIG, i);
        return;
    }
    if (off + K > p.n_tree_rows) {
        if (threadIdx.x == 0 && rb == 0 && g == 0) set_dev_error(p.ws, AS_DEV_ROWS_OVERFLOW, i);
        return;
    }
    // kv_len outside [0, max_pages * page_size] would read another request's
    // page-table row (or past the table): flag it and clamp, as the tcgen05 path does
    int L = p.kv_len[i];
    if (L < 0 || L > p.max_pages * p.page_size) {
        if (threadIdx.x == 0 && rb == 0 && g == 0) set_dev_error(p.ws, AS_DEV_PAGE_OVERFLOW, i);
        L = min(max(L, 0), p.max_pages * p.page_size);
    }
    const int lane = lane_id();
    const int warp = warp_id();

    // ancestor-or-self bitmasks (u in anc(j) <=> bit u of anc[j])
    for (int j = threadIdx.x; j < K; j += blockDim.x) spar[j] = p.tree_parent[off + j];
    __syncthreads();
    for (int j = threadIdx.x; j < K; j += blockDim.x) {
        for (int w = 0; w < AS_MAX_TREE / 64; ++w) anc[j][w] = 0;
        int u = j, steps = 0;
        bool bad = false;
        for (;;) {
            anc[j][u >> 6] |= 1ull << (u & 63);
            if (u == 0) break;
            int pu = spar[u];
            if (pu < 0 || pu >= u || ++steps > K) { bad = true; break; }
            u = pu;
        }
        if (bad && g == 0 && rb == 0) set_dev_error(p.ws, AS_DEV_BAD_PARENT, i);
    }
    // this block's query rows
    for (int x = threadIdx.x; x < kSimtRows * D; x += blockDim.x) {
        const int rl = x / D, e = x % D;
        const int r = rb * kSimtRows + rl;
        float val = 0.f;
        if (r < rows) {
            const int node = r / G, hh = r % G;
            val = p.q[((size_t)(off + node) * p.n_q + g * G + hh) * D + e];
        }
        sq[rl * D + e] = val;
    }

    float m[kRowsPerWarp], l[kRowsPerWarp], o[kRowsPerWarp][DL];
#pragma unroll
    for (int k = 0; k < kRowsPerWarp; ++k) {
        m[k] = -INFINITY;
        l[k] = 0.f;
#pragma unroll
        for (int c = 0; c < DL; ++c) o[k][c] = 0.f;
    }
    const int n_keys = L + K;  // prefix keys, then the tree's keys
    for (int k0 = 0; k0 < n_keys; k0 += KC) {
        const int nk = min(KC, n_keys - k0);
        __syncthreads();  // previous chunk fully consumed
        // page ids of the chunk's prefix keys (one dependent global load per key, all in parallel)
        for (int kk = threadIdx.x; kk < nk; kk += blockDim.x) {
            const int key = k0 + kk;
            int pg = -1;
            if (key < L) {
                pg = p.page_table[(size_t)i * p.max_pages + key / p.page_size];
                if (pg < 0 || pg >= p.num_pages) {
                    set_dev_error(p.ws, AS_DEV_BAD_PAGE, i);
                    pg = -1;
                }
            }
            spage[kk] = pg;
        }
        __syncthreads();
        // K/V rows as 16-byte vectors, 4 independent loads in flight per thread
        constexpr int V4 = D / 4;
#pragma unroll 4
        for (int x = threadIdx.x; x < nk * V4; x += blockDim.x) {
            const int kk = x / V4, e4 = x % V4;
            const int key = k0 + kk;
            float4 kv = make_float4(0.f, 0.f, 0.f, 0.f), vv = kv;
            if (key < L) {
                const int pg = spage[kk];
                if (pg >= 0) {
                    const size_t src = (((size_t)pg * p.n_kv + g) * p.page_size + key % p.page_size) * D + 4 * e4;
                    kv = *reinterpret_cast<const float4*>(p.k_cache + src);
                    vv = *reinterpret_cast<const float4*>(p.v_cache + src);
                }
            } else {
                const size_t src = ((size_t)(off + key - L) * p.n_kv + g) * D + 4 * e4;
                kv = *reinterpret_cast<const float4*>(p.k_tree + src);
                vv = *reinterpret_cast<const float4*>(p.v_tree + src);
            }
            float* kd = sk + kk * DP + 4 * e4;  // padded rows: scalar stores
            kd[0] = kv.x;
            kd[1] = kv.y;
            kd[2] = kv.z;
            kd[3] = kv.w;
            *reinterpret_cast<float4*>(sv + kk * D + 4 * e4) = vv;
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kRowsPerWarp; ++k) {
            const int rl = warp * kRowsPerWarp + k;
            const int r = rb * kSimtRows + rl;
            if (r >= rows) continue;  // warp-uniform
            const int node = r / G;
            const float* qr = sq + rl * D;
            // scores: lane owns keys lane + 32*j of the chunk
            float s[KL];
            float cmax = -INFINITY;
#pragma unroll
            for (int j = 0; j < KL; ++j) {
                const int kk = lane + 32 * j;
                const float* kr = sk + kk * DP;
                float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll 4
                for (int e = 0; e < D; e += 4) {
                    a0 = fmaf(qr[e], kr[e], a0);
                    a1 = fmaf(qr[e + 1], kr[e + 1], a1);
                    a2 = fmaf(qr[e + 2], kr[e + 2], a2);
                    a3 = fmaf(qr[e + 3], kr[e + 3], a3);
                }
                const float dot = (a0 + a1) + (a2 + a3);
                bool ok = kk < nk;
                const int key = k0 + kk;
                if (ok && key >= L) {
                    const int u = key - L;
                    ok = (anc[node][u >> 6] >> (u & 63)) & 1ull;
                }
                s[j] = ok ? dot * p.sm_scale : -INFINITY;
                cmax = fmaxf(cmax, s[j]);
            }
            cmax = warp_max(cmax);
            const float mn = fmaxf(m[k], cmax);
            if (mn == -INFINITY) continue;  // nothing visible yet (warp-uniform)
            const float alpha = expf(m[k] - mn);
            float psum = 0.f;
            float* prow = sp + rl * KC;
#pragma unroll
            for (int j = 0; j < KL; ++j) {
                const float pr = s[j] == -INFINITY ? 0.f : expf(s[j] - mn);
                psum += pr;
                prow[lane + 32 * j] = pr;
            }
            l[k] = l[k] * alpha + warp_sum(psum);
            m[k] = mn;
            __syncwarp();
            // output dims of this lane: d = lane + 32c; two independent chains over the keys
            float acc0[DL], acc1[DL];
#pragma unroll
            for (int c = 0; c < DL; ++c) {
                acc0[c] = 0.f;
                acc1[c] = 0.f;
            }
            int kk = 0;
            for (; kk + 1 < nk; kk += 2) {
                const float p0 = prow[kk], p1 = prow[kk + 1];
#pragma unroll
                for (int c = 0; c < DL; ++c) {
                    acc0[c] = fmaf(p0, sv[kk * D + lane + 32 * c], acc0[c]);
                    acc1[c] = fmaf(p1, sv[(kk + 1) * D + lane + 32 * c], acc1[c]);
                }
            }
            if (kk < nk) {
                const float p0 = prow[kk];
#pragma unroll
                for (int c = 0; c < DL; ++c) acc0[c] = fmaf(p0, sv[kk * D + lane + 32 * c], acc0[c]);
            }
#pragma unroll
            for (int c = 0; c < DL; ++c) o[k][c] = o[k][c] * alpha + (acc0[c] + acc1[c]);
            __syncwarp();
        }
    }
#pragma unroll
    for (int k = 0; k < kRowsPerWarp; ++k) {
        const int rl = warp * kRowsPerWarp + k;
        const int r = rb * kSimtRows + rl;
        if (r >= rows) continue;
        const int node = r / G, hh = r % G;
        const size_t orow = (size_t)(off + node) * p.n_q + g * G + hh;
        const float inv = 1.f / l[k];
#pragma unroll
        for (int c = 0; c < DL; ++c) p.out[orow * D + lane + 32 * c] = o[k][c] * inv;
        if (p.lse && lane == 0) p.lse[orow] = m[k] + logf(l[k]);
    }
}

template <int D>
static int launch_simt(const SimtParams& p, cudaStream_t stream) {
    constexpr int KC = SimtCfg<D>::KC;
    const int smem = (KC * SimtCfg<D>::DP + KC * D + kSimtRows * D + kSimtRows * KC) * 4;
    if (cudaFuncSetAttribute(tree_attn_simt_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) !=
        cudaSuccess)
        return -1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p.n_req, p.n_kv, (AS_MAX_TREE * p.G + kSimtRows - 1) / kSimtRows);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    cfg.attrs = attr;
    cfg.numAttrs = fill_launch_attrs(attr);
    if (cudaLaunchKernelEx(&cfg, tree_attn_simt_kernel<D>, p) != cudaSuccess) return -1;
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int launch_attn_simt(const SimtParams& p, int head_dim, cudaStream_t stream) {
    return head_dim == 64 ? launch_simt<64>(p, stream) : launch_simt<128>(p, stream);
}

}  // namespace as
