// attn_simt.cu -- K2f: as_tree_verify_attn for dtype AS_F32 (CUDA cores).
//
// Verification attention with reading R15: node j of request i
// attends to the committed prefix [0, kv_len[i]) (paged) plus its tree
// ancestors-or-self.  This fp32 path exists for the 1e-5 parity configuration
// (BASELINE config 1); the bf16 product path is attn_tc.cu (tcgen05/TMEM).
//
// CTA = (request i, kv head g, block of 16 query rows); rows r = node*G + hh.
// 8 warps x 2 rows each.  Keys are staged 32 at a time in shared memory (rows
// padded to d+1 floats: conflict-free column reads); each lane owns one key of
// the tile for the q.k dot product and d/32 output dims for P.V; online
// softmax in fp32 with accurate expf.
#include "params.cuh"

namespace as {

constexpr int kSimtRows = 16;  // 8 warps x 2 rows
constexpr int kRowsPerWarp = 2;
constexpr int kSimtKeys = 32;


template <int D>
__global__ void __launch_bounds__(256) tree_attn_simt_kernel(SimtParams p) {
    constexpr int DP = D + 1;
    constexpr int DL = D / 32;  // output dims per lane
    __shared__ float sq[kSimtRows][D];  // broadcast reads: no padding needed
    __shared__ float sk[kSimtKeys][DP];
    __shared__ float sv[kSimtKeys][D];
    __shared__ unsigned long long anc[AS_MAX_TREE][2];
    __shared__ int spar[AS_MAX_TREE];
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
    const int L = p.kv_len[i];
    const int lane = lane_id();
    const int warp = warp_id();

    // ancestor-or-self bitmasks (u in anc(j) <=> bit u of anc[j])
    for (int j = threadIdx.x; j < K; j += blockDim.x) spar[j] = p.tree_parent[off + j];
    __syncthreads();
    for (int j = threadIdx.x; j < K; j += blockDim.x) {
        unsigned long long a0 = 0, a1 = 0;
        int u = j, steps = 0;
        bool bad = false;
        for (;;) {
            if (u < 64) a0 |= 1ull << u; else a1 |= 1ull << (u - 64);
            if (u == 0) break;
            int pu = spar[u];
            if (pu < 0 || pu >= u || ++steps > K) { bad = true; break; }
            u = pu;
        }
        if (bad && g == 0 && rb == 0) set_dev_error(p.ws, AS_DEV_BAD_PARENT, i);
        anc[j][0] = a0;
        anc[j][1] = a1;
    }
    // stage this block's query rows
    for (int x = threadIdx.x; x < kSimtRows * D; x += blockDim.x) {
        const int rl = x / D, e = x % D;
        const int r = rb * kSimtRows + rl;
        float val = 0.f;
        if (r < rows) {
            const int node = r / G, hh = r % G;
            val = p.q[((size_t)(off + node) * p.n_q + g * G + hh) * D + e];
        }
        sq[rl][e] = val;
    }
    __syncthreads();

    float m[kRowsPerWarp], l[kRowsPerWarp], o[kRowsPerWarp][DL];
#pragma unroll
    for (int k = 0; k < kRowsPerWarp; ++k) {
        m[k] = -INFINITY;
        l[k] = 0.f;
#pragma unroll
        for (int c = 0; c < DL; ++c) o[k][c] = 0.f;
    }
    const int n_prefix_tiles = (L + kSimtKeys - 1) / kSimtKeys;
    const int n_tree_tiles = (K + kSimtKeys - 1) / kSimtKeys;
    const int n_tiles = n_prefix_tiles + n_tree_tiles;
    for (int t = 0; t < n_tiles; ++t) {
        const bool is_tree = t >= n_prefix_tiles;
        const int key0 = is_tree ? (t - n_prefix_tiles) * kSimtKeys : t * kSimtKeys;
        const int nvalid = is_tree ? min(kSimtKeys, K - key0) : min(kSimtKeys, L - key0);
        __syncthreads();
        for (int x = threadIdx.x; x < kSimtKeys * D; x += blockDim.x) {
            const int kk = x / D, e = x % D;
            float kv = 0.f, vv = 0.f;
            if (kk < nvalid) {
                if (is_tree) {
                    const size_t src = ((size_t)(off + key0 + kk) * p.n_kv + g) * D + e;
                    kv = p.k_tree[src];
                    vv = p.v_tree[src];
                } else {
                    const int tpos = key0 + kk;
                    const int page = p.page_table[(size_t)i * p.max_pages + tpos / p.page_size];
                    if (page >= 0 && page < p.num_pages) {
                        const size_t src = (((size_t)page * p.n_kv + g) * p.page_size + tpos % p.page_size) * D + e;
                        kv = p.k_cache[src];
                        vv = p.v_cache[src];
                    } else if (e == 0) {
                        set_dev_error(p.ws, AS_DEV_BAD_PAGE, i);
                    }
                }
            }
            sk[kk][e] = kv;
            sv[kk][e] = vv;
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kRowsPerWarp; ++k) {
            const int rl = warp * kRowsPerWarp + k;
            const int r = rb * kSimtRows + rl;
            if (r >= rows) continue;  // warp-uniform
            const int node = r / G;
            // lane = key of this tile
            float dot = 0.f;
#pragma unroll 8
            for (int e = 0; e < D; ++e) dot = fmaf(sq[rl][e], sk[lane][e], dot);
            float s = dot * p.sm_scale;
            bool ok = lane < nvalid;
            if (is_tree && ok) {
                const int u = key0 + lane;
                ok = (anc[node][u >> 6] >> (u & 63)) & 1ull;
            }
            s = ok ? s : -INFINITY;
            const float tmax = warp_max(s);
            const float mn = fmaxf(m[k], tmax);
            if (mn == -INFINITY) continue;  // nothing visible yet
            const float alpha = expf(m[k] - mn);
            const float pr = ok ? expf(s - mn) : 0.f;
            l[k] = l[k] * alpha + warp_sum(pr);
            m[k] = mn;
#pragma unroll
            for (int c = 0; c < DL; ++c) o[k][c] *= alpha;
            for (int j = 0; j < nvalid; ++j) {
                const float pj = __shfl_sync(0xffffffffu, pr, j);
#pragma unroll
                for (int c = 0; c < DL; ++c) o[k][c] = fmaf(pj, sv[j][lane + 32 * c], o[k][c]);
            }
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

int launch_attn_simt(const SimtParams& p, int head_dim, cudaStream_t stream) {
    dim3 grid(p.n_req, p.n_kv, (AS_MAX_TREE * p.G + kSimtRows - 1) / kSimtRows);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(256);
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    cfg.attrs = attr;
    cfg.numAttrs = fill_launch_attrs(attr);
    const cudaError_t e = head_dim == 64 ? cudaLaunchKernelEx(&cfg, tree_attn_simt_kernel<64>, p)
                                         : cudaLaunchKernelEx(&cfg, tree_attn_simt_kernel<128>, p);
    if (e != cudaSuccess) return -1;
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace as
