// accept.cu -- K3: as_accept_tokens.  The acceptance walk "uses these logits
// to identify the verified tokens" under reading R13 (greedy argmax,
// lowest index on ties / caller-supplied per-node target samples) and the
// commit of the accepted path's K/V into the paged cache (R14, R16).
//
// Kernels:
//   argmax_rows_kernel   logits mode only: one CTA per tree row streams the
//                        vocab (16-byte vector loads) -> target token (HBM-bound).
//   walk_commit_kernel   one warp per request: the walk is a pointer chase, each
//                        step a 32-wide ballot over the request's nodes (children
//                        are located after their parent in topological order);
//                        FUSED mode then copies the path rows with 16-byte
//                        vectors through the page table and bumps kv_len.
#include "params.cuh"

namespace as {


// ---------------------------------------------------------------------------
// Greedy target tokens from logits: argmax with the lowest index on ties.
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ float to_f(T v);
template <>
__device__ __forceinline__ float to_f<float>(float v) { return v; }
template <>
__device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }

__device__ __forceinline__ void better(float& bv, int& bi, float v, int i) {
    // larger value wins; equal values -> lower index
    if (v > bv || (v == bv && i < bi)) { bv = v; bi = i; }
}

template <typename T>
__global__ void __launch_bounds__(512) argmax_rows_kernel(const T* __restrict__ logits, int vocab,
                                                          const int32_t* tree_offsets, int req_begin,
                                                          int req_end, int32_t* __restrict__ out, void* ws) {
    const int row_lo = tree_offsets[req_begin];
    const int row_hi = tree_offsets[req_end];
    const int row = row_lo + blockIdx.x;
    if (row >= row_hi) return;
    const T* r = logits + (size_t)row * vocab;
    float bv = -INFINITY;
    int bi = 0x7fffffff;
    bool nan = false;
    constexpr int kVec = 16 / sizeof(T);
    const bool aligned = ((reinterpret_cast<uintptr_t>(r) & 15u) == 0);
    int head = 0;
    if (aligned) {
        const int nvec = vocab / kVec;
        const uint4* rv = reinterpret_cast<const uint4*>(r);
        for (int v = threadIdx.x; v < nvec; v += blockDim.x) {
            uint4 raw = __ldcs(rv + v);  // streamed once: evict-first
            const T* e = reinterpret_cast<const T*>(&raw);
#pragma unroll
            for (int q = 0; q < kVec; ++q) {
                float x = to_f<T>(e[q]);
                nan |= (x != x);
                better(bv, bi, x, v * kVec + q);
            }
        }
        head = nvec * kVec;
    }
    for (int t = head + threadIdx.x; t < vocab; t += blockDim.x) {
        float x = to_f<T>(r[t]);
        nan |= (x != x);
        better(bv, bi, x, t);
    }
    // -inf rows: index stays at the first -inf -> handle with bi init
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        float ov = __shfl_xor_sync(0xffffffffu, bv, o);
        int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        better(bv, bi, ov, oi);
    }
    __shared__ float sv[32];
    __shared__ int si[32];
    __shared__ int snan;
    if (threadIdx.x == 0) snan = 0;
    __syncthreads();
    if (nan) snan = 1;
    if (lane_id() == 0) { sv[warp_id()] = bv; si[warp_id()] = bi; }
    __syncthreads();
    if (threadIdx.x < 32) {
        const int nw = blockDim.x / 32;
        bv = threadIdx.x < (unsigned)nw ? sv[threadIdx.x] : -INFINITY;
        bi = threadIdx.x < (unsigned)nw ? si[threadIdx.x] : 0x7fffffff;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            float ov = __shfl_xor_sync(0xffffffffu, bv, o);
            int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            better(bv, bi, ov, oi);
        }
        if (threadIdx.x == 0) {
            out[row] = (bi == 0x7fffffff) ? 0 : bi;  // all -inf row: index 0 (oracle: strict '>' from 0)
            if (snan) {
                // find the request of this row for the error record
                set_dev_error(ws, AS_DEV_NAN_LOGIT, -1);
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Walk + commit: one warp per request.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void commit_request(const AcceptParams& p, int i, int len, int p0, int p1) {
    const int lane = lane_id();
    const int off = p.tree_offsets[i];
    const int L = p.kv_len[i];
    const size_t row_bytes = (size_t)p.head_dim * p.elem_bytes;
    const int vec_per_row = (int)(row_bytes / 16);
    const int per_node = p.n_kv * vec_per_row;  // 16-byte vectors per node per tensor
    bool bad = false;
    for (int k = 0; k < len; ++k) {
        const int pk = (k < 32) ? __shfl_sync(0xffffffffu, p0, k) : __shfl_sync(0xffffffffu, p1, k - 32);
        const int node = off + pk;
        const int slot = L + k;
        const int pi = slot / p.page_size;
        if (pi >= p.max_pages) { bad = true; break; }
        const int page = p.page_table[(size_t)i * p.max_pages + pi];
        if (page < 0 || page >= p.num_pages) {
            if (lane == 0) set_dev_error(p.ws, AS_DEV_BAD_PAGE, i);
            continue;
        }
        for (int v = lane; v < per_node; v += 32) {
            const int h = v / vec_per_row;
            const int c = v % vec_per_row;
            const size_t src = ((size_t)node * p.n_kv + h) * row_bytes + (size_t)c * 16;
            const size_t dst = (((size_t)page * p.n_kv + h) * p.page_size + slot % p.page_size) * row_bytes +
                               (size_t)c * 16;
            *reinterpret_cast<uint4*>(p.k_cache + dst) = *reinterpret_cast<const uint4*>(p.k_tree + src);
            *reinterpret_cast<uint4*>(p.v_cache + dst) = *reinterpret_cast<const uint4*>(p.v_tree + src);
        }
    }
    if (bad && lane == 0) set_dev_error(p.ws, AS_DEV_PAGE_OVERFLOW, i);
    __syncwarp();
    if (lane == 0) p.kv_len[i] = L + len;
}

__global__ void __launch_bounds__(256) walk_commit_kernel(AcceptParams p) {
    const int lane = lane_id();
    const int wid = blockIdx.x * (blockDim.x / 32) + warp_id();
    if (p.do_walk) {
        const int i = p.req_begin + wid;
        if (i >= p.req_end) return;
        const int off = p.tree_offsets[i];
        const int K = p.tree_offsets[i + 1] - off;
        int32_t* path = p.accept_path + (size_t)i * p.max_path;
        if (off + K > p.n_tree_rows) {
            if (lane == 0) set_dev_error(p.ws, AS_DEV_ROWS_OVERFLOW, i);
            return;
        }
        int len = 0, tstar = -1;
        int p0 = -1, p1 = -1;  // path held in registers: lane k -> path[k], path[32+k]
        if (K > 0) {
            int v = 0;
            len = 1;
            if (lane == 0) p0 = 0;
            for (;;) {
                tstar = p.target_tokens[off + v];
                int next = -1;
                for (int c0 = v + 1; c0 < K; c0 += 32) {
                    const int c = c0 + lane;
                    const bool m = c < K && p.tree_parent[off + c] == v && p.tree_tokens[off + c] == tstar;
                    const unsigned b = __ballot_sync(0xffffffffu, m);
                    if (b) { next = c0 + __ffs(b) - 1; break; }
                }
                if (next < 0) break;
                if (len >= p.max_path || len >= 64) {
                    if (lane == 0) set_dev_error(p.ws, AS_DEV_PATH_TOO_LONG, i);
                    break;
                }
                if (len < 32) { if (lane == len) p0 = next; }
                else { if (lane == len - 32) p1 = next; }
                ++len;
                v = next;
            }
        }
        for (int k = lane; k < p.max_path; k += 32) {
            int val = -1;
            if (k < len) val = (k < 32) ? p0 : p1;
            path[k] = val;
        }
        // lanes >= 32 of the path live in p1; lanes write their own slots above
        // only for k < 64, which covers every walk (len <= 64).
        if (lane == 0) {
            p.accept_len[i] = len;
            p.bonus_token[i] = tstar;
        }
        if (p.do_commit) commit_request(p, i, len, p0, p1);
    } else if (p.do_commit) {
        // COMMIT_ONLY over all requests [0, n_req)
        const int i = wid;
        if (i >= p.n_req) return;
        int len = p.accept_len[i];
        if (len > p.max_path) len = p.max_path;
        if (len > 64) len = 64;
        const int32_t* path = p.accept_path + (size_t)i * p.max_path;
        const int p0 = (lane < len) ? path[lane] : -1;
        const int p1 = (lane + 32 < len) ? path[lane + 32] : -1;
        commit_request(p, i, len, p0, p1);
    }
}

int launch_accept(const AcceptParams& p, const void* target_logits, int logits_bf16, int vocab,
                  int32_t* argmax_buf, cudaStream_t stream) {
    AcceptParams q = p;
    if (q.do_walk && q.target_tokens == nullptr) {
        const int rows = q.n_tree_rows;
        if (rows > 0) {
            if (logits_bf16)
                argmax_rows_kernel<__nv_bfloat16><<<rows, 512, 0, stream>>>(
                    reinterpret_cast<const __nv_bfloat16*>(target_logits), vocab, q.tree_offsets, q.req_begin,
                    q.req_end, argmax_buf, q.ws);
            else
                argmax_rows_kernel<float><<<rows, 512, 0, stream>>>(reinterpret_cast<const float*>(target_logits),
                                                                   vocab, q.tree_offsets, q.req_begin, q.req_end,
                                                                   argmax_buf, q.ws);
            if (cudaGetLastError() != cudaSuccess) return -1;
        }
        q.target_tokens = argmax_buf;
    }
    const int nw = q.do_walk ? (q.req_end - q.req_begin) : q.n_req;
    if (nw <= 0) return 0;
    const int warps_per_block = 8;
    walk_commit_kernel<<<(nw + warps_per_block - 1) / warps_per_block, warps_per_block * 32, 0, stream>>>(q);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace as
