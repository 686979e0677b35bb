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
                                                          int req_end, int n_tree_rows, int32_t* __restrict__ out,
                                                          void* ws) {
    const int row_lo = tree_offsets[req_begin];
    int row_hi = tree_offsets[req_end];
    if (row_lo < 0 || row_hi > n_tree_rows) {  // rows past the logits tensor / the argmax buffer: flag, clamp
        if (blockIdx.x == 0 && threadIdx.x == 0) set_dev_error(ws, AS_DEV_ROWS_OVERFLOW, req_end - 1);
        row_hi = min(row_hi, n_tree_rows);
    }
    const int row = row_lo + blockIdx.x;
    if (row_lo < 0 || row >= row_hi) return;
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
        constexpr int U = 4;  // 16-byte loads in flight per thread
        int v0 = threadIdx.x;
        for (; v0 + (U - 1) * (int)blockDim.x < nvec; v0 += U * blockDim.x) {
            uint4 raw[U];
#pragma unroll
            for (int u = 0; u < U; ++u) raw[u] = __ldcs(rv + v0 + u * blockDim.x);  // streamed once: evict-first
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const T* e = reinterpret_cast<const T*>(&raw[u]);
                const int vb = (v0 + u * blockDim.x) * kVec;
#pragma unroll
                for (int q = 0; q < kVec; ++q) {
                    float x = to_f<T>(e[q]);
                    nan |= (x != x);
                    better(bv, bi, x, vb + q);
                }
            }
        }
        for (int v = v0; v < nvec; v += blockDim.x) {
            uint4 raw = __ldcs(rv + v);
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
// Walk + commit: one CTA per request.  The request's tree (parent, draft token,
// target token) is staged in shared memory with coalesced loads; warp 0 walks
// it (each step = a few shared-memory round trips and one ballot per 32 nodes);
// then all 8 warps commit the path: every (path node, kv head, 16-byte chunk)
// vector of K and V is copied in one flattened, unrolled sweep, so the copy
// costs ~one memory round trip.
// ---------------------------------------------------------------------------
constexpr int kAccThreads = 256;
constexpr int kAccMaxNodes = 256;  // staged in smem; larger trees walk from global memory
constexpr int kAccMaxPath = 64;

struct AccSmem {
    int parent[kAccMaxNodes];
    int token[kAccMaxNodes];
    int target[kAccMaxNodes];
    int next[kAccMaxNodes];  // lowest-index child c of v with token[c] == target[v] (or INT_MAX)
    int path[kAccMaxPath];
    long long dst[kAccMaxPath];  // byte offset of the cache row for path position k (-1: skip)
    long long src[kAccMaxPath];  // byte offset of the k_tree/v_tree row of path node k
    int len;
};

// Cache-row byte offset of path position k (slot L + k of request i) or a
// negative code: -1 no slot, -2 page-table overflow, -3 page id out of range.
__device__ __forceinline__ long long slot_dst(const AcceptParams& p, int i, int L, int k, long long row_bytes) {
    const int slot = L + k;
    const int pi = slot / p.page_size;
    if (pi >= p.max_pages) return -2;
    const int page = __ldg(p.page_table + (size_t)i * p.max_pages + pi);
    if (page < 0 || page >= p.num_pages) return -3;
    return ((long long)page * p.n_kv * p.page_size + slot % p.page_size) * row_bytes;
}

// Copy the path rows' K/V (every (path node, kv head, 16-byte chunk) vector in
// one flattened, unrolled sweep) into the cache rows sm.dst[k]; kv_len_out = L + len.
__device__ __forceinline__ void commit_copy(const AcceptParams& p, AccSmem& sm, int i, int off, int L, int len) {
    const int tid = threadIdx.x;
    const long long row_bytes = (long long)p.head_dim * p.elem_bytes;
    const int vpr = (int)(row_bytes / 16);
    if (tid < kAccMaxPath) {
        const int k = tid;
        long long d = -1;
        if (k < len) {
            d = sm.dst[k];
            if (d == -2) set_dev_error(p.ws, AS_DEV_PAGE_OVERFLOW, i);
            if (d == -3) set_dev_error(p.ws, AS_DEV_BAD_PAGE, i);
        }
        sm.dst[k] = d;
        sm.src[k] = (k < len) ? (long long)(off + sm.path[k]) * p.n_kv * row_bytes : 0;
    }
    __syncthreads();
    const int per_k = p.n_kv * vpr;
    const int total = len * per_k;
    const long long head_dst = (long long)p.page_size * row_bytes;  // cache: [page][h][slot][d]
    constexpr int U = 4;
    for (int v0 = tid; v0 < total; v0 += U * kAccThreads) {
        uint4 kv[U], vv[U];
        long long dd[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int v = v0 + u * kAccThreads;
            dd[u] = -1;
            if (v < total) {
                const int k = v / per_k;
                const int rem = v - k * per_k;
                const int h = rem / vpr, c = rem - h * vpr;
                const long long d = sm.dst[k];
                if (d >= 0) {
                    const long long so = sm.src[k] + h * row_bytes + c * 16;
                    kv[u] = *reinterpret_cast<const uint4*>(p.k_tree + so);
                    vv[u] = *reinterpret_cast<const uint4*>(p.v_tree + so);
                    dd[u] = d + h * head_dst + c * 16;
                }
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (dd[u] >= 0) {
                *reinterpret_cast<uint4*>(p.k_cache + dd[u]) = kv[u];
                *reinterpret_cast<uint4*>(p.v_cache + dd[u]) = vv[u];
            }
        }
    }
    if (tid == 0) p.kv_len_out[i] = L + len;
}

__global__ void __launch_bounds__(kAccThreads) walk_commit_kernel(AcceptParams p) {
    __shared__ AccSmem sm;
    pdl_launch_dependents();
    pdl_wait();  // trees (select) and the attention's reads of kv_len / the cache
    const int tid = threadIdx.x;
    const int lane = lane_id();
    const long long row_bytes = (long long)p.head_dim * p.elem_bytes;
    if (p.do_walk) {
        const int i = p.req_begin + blockIdx.x;
        if (i >= p.req_end) return;
        // independent loads first: the commit's cache rows (kv_len -> page table)
        // resolve while the tree is staged and walked
        const int L = p.do_commit ? __ldg(p.kv_len + i) : 0;
        const int off = __ldg(p.tree_offsets + i);
        const int K = __ldg(p.tree_offsets + i + 1) - off;
        const int npath = min(p.max_path, kAccMaxPath);
        if (p.do_commit && tid >= kAccThreads - kAccMaxPath) {
            const int k = tid - (kAccThreads - kAccMaxPath);
            sm.dst[k] = k < npath ? slot_dst(p, i, L, k, row_bytes) : -1;
        }
        if (off + K > p.n_tree_rows) {
            if (tid == 0) set_dev_error(p.ws, AS_DEV_ROWS_OVERFLOW, i);
            return;
        }
        const bool staged = K <= kAccMaxNodes;
        if (staged) {
            for (int c = tid; c < K; c += kAccThreads) {
                sm.parent[c] = __ldg(p.tree_parent + off + c);
                sm.token[c] = __ldg(p.tree_tokens + off + c);
                sm.target[c] = __ldg(p.target_tokens + off + c);
                sm.next[c] = 0x7fffffff;
            }
            __syncthreads();
            // every edge at once: c is v's accepted child candidate when its draft
            // token equals v's target token; the lowest index wins (R13)
            for (int c = 1 + tid; c < K; c += kAccThreads) {
                const int v = sm.parent[c];
                if (v >= 0 && v < c && sm.token[c] == sm.target[v]) atomicMin(&sm.next[v], c);
            }
        }
        __syncthreads();
        if (warp_id() == 0) {
            int len = 0, tstar = -1;
            if (staged) {
                // the walk is now a pointer chase through next[] (lane 0)
                if (lane == 0 && K > 0) {
                    int v = 0;
                    len = 1;
                    sm.path[0] = 0;
                    for (;;) {
                        const int nx = sm.next[v];
                        if (nx == 0x7fffffff) break;
                        if (len >= p.max_path || len >= kAccMaxPath) {
                            set_dev_error(p.ws, AS_DEV_PATH_TOO_LONG, i);
                            break;
                        }
                        sm.path[len++] = nx;
                        v = nx;
                    }
                    tstar = sm.target[v];
                }
                len = __shfl_sync(0xffffffffu, len, 0);
                tstar = __shfl_sync(0xffffffffu, tstar, 0);
            } else if (K > 0) {
                // large trees: walk from global memory, one ballot per 32 nodes
                const int* par = p.tree_parent + off;
                const int* tok = p.tree_tokens + off;
                const int* tgt = p.target_tokens + off;
                int v = 0;
                len = 1;
                if (lane == 0) sm.path[0] = 0;
                for (;;) {
                    tstar = tgt[v];
                    int next = -1;
                    for (int c0 = v + 1; c0 < K; c0 += 32) {  // children follow their parent
                        const int c = c0 + lane;
                        const bool m = c < K && par[c] == v && tok[c] == tstar;
                        const unsigned b = __ballot_sync(0xffffffffu, m);
                        if (b) { next = c0 + __ffs(b) - 1; break; }
                    }
                    if (next < 0) break;
                    if (len >= p.max_path || len >= kAccMaxPath) {
                        if (lane == 0) set_dev_error(p.ws, AS_DEV_PATH_TOO_LONG, i);
                        break;
                    }
                    if (lane == 0) sm.path[len] = next;
                    ++len;
                    v = next;
                }
            }
            __syncwarp();
            // records: row i = {len, bonus, path[max_path]} (one contiguous int32 row per request)
            int32_t* rec = p.records ? p.accept_path + (size_t)i * (p.max_path + 2) : nullptr;
            int32_t* path = p.records ? rec + 2 : p.accept_path + (size_t)i * p.max_path;
            for (int k = lane; k < p.max_path; k += 32) path[k] = (k < len) ? sm.path[k] : -1;
            if (lane == 0) {
                if (p.records) {
                    rec[0] = len;
                    rec[1] = tstar;
                } else {
                    p.accept_len[i] = len;
                    p.bonus_token[i] = tstar;
                }
                sm.len = len;
            }
        }
        __syncthreads();
        if (p.do_commit) commit_copy(p, sm, i, off, L, sm.len);
    } else if (p.do_commit) {
        // COMMIT_ONLY over all requests [0, n_req)
        const int i = blockIdx.x;
        if (i >= p.n_req) return;
        const int L = __ldg(p.kv_len + i);
        const int off = __ldg(p.tree_offsets + i);
        const int32_t* rec = p.accept_path + (size_t)i * (p.max_path + 2);
        int len = p.records ? rec[0] : p.accept_len[i];
        if (len > p.max_path) len = p.max_path;
        if (len > kAccMaxPath) len = kAccMaxPath;
        if (len < 0) len = 0;
        const int32_t* path = p.records ? rec + 2 : p.accept_path + (size_t)i * p.max_path;
        if (tid < len) {
            sm.path[tid] = path[tid];
            sm.dst[tid] = slot_dst(p, i, L, tid, row_bytes);
        }
        __syncthreads();
        commit_copy(p, sm, i, off, L, len);
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
                    q.req_end, rows, argmax_buf, q.ws);
            else
                argmax_rows_kernel<float><<<rows, 512, 0, stream>>>(reinterpret_cast<const float*>(target_logits),
                                                                   vocab, q.tree_offsets, q.req_begin, q.req_end,
                                                                   rows, argmax_buf, q.ws);
            if (cudaGetLastError() != cudaSuccess) return -1;
        }
        q.target_tokens = argmax_buf;
    }
    const int nw = q.do_walk ? (q.req_end - q.req_begin) : q.n_req;
    if (nw <= 0) return 0;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nw);
    cfg.blockDim = dim3(kAccThreads);
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    cfg.attrs = attr;
    cfg.numAttrs = fill_launch_attrs(attr);
    if (cudaLaunchKernelEx(&cfg, walk_commit_kernel, q) != cudaSuccess) return -1;
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace as
