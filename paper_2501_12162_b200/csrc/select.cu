// select.cu -- K1: as_select_trees, Alg. 2 as a data-parallel
// kernel that is bit-identical to the sequential algorithm.
//
// The sequential loops of Alg. 2 are restated in closed form (DESIGN.md
// §Select, "O2"):
//   (1) pi_i = request i's non-root candidates sorted by (f-hat desc, idx asc)
//       -- GetTop inside one request always returns the next element of pi_i
//       because requests' candidate sets are disjoint;
//   (2) desired_i = number of pi_i entries the SLO loop would take
//       with unlimited budget: first k with 1 + sum_{t<k} f-hat >= A_cap, capped
//       by n_max and by C_i - 1; the fp64 sum runs in pi order, exactly as the
//       sequential loop adds (R9);
//   (3) the single shared budget is consumed in (A desc, id asc) order (P:L821,
//       R5): s_i = clamp(B0 - sum_{j before i} desired_j, 0, desired_i);
//   (4) the throughput loop takes the global top-R of the
//       remaining tails under (f-hat desc, req asc, idx asc) (R8),
//       R = min(B0 - sum s, sum tails); m_i = how many land in request i;
//   (5) tree i = root + pi_i[0 : s_i + m_i], emitted in ascending candidate
//       index (topological; ancestor-closed by App. B).
//
// One cooperative kernel launch:  every CTA sorts/thresholds 32 requests (one
// warp each: register bitonic sort with __shfl_xor_sync, lane-uniform fp64
// prefix loop); the last CTA to finish (threadfence + ticket) does (3)-(4):
// rank by A, block scan, an 8-bit-digit radix select over the 64-bit tail keys
// with warp-aggregated shared-memory histograms, ballot counts and the tree
// offsets; it then releases a generation flag and every CTA emits (5) its own
// 32 trees in parallel.
#include "common.cuh"

namespace as {

constexpr int kSelThreads = 1024;
constexpr int kSelWarps = kSelThreads / 32;
constexpr int kSelMaxReq = 4096;                // requests handled by one call
constexpr int kRemapWords = AS_MAX_CAND + 1;    // local indices 0..AS_MAX_CAND
constexpr int kBitmapWords = (AS_MAX_CAND + 1 + 31) / 32;

struct SelectParams {
    int n_req;
    const int32_t* cand_offsets;
    const int32_t* cand_parent;
    const float* cand_prob;
    const int32_t* cand_token;
    const double* A;
    int depth_d, n_max, budget;
    int32_t* tree_offsets;
    int32_t* tree_parent;
    int32_t* tree_src;
    int32_t* tree_depth;
    int32_t* tree_token;
    int32_t* slo_count;
    void* ws;
    int32_t* desired;   // [n]
    int32_t* take;      // [n]  s_i + m_i
    int32_t* stage_s;   // [n]  s_i
    int32_t* toff;      // [n+1] tree offsets (workspace copy)
    uint64_t* skey;     // [N - n] per-request sorted keys (f-hat bits << 32 | ~local idx)
};

__device__ __forceinline__ int n_nonroot(const SelectParams& p, int i, int* off_out) {
    int off = p.cand_offsets[i];
    int C = p.cand_offsets[i + 1] - off;
    *off_out = off;
    int nr = C - 1;
    if (nr < 0) nr = 0;
    if (nr > AS_MAX_CAND) nr = AS_MAX_CAND;
    return nr;
}

// ---------------------------------------------------------------------------
// Phase 1: warp per request -- sort pi_i and compute desired_i.
// ---------------------------------------------------------------------------
template <int E>
__device__ __forceinline__ void sort_request(const SelectParams& p, int i, int off, int nr) {
    constexpr int P = 32 * E;
    const int lane = lane_id();
    uint64_t key[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
        int s = e * 32 + lane;
        key[e] = 0ull;
        if (s < nr) {
            int j = s + 1;
            float f = p.cand_prob[off + j];
            int par = p.cand_parent[off + j];
            if (par < 0 || par >= j) {
                set_dev_error(p.ws, AS_DEV_BAD_PARENT, i);
            } else {
                float fp = p.cand_prob[off + par];
                if (!(f > 0.f) || !(f <= fp)) set_dev_error(p.ws, AS_DEV_BAD_PROB, i);
            }
            uint32_t fb = (f > 0.f) ? __float_as_uint(f) : 0u;   // positive floats order as uint32
            key[e] = ((uint64_t)fb << 32) | (uint64_t)(0xFFFFFFFFu - (uint32_t)j);
        }
    }
    // Bitonic sort, descending in position s = e*32 + lane.
#pragma unroll
    for (int k = 2; k <= P; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            uint64_t nk[E];
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int s = e * 32 + lane;
                uint64_t pv;
                if (j < 32) pv = __shfl_xor_sync(0xffffffffu, key[e], j);
                else pv = key[e ^ (j >> 5)];
                const bool desc = (s & k) == 0;
                const bool lo = (s & j) == 0;
                const uint64_t mx = key[e] > pv ? key[e] : pv;
                const uint64_t mn = key[e] > pv ? pv : key[e];
                nk[e] = (desc == lo) ? mx : mn;
            }
#pragma unroll
            for (int e = 0; e < E; ++e) key[e] = nk[e];
        }
    }
    const int sbase = off - i;  // sum_{j<i} (C_j - 1)
#pragma unroll
    for (int e = 0; e < E; ++e) {
        int s = e * 32 + lane;
        if (s < nr) p.skey[sbase + s] = key[e];
    }
    // SLO stage threshold with unlimited budget; lane-uniform,
    // sequential fp64 accumulation in pi order (identical to the oracle).
    const double a_cap = fmin(p.A[i], (double)p.depth_d + 1.0);
    const int lim = min(p.n_max, nr);
    double nacc = 1.0;
    int k = 0;
    while (k < lim && nacc < a_cap) {
        uint64_t v = key[0];
#pragma unroll
        for (int e = 1; e < E; ++e)
            if ((k >> 5) == e) v = key[e];
        v = __shfl_sync(0xffffffffu, v, k & 31);
        nacc += (double)__uint_as_float((uint32_t)(v >> 32));
        ++k;
    }
    if (lane == 0) p.desired[i] = k;
}

// ---------------------------------------------------------------------------
// Block-level helpers for the last CTA.
// ---------------------------------------------------------------------------
__device__ int block_sum_int(int v, int* red) {
    v = warp_sum(v);
    __syncthreads();
    if (lane_id() == 0) red[warp_id()] = v;
    __syncthreads();
    int t = 0;
    if (threadIdx.x < 32) {
        t = (threadIdx.x < (unsigned)kSelWarps) ? red[threadIdx.x] : 0;
        t = warp_sum(t);
        if (threadIdx.x == 0) red[32] = t;
    }
    __syncthreads();
    return red[32];
}

// Exclusive scan of data[0..n) in place (shared memory); returns the total.
__device__ int block_exclusive_scan(int* data, int n, int* red) {
    const int tid = threadIdx.x;
    const int chunk = (n + kSelThreads - 1) / kSelThreads;
    const int b = tid * chunk;
    const int e = min(n, b + chunk);
    int local = 0;
    for (int x = b; x < e; ++x) local += data[x];
    // warp inclusive scan of local
    int incl = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, incl, o);
        if ((int)lane_id() >= o) incl += y;
    }
    __syncthreads();
    if (lane_id() == 31) red[warp_id()] = incl;
    __syncthreads();
    if (threadIdx.x < 32) {
        int w = red[threadIdx.x];
        int wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, wi, o);
            if ((int)threadIdx.x >= o) wi += y;
        }
        red[threadIdx.x] = wi - w;  // exclusive warp offsets
        if (threadIdx.x == 31) red[32] = wi;
    }
    __syncthreads();
    int run = red[warp_id()] + incl - local;
    for (int x = b; x < e; ++x) {
        int v = data[x];
        data[x] = run;
        run += v;
    }
    int total = red[32];
    __syncthreads();
    return total;
}

__device__ __forceinline__ uint64_t tail_key(uint64_t sk, int i) {
    // global order (f-hat desc, req asc, idx asc): low word = ~(i*512 + idx)
    uint32_t idx = 0xFFFFFFFFu - (uint32_t)(sk & 0xFFFFFFFFull);
    return (sk & 0xFFFFFFFF00000000ull) | (uint64_t)(0xFFFFFFFFu - ((uint32_t)i * 512u + idx));
}

// ---------------------------------------------------------------------------
// The kernel.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kSelThreads, 1) select_trees_kernel(SelectParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ int red[33];
    __shared__ int hist[256];
    __shared__ int s_bcast[4];
    __shared__ int s_is_last;
    const int n = p.n_req;
    const int lane = lane_id();

    // ---- phase 1 ----
    {
        const int i = blockIdx.x * kSelWarps + (int)warp_id();
        if (i < n) {
            int off;
            int C = p.cand_offsets[i + 1] - p.cand_offsets[i];
            if (C < 1 || C - 1 > AS_MAX_CAND) {
                if (lane == 0) set_dev_error(p.ws, C < 1 ? AS_DEV_BAD_PARENT : AS_DEV_TOO_MANY_CAND, i);
            }
            int nr = n_nonroot(p, i, &off);
            if (nr <= 32) sort_request<1>(p, i, off, nr);
            else if (nr <= 64) sort_request<2>(p, i, off, nr);
            else if (nr <= 128) sort_request<4>(p, i, off, nr);
            else sort_request<8>(p, i, off, nr);
        }
    }
    __syncthreads();
    WsHeader* hdr = reinterpret_cast<WsHeader*>(p.ws);
    __shared__ unsigned s_gen0;
    if (threadIdx.x == 0) {
        s_gen0 = *reinterpret_cast<volatile unsigned*>(&hdr->pad[0]);  // generation before arriving
        __threadfence();
        unsigned t = atomicAdd(&hdr->ticket, 1u);
        s_is_last = (t == gridDim.x - 1);
        if (s_is_last) atomicExch(&hdr->ticket, 0u);  // everyone has arrived: reusable
    }
    __syncthreads();
    if (s_is_last) {
    __threadfence();

    // ---- phase 2 (last CTA) ----
    double* A_s = reinterpret_cast<double*>(smem_raw);                    // [n]
    int* ord_s = reinterpret_cast<int*>(A_s + n);                         // [n] desired in A order -> cum
    int* rank_s = ord_s + n;                                              // [n]

    for (int i = threadIdx.x; i < n; i += kSelThreads) A_s[i] = p.A[i];
    __syncthreads();
    // (3) rank by (A desc, id asc)
    for (int i = threadIdx.x; i < n; i += kSelThreads) {
        const double a = A_s[i];
        int r = 0;
        for (int j = 0; j < n; ++j) {
            const double b = A_s[j];
            r += (b > a) || (b == a && j < i);
        }
        rank_s[i] = r;
        ord_s[r] = __ldcg(p.desired + i);
    }
    __syncthreads();
    block_exclusive_scan(ord_s, n, red);
    const int B0 = p.budget - n;
    int my_s = 0, my_tail = 0;
    for (int i = threadIdx.x; i < n; i += kSelThreads) {
        int off;
        const int nr = n_nonroot(p, i, &off);
        const int des = __ldcg(p.desired + i);
        int s = B0 - ord_s[rank_s[i]];
        s = max(0, min(s, des));
        p.stage_s[i] = s;
        if (p.slo_count) p.slo_count[i] = s;
        my_s += s;
        my_tail += nr - s;
    }
    const int sum_s = block_sum_int(my_s, red);
    const int sum_tail = block_sum_int(my_tail, red);
    const int R = min(B0 - sum_s, sum_tail);
    __syncthreads();

    // (4) global top-R of the tails: radix select of the R-th largest key.
    int sh = 64;
    uint64_t prefix = 0;
    const bool select_all = (R >= sum_tail);
    const bool select_none = (R <= 0);
    if (!select_all && !select_none) {
        int need = R;
        bool done = false;
        while (!done && sh > 0) {
            sh -= 8;
            for (int x = threadIdx.x; x < 256; x += kSelThreads) hist[x] = 0;
            __syncthreads();
            for (int i = warp_id(); i < n; i += kSelWarps) {
                int off;
                const int nr = n_nonroot(p, i, &off);
                const int s = __ldcg(p.stage_s + i);
                const int sbase = off - i;
                for (int t0 = s; t0 < nr; t0 += 32) {  // warp-uniform trip count
                    const int t = t0 + lane;
                    const bool valid = t < nr;
                    const uint64_t k = valid ? tail_key(__ldcg(p.skey + sbase + t), i) : 0ull;
                    const bool match = valid && (sh + 8 == 64 || (k >> (sh + 8)) == prefix);
                    const int dig = (int)((k >> sh) & 255ull);
                    // warp-aggregated increment: one shared atomic per distinct digit
                    const unsigned same = __match_any_sync(0xffffffffu, match ? dig : -1);
                    if (match && (__ffs(same) - 1) == lane) atomicAdd(&hist[dig], __popc(same));
                }
            }
            __syncthreads();
            if (threadIdx.x < 32) {
                int loc[8];
                int lsum = 0;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    loc[q] = hist[255 - 8 * lane - q];
                    lsum += loc[q];
                }
                int incl = lsum;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    int y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += y;
                }
                const int excl = incl - lsum;
                const unsigned hit = __ballot_sync(0xffffffffu, excl < need && need <= incl);
                const int L = __ffs(hit) - 1;
                if (lane == L) {
                    int c = excl;
                    for (int q = 0; q < 8; ++q) {
                        if (c + loc[q] >= need) {
                            s_bcast[0] = 255 - 8 * lane - q;
                            s_bcast[1] = c;
                            s_bcast[2] = loc[q];
                            break;
                        }
                        c += loc[q];
                    }
                }
            }
            __syncthreads();
            const int b = s_bcast[0];
            need -= s_bcast[1];
            prefix = (prefix << 8) | (uint64_t)b;
            done = (s_bcast[2] == need);
            __syncthreads();
        }
    }
    // m_i and take_i; tree sizes into ord_s for the offsets scan.
    for (int i = warp_id(); i < n; i += kSelWarps) {
        int off;
        const int nr = n_nonroot(p, i, &off);
        const int s = __ldcg(p.stage_s + i);
        int m = 0;
        if (select_all) {
            m = nr - s;
        } else if (!select_none) {
            const int sbase = off - i;
            for (int t0 = s; t0 < nr; t0 += 32) {
                const int t = t0 + lane;
                bool in = false;
                if (t < nr) {
                    uint64_t k = tail_key(__ldcg(p.skey + sbase + t), i);
                    in = (k >> sh) >= prefix;
                }
                m += __popc(__ballot_sync(0xffffffffu, in));
            }
        }
        if (lane == 0) {
            p.take[i] = s + m;
            ord_s[i] = 1 + s + m;
        }
    }
    __syncthreads();
    const int used = block_exclusive_scan(ord_s, n, red);
    for (int i = threadIdx.x; i < n; i += kSelThreads) {
        p.tree_offsets[i] = ord_s[i];
    }
    if (threadIdx.x == 0) p.tree_offsets[n] = used;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) atomicAdd(&hdr->pad[0], 1u);  // release phase 3 in every CTA
    }  // last CTA
    // ---- phase 3 (every CTA, its own 32 requests): wait for the global phase ----
    if (threadIdx.x == 0) {
        while (*reinterpret_cast<volatile unsigned*>(&hdr->pad[0]) == s_gen0) __nanosleep(64);
        __threadfence();
    }
    __syncthreads();

    // (5) emit: warp per request.
    double* A_s2 = reinterpret_cast<double*>(smem_raw);
    int* remap_all = reinterpret_cast<int*>(A_s2 + n) + 2 * n;                                 // [32][kRemapWords]
    unsigned* bitmap_all = reinterpret_cast<unsigned*>(remap_all + kSelWarps * kRemapWords);  // [32][kBitmapWords]
    int* parent_all = reinterpret_cast<int*>(bitmap_all + kSelWarps * kBitmapWords);          // [32][kRemapWords]
    int* remap = remap_all + warp_id() * kRemapWords;
    unsigned* bits = bitmap_all + warp_id() * kBitmapWords;
    int* cpar = parent_all + warp_id() * kRemapWords;
    {
        const int i = blockIdx.x * kSelWarps + (int)warp_id();
        if (i < n) {
        int off;
        const int nr = n_nonroot(p, i, &off);
        const int take = __ldcg(p.take + i);
        const int tbase = __ldcg(p.tree_offsets + i);
        const int sbase = off - i;
        for (int w = lane; w < kBitmapWords; w += 32) bits[w] = 0u;
        for (int c = lane; c <= nr; c += 32) cpar[c] = p.cand_parent[off + c];  // staged: depth walks stay on chip
        __syncwarp();
        for (int t = lane; t < take; t += 32) {
            uint32_t idx = 0xFFFFFFFFu - (uint32_t)(__ldcg(p.skey + sbase + t) & 0xFFFFFFFFull);
            atomicOr(&bits[idx >> 5], 1u << (idx & 31));
        }
        __syncwarp();
        int running = 0;
        for (int c0 = 1; c0 <= nr; c0 += 32) {
            const int c = c0 + lane;
            const bool sel = c <= nr && ((bits[c >> 5] >> (c & 31)) & 1u);
            const unsigned mm = __ballot_sync(0xffffffffu, sel);
            if (sel) remap[c] = 1 + running + __popc(mm & ((1u << lane) - 1u));
            running += __popc(mm);
        }
        __syncwarp();
        if (lane == 0) {
            p.tree_src[tbase] = 0;
            p.tree_parent[tbase] = 0;
            if (p.tree_depth) p.tree_depth[tbase] = 0;
            if (p.tree_token) p.tree_token[tbase] = p.cand_token[off];
        }
        for (int c0 = 1; c0 <= nr; c0 += 32) {
            const int c = c0 + lane;
            const bool sel = c <= nr && ((bits[c >> 5] >> (c & 31)) & 1u);
            if (sel) {
                const int row = tbase + remap[c];
                const int par = cpar[c];
                const bool ok = par >= 0 && par < c;
                p.tree_src[row] = c;
                p.tree_parent[row] = (ok && par > 0) ? remap[par] : 0;
                if (p.tree_depth) {
                    int dep = 1, u = par, guard = 0;
                    while (u > 0 && guard < AS_MAX_CAND + 1) {
                        int pu = cpar[u];
                        u = (pu >= 0 && pu < u) ? pu : 0;
                        ++dep;
                        ++guard;
                    }
                    p.tree_depth[row] = dep;
                }
                if (p.tree_token) p.tree_token[row] = p.cand_token[off + c];
            }
        }
        __syncwarp();
        }
    }
}

size_t select_smem_bytes(int n) {
    return (size_t)n * sizeof(double) + 2 * (size_t)n * sizeof(int) +
           2 * (size_t)kSelWarps * kRemapWords * sizeof(int) + (size_t)kSelWarps * kBitmapWords * sizeof(unsigned);
}

size_t select_ws_bytes(int n_req, int n_cand_total) {
    size_t b = kWsHeaderBytes;
    b += align_up((size_t)n_req * 4, 256) * 4;        // desired, take, stage_s, toff
    b += align_up((size_t)(n_req + 1) * 4, 256);
    b += align_up((size_t)(n_cand_total > 0 ? n_cand_total : 1) * 8, 256);
    return b;
}

int launch_select(int n_req, int n_cand_total, const int32_t* cand_offsets, const int32_t* cand_parent,
                  const float* cand_prob, const int32_t* cand_token, const double* A, int depth_d,
                  int n_max, int budget, int32_t* tree_offsets, int32_t* tree_parent, int32_t* tree_src,
                  int32_t* tree_depth, int32_t* tree_token, int32_t* slo_count, void* ws,
                  cudaStream_t stream) {
    SelectParams p;
    p.n_req = n_req;
    p.cand_offsets = cand_offsets;
    p.cand_parent = cand_parent;
    p.cand_prob = cand_prob;
    p.cand_token = cand_token;
    p.A = A;
    p.depth_d = depth_d;
    p.n_max = n_max;
    p.budget = budget;
    p.tree_offsets = tree_offsets;
    p.tree_parent = tree_parent;
    p.tree_src = tree_src;
    p.tree_depth = tree_depth;
    p.tree_token = tree_token;
    p.slo_count = slo_count;
    p.ws = ws;
    unsigned char* b = reinterpret_cast<unsigned char*>(ws) + kWsHeaderBytes;
    const size_t nb = align_up((size_t)n_req * 4, 256);
    p.desired = reinterpret_cast<int32_t*>(b);
    p.take = reinterpret_cast<int32_t*>(b + nb);
    p.stage_s = reinterpret_cast<int32_t*>(b + 2 * nb);
    p.toff = reinterpret_cast<int32_t*>(b + 3 * nb);
    p.skey = reinterpret_cast<uint64_t*>(b + 4 * nb + align_up((size_t)(n_req + 1) * 4, 256));
    const size_t smem = select_smem_bytes(n_req);
    if (smem > 48 * 1024 &&
        cudaFuncSetAttribute(select_trees_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess)
        return -1;
    const int grid = (n_req + kSelWarps - 1) / kSelWarps;
    // cooperative launch: every CTA waits for the global phase run by the last
    // one to arrive, so all CTAs must be co-resident (grid <= 128 CTAs)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kSelThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, select_trees_kernel, p) != cudaSuccess) return -1;
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace as
