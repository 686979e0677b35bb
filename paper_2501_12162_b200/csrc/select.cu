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
//       by n_max and by C_i - 1; the fp64 sum equals the sequential loop's (R9);
//   (3) the single shared budget is consumed in (A desc, id asc) order (P:L821,
//       R5): s_i = clamp(B0 - sum_{j before i} desired_j, 0, desired_i);
//   (4) the throughput loop takes the global top-R of the
//       remaining tails under (f-hat desc, req asc, idx asc) (R8),
//       R = min(B0 - sum s, sum tails); m_i = how many land in request i;
//   (5) tree i = root + pi_i[0 : s_i + m_i], emitted in ascending candidate
//       index (topological; ancestor-closed by App. B).
//
// One launch of ONE thread-block cluster (CS <= 16 CTAs of 512 threads; CTA c
// owns a contiguous block of requests).  Everything stays on chip:
//   * each CTA stages its requests' offsets, f-hat and parents in shared memory
//     with coalesced loads; one warp per request sorts pi_i in registers
//     (bitonic, __shfl_xor_sync) and finds desired_i with a warp fp64 scan +
//     ballot when the sum is provably exact in any order (R9), else with the
//     lane-uniform sequential loop; the rank of the request in (A desc, id asc)
//     order is a warp-parallel count;
//   * exchange 1 (DSMEM): every CTA writes desired_i at position rank_i into
//     every peer's shared array; after one cluster barrier each CTA redundantly
//     scans it (s_i, sum s, R) -- no global round trip, no spin-waits;
//   * the global top-R is a radix select (8-bit digits, MSB first) whose
//     per-CTA shared histograms are summed through DSMEM, one cluster barrier
//     per digit (double-buffered), with an early exit once the bucket holding
//     the R-th key is taken whole;
//   * exchange 2 (DSMEM): per-CTA tree-size totals -> tree offsets; each CTA
//     emits its own trees (ballot-rank compaction, parent remap).
// Requests whose candidates do not fit the shared staging area (very large
// batches) read f-hat/parents from global memory and keep pi_i in the
// workspace instead (same code path, generic pointers).
#include <cooperative_groups.h>
#include <cstdlib>
#include <mutex>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace as {

#ifndef AS_SEL_THREADS
#define AS_SEL_THREADS 512
#endif
constexpr int kSelThreads = AS_SEL_THREADS;
constexpr int kSelWarps = kSelThreads / 32;
constexpr int kSelMaxReq = 4096;                // requests handled by one call
constexpr int kSelMaxCluster = 16;
constexpr int kRemapWords = AS_MAX_CAND + 1;    // local indices 0..AS_MAX_CAND
constexpr int kBitmapWords = (AS_MAX_CAND + 1 + 31) / 32;
constexpr int kSelSmemLimit = 200 * 1024;

struct SelectParams {
    int n_req, rpc;   // requests, requests per CTA
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
    uint64_t* skey_g;   // [N - n] workspace pi keys (used when a CTA's candidates do not fit smem)
    int cand_cap;       // candidates a CTA can stage in shared memory
    int topm;           // 1: per-request greedy caps (as_select_topm): request i keeps
                        //    min(n_max + (i < n_max_extra), C_i - 1) best candidates, no budget
    int n_max_extra;
    int dbg_stop;       // latency profiling only (AS_SEL_STOP): return after phase k (wrong outputs)
};

// Shared-memory layout (dynamic part), sized by the host from n, rpc and the
// per-CTA candidate capacity `cap` (36 bytes per staged candidate).
struct SelLayout {
    int o_A, o_des, o_exc, o_own, o_remap, o_bits, o_ukey, o_key, o_prob, o_par, o_rank, o_tok, o_dep, bytes;
    __host__ __device__ SelLayout(int n, int rpc, int cap) {
        int o = 0;
        o_A = o;     o += 8 * n;                                 // A(r) of every request
        o_des = o;   o += 4 * n;                                 // desired in A order (exchange 1)
        o_exc = o;   o += 4 * n;                                 // exclusive scan of o_des
        o_own = o;   o += 4 * 8 * (rpc + 1);                     // own: off, desired, arank, nr, s, take, size
        o = (o + 15) & ~15;
        o_remap = o; o += 2 * kSelWarps * kRemapWords;           // u16 remap per request group
        o = (o + 15) & ~15;
        o_bits = o;  o += 4 * kSelWarps * kBitmapWords;
        o = (o + 15) & ~15;
        o_ukey = o;  o += 8 * cap;                               // keys in candidate order
        o_key = o;   o += 8 * cap;                               // pi keys (sorted, non-root)
        o_prob = o;  o += 4 * cap;
        o_par = o;   o += 4 * cap;
        o_rank = o;  o += 4 * cap;
        o_tok = o;   o += 4 * cap;
        o_dep = o;   o += cap;
        o = (o + 15) & ~15;
        bytes = o;
    }
};
constexpr int kSelBytesPerCand = 37;

__device__ __forceinline__ void cl_arrive_relaxed() { asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory"); }
__device__ __forceinline__ void cl_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cl_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
__device__ __forceinline__ void cl_sync() { cl_arrive(); cl_wait(); }
__device__ __forceinline__ void red_add_cluster(int* local_addr, int rank, int v) {
    // fire-and-forget atomic add into CTA `rank`'s shared memory (DSMEM)
    uint32_t a = (uint32_t)__cvta_generic_to_shared(local_addr), ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
    asm volatile("red.relaxed.cluster.shared::cluster.add.u32 [%0], %1;" ::"r"(ra), "r"(v) : "memory");
}

// Warp-0 exclusive scan of data[0..n) (shared) into out[0..n) (may alias);
// returns the total to lane 0..31 of warp 0 (others: undefined).
__device__ __forceinline__ int warp_exclusive_scan(const int* data, int* out, int n) {
    const int lane = lane_id();
    const int chunk = (n + 31) >> 5;
    const int b = lane * chunk, e = min(n, b + chunk);
    int local = 0;
    for (int x = b; x < e; ++x) local += data[x];
    int incl = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    int run = incl - local;
    for (int x = b; x < e; ++x) {
        const int v = data[x];
        out[x] = run;
        run += v;
    }
    return __shfl_sync(0xffffffffu, incl, 31);
}

__device__ __forceinline__ uint64_t tail_key(uint64_t sk, int i) {
    // global order (f-hat desc, req asc, idx asc): low word = ~(i*512 + idx)
    const uint32_t idx = 0xFFFFFFFFu - (uint32_t)(sk & 0xFFFFFFFFull);
    return (sk & 0xFFFFFFFF00000000ull) | (uint64_t)(0xFFFFFFFFu - ((uint32_t)i * 512u + idx));
}

// ---------------------------------------------------------------------------
// Warp per request: sort pi_i, desired_i.
// prob/par: the request's candidates (local index c -> prob[c]), staged in
// shared memory or global; key_out: where pi_i's keys go (smem or workspace).
//
// pi_i is built by rank counting: the key of candidate j is (f-hat bits << 32
// | ~j) -- positive floats order as uint32, the complemented index breaks ties
// toward the lower index (R8) -- and its position in pi_i is the number of
// larger keys.  Keys are distinct, so the ranks are a permutation.  Every
// compare is independent (no shuffle chain), which is what a single warp per
// request needs for latency: the kernel is latency-bound, not ALU-bound.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t cand_key(float f, int j) {
    const uint32_t fb = (f > 0.f) ? __float_as_uint(f) : 0u;
    return ((uint64_t)fb << 32) | (uint64_t)(0xFFFFFFFFu - (uint32_t)j);
}

// desired_i (SLO stage length with unlimited budget) from request i's sorted
// keys ks[0..nr), one warp.  The result is the sequential fp64 loop's (R9):
//   * warp fp64 scans over 32-key chunks while every f-hat so far is >= 2^-24
//     and the sums stay < 64 -- all partial sums are then exact, so the scan's
//     values ARE the loop's (f-hat = m 2^(e-23), e >= -24: multiples of 2^-47);
//   * at the first f-hat < 2^-24 (pi is sorted, so every later one is smaller
//     too) the exact state n_acc after the prefix is known; the loop cannot
//     cross a_cap in the remaining rem entries when n_acc + rem (f + 2^-40) <
//     a_cap (each remaining add contributes at most f plus half an ulp <= 2^-48
//     of a sum < 64; the slack also covers the bound's own rounding), so
//     desired = lim without running it;
//   * otherwise the lane-uniform sequential loop resumes from that exact state
//     (identical to the oracle).
__device__ int slo_prefix_len(const SelectParams& p, double A_i, const uint64_t* ks, int nr) {
    const int lane = lane_id();
    const double a_cap = fmin(A_i, (double)p.depth_d + 1.0);
    const int lim = min(p.n_max, nr);
    if (!(1.0 < a_cap) || lim == 0) return 0;
    double run = 1.0;  // the loop's n_acc after t0 entries (exact)
    int t0 = 0;
    for (int c0 = 0; c0 < lim; c0 += 32) {
        const int s = c0 + lane;
        const float f = s < lim ? __uint_as_float((uint32_t)(ks[s] >> 32)) : 0.f;
        const unsigned tiny = __ballot_sync(0xffffffffu, s < lim && !(f >= 5.9604644775390625e-08f));
        const int nv = tiny ? __ffs(tiny) - 1 : 32;  // exact entries of this chunk
        double incl = (lane < nv) ? (double)f : 0.0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        incl += run;
        const double tot = __shfl_sync(0xffffffffu, incl, 31);
        if (!(tot < 64.0)) {  // partial sums may round: the sequential loop from the start
            run = 1.0;
            t0 = 0;
            break;
        }
        const unsigned hit = __ballot_sync(0xffffffffu, lane < nv && s < lim && incl >= a_cap);
        if (hit) return c0 + __ffs(hit);  // count includes the crossing element
        run = tot;
        t0 = min(lim, c0 + nv);
        if (tiny) {
            const int rem = lim - t0;
            const double fmax_rem = (double)__uint_as_float((uint32_t)(ks[t0] >> 32));
            if (run + (double)rem * (fmax_rem + 0x1p-40) < a_cap) return lim;  // cannot cross
            break;
        }
        if (t0 >= lim) return lim;
    }
    double nacc = run;  // the lane-uniform sequential loop from the exact state at t0
    int t = t0;
    while (t < lim && nacc < a_cap) {
        nacc += (double)__uint_as_float((uint32_t)(ks[t] >> 32));
        ++t;
    }
    return t;
}

template <int E>
__device__ __forceinline__ int sort_request(const SelectParams& p, int i, const float* prob, const int* par,
                                            int nr, uint64_t* key_out) {
    const int lane = lane_id();
    uint64_t key[E];
    int cnt[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int s = e * 32 + lane;
        key[e] = 0ull;  // padding: never counted (positions >= nr are not stored)
        cnt[e] = 0;
        if (s < nr) {
            const int j = s + 1;
            const float f = prob[j];
            const int pj = par[j];
            if (pj < 0 || pj >= j) {
                set_dev_error(p.ws, AS_DEV_BAD_PARENT, i);
            } else {
                const float fp = prob[pj];
                if (!(f > 0.f) || !(f <= fp)) set_dev_error(p.ws, AS_DEV_BAD_PROB, i);
            }
            key[e] = cand_key(f, j);
        }
    }
    // rank = #{k : key_k > key_j}, k over the request's non-root candidates
    int k = 1;
#pragma unroll 1
    for (; k + 3 <= nr; k += 4) {
        uint64_t kk[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) kk[u] = cand_key(prob[k + u], k + u);
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int e = 0; e < E; ++e) cnt[e] += kk[u] > key[e] ? 1 : 0;
    }
#pragma unroll 1
    for (; k <= nr; ++k) {
        const uint64_t kk = cand_key(prob[k], k);
#pragma unroll
        for (int e = 0; e < E; ++e) cnt[e] += kk > key[e] ? 1 : 0;
    }
#pragma unroll
    for (int e = 0; e < E; ++e)
        if (e * 32 + lane < nr) key_out[cnt[e]] = key[e];
    __syncwarp();
    if (p.topm) return min(p.n_max + (i < p.n_max_extra ? 1 : 0), nr);  // per-request greedy cap
    return slo_prefix_len(p, p.A[i], key_out, nr);
}

// Exclusive scan of data[0..n) (shared) into out[0..n); returns the total.
__device__ int block_exclusive_scan(const int* data, int* out, int n, int* red) {
    const int tid = threadIdx.x;
    const int chunk = (n + kSelThreads - 1) / kSelThreads;
    const int b = tid * chunk;
    const int e = min(n, b + chunk);
    int local = 0;
    for (int x = b; x < e; ++x) local += data[x];
    int incl = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if ((int)lane_id() >= o) incl += y;
    }
    __syncthreads();
    if (lane_id() == 31) red[warp_id()] = incl;
    __syncthreads();
    if (threadIdx.x < 32) {
        const int w = threadIdx.x < (unsigned)kSelWarps ? red[threadIdx.x] : 0;
        int wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, wi, o);
            if ((int)threadIdx.x >= o) wi += y;
        }
        red[threadIdx.x] = wi - w;
        if (threadIdx.x == 31) red[32] = wi;
    }
    __syncthreads();
    int run = red[warp_id()] + incl - local;
    for (int x = b; x < e; ++x) {
        const int v = data[x];
        out[x] = run;
        run += v;
    }
    const int total = red[32];
    __syncthreads();
    return total;
}

__device__ int block_sum(int v, int* red) {
    v = warp_sum(v);
    __syncthreads();
    if (lane_id() == 0) red[warp_id()] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        int t = threadIdx.x < (unsigned)kSelWarps ? red[threadIdx.x] : 0;
        t = warp_sum(t);
        if (threadIdx.x == 0) red[32] = t;
    }
    __syncthreads();
    const int r = red[32];
    __syncthreads();
    return r;
}

// ---------------------------------------------------------------------------
// The kernel (one cluster).  Own requests are processed by groups of W warps
// (W = warps / requests-per-CTA, at least 1); every phase ends at a CTA
// barrier, and all groups run the same number of rounds, so the barriers are
// uniform.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kSelThreads, 1) select_trees_kernel(SelectParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int hist[256];
    __shared__ int hsum[2][256];
    __shared__ int part_nr[kSelMaxCluster];
    __shared__ int part_tot[kSelMaxCluster];
    __shared__ int s_bcast[8];
    cg::cluster_group cluster = cg::this_cluster();
    const int CS = (int)cluster.num_blocks();
    const int c = (int)cluster.block_rank();
    const int n = p.n_req;
    const int lane = lane_id();
    const int warp = warp_id();
    const int tid = threadIdx.x;
    // zero what peers accumulate into before anyone can reach exchange 1
    for (int x = tid; x < 512; x += kSelThreads) (&hsum[0][0])[x] = 0;
    for (int x = tid; x < 256; x += kSelThreads) hist[x] = 0;
    cl_arrive_relaxed();  // "started": waited on before the first remote access
    pdl_launch_dependents();  // let the attention kernel run its prologue meanwhile
    pdl_wait();               // the previous step's accept may still read our outputs

    const SelLayout Lo(n, p.rpc, p.cand_cap);
    double* A_s = reinterpret_cast<double*>(smem + Lo.o_A);
    int* des_all = reinterpret_cast<int*>(smem + Lo.o_des);
    int* exc_all = reinterpret_cast<int*>(smem + Lo.o_exc);
    int* own = reinterpret_cast<int*>(smem + Lo.o_own);
    const int rpc = p.rpc;
    int* off_s = own;                      // [rpc+1] cand offsets of own requests
    int* desired_s = off_s + (rpc + 1);    // [rpc] desired, later the tree size
    int* arank_s = desired_s + (rpc + 1);  // [rpc] position in (A desc, id asc) order
    int* nr_s = arank_s + (rpc + 1);
    int* s_s = nr_s + (rpc + 1);
    int* take_s = s_s + (rpc + 1);
    int* size_s = take_s + (rpc + 1);      // scanned tree offsets (CTA-local)
    uint64_t* ukey_s = reinterpret_cast<uint64_t*>(smem + Lo.o_ukey);
    uint64_t* key_s = reinterpret_cast<uint64_t*>(smem + Lo.o_key);
    float* prob_s = reinterpret_cast<float*>(smem + Lo.o_prob);
    int* par_s = reinterpret_cast<int*>(smem + Lo.o_par);
    int* rank_s = reinterpret_cast<int*>(smem + Lo.o_rank);
    int* tok_s = reinterpret_cast<int*>(smem + Lo.o_tok);
    uint8_t* dep_s = reinterpret_cast<uint8_t*>(smem + Lo.o_dep);

    const int r0 = min(n, c * rpc);
    const int r1 = min(n, r0 + rpc);
    const int nown = r1 - r0;
    // request groups: W warps per request, G groups
    const int W = max(1, kSelWarps / max(1, nown));
    const int G = kSelWarps / W;
    const int grp = warp / W, wg = warp - grp * W;
    const int rounds = (nown + G - 1) / G;

    if (p.dbg_stop == 0) return;
    // ---- stage: own offsets, every A(r); then f-hat, parents (and tokens) ----
    for (int k = tid; k <= nown; k += kSelThreads) off_s[k] = p.cand_offsets[r0 + k];
    if (!p.topm)
        for (int k = tid; k < n; k += kSelThreads) A_s[k] = p.A[k];
    __syncthreads();
    const int cbase = off_s[0];
    const int ncand = off_s[nown] - cbase;
    const bool staged = ncand <= p.cand_cap;
    const bool want_tok = p.tree_token != nullptr;
    if (staged) {
        for (int k = tid; k < ncand; k += kSelThreads) {
            prob_s[k] = p.cand_prob[cbase + k];
            par_s[k] = p.cand_parent[cbase + k];
            if (want_tok) tok_s[k] = p.cand_token[cbase + k];
        }
    }
    __syncthreads();
    // candidate arrays indexed by GLOBAL candidate id (staged: shifted smem)
    const float* probc = staged ? prob_s - cbase : p.cand_prob;
    const int* parc = staged ? par_s - cbase : p.cand_parent;
    // pi keys: own request k's sorted keys start at keyc + (off - i)
    uint64_t* keyc = staged ? key_s - (cbase - r0) : p.skey_g;

    if (p.dbg_stop == 1) return;
    // ---- phase 1: pi_i, desired_i, rank of A_i ----
    for (int k = tid; k < nown; k += kSelThreads) {
        const int C = off_s[k + 1] - off_s[k];
        if (C < 1 || C - 1 > AS_MAX_CAND) set_dev_error(p.ws, C < 1 ? AS_DEV_BAD_PARENT : AS_DEV_TOO_MANY_CAND, r0 + k);
        nr_s[k] = max(0, min(C - 1, AS_MAX_CAND));
    }
    __syncthreads();
    if (staged) {
        for (int rd = 0; rd < rounds; ++rd) {
            const int k = rd * G + grp;
            const bool active = grp < G && k < nown;
            const int i = r0 + k;
            const int off = active ? off_s[k] : 0;
            const int nr = active ? nr_s[k] : 0;
            const int lo = off - cbase;  // request's first staged candidate (its root)
            // (1a) keys in candidate order, validation, depth; ranks zeroed
            for (int s = wg * 32 + lane; s < nr; s += W * 32) {
                const int j = s + 1;
                const float f = prob_s[lo + j];
                const int pj = par_s[lo + j];
                int dep = 1;
                if (pj < 0 || pj >= j) {
                    set_dev_error(p.ws, AS_DEV_BAD_PARENT, i);
                } else {
                    if (!(f > 0.f) || !(f <= prob_s[lo + pj])) set_dev_error(p.ws, AS_DEV_BAD_PROB, i);
                    for (int u = pj, guard = 0; u > 0 && guard <= AS_MAX_CAND; ++guard) {  // depth walk
                        const int pu = par_s[lo + u];
                        u = (pu >= 0 && pu < u) ? pu : 0;
                        ++dep;
                    }
                }
                dep_s[lo + j] = (uint8_t)min(dep, 255);
                ukey_s[lo - k + s] = cand_key(f, j);
                rank_s[lo - k + s] = 0;
            }
            __syncthreads();
            if (p.dbg_stop == 11) return;
            // (1b) rank counting: warp wg compares every element with its slice of keys
            if (active) {
                const int per = (nr + W - 1) / W;
                const int kb = wg * per, ke = min(nr, kb + per);
                const uint64_t* uk = ukey_s + (lo - k);
                for (int s = lane; s < nr; s += 32) {
                    const uint64_t key = uk[s];
                    int cnt = 0;
                    int t = kb;
#pragma unroll 1
                    for (; t + 3 < ke; t += 4)
                        cnt += (uk[t] > key) + (uk[t + 1] > key) + (uk[t + 2] > key) + (uk[t + 3] > key);
                    for (; t < ke; ++t) cnt += uk[t] > key;
                    if (cnt) atomicAdd(&rank_s[lo - k + s], cnt);
                }
            }
            __syncthreads();
            if (p.dbg_stop == 12) return;
            // (1c) scatter into pi order
            for (int s = wg * 32 + lane; s < nr; s += W * 32) keyc[off - i + rank_s[lo - k + s]] = ukey_s[lo - k + s];
            __syncthreads();
            if (p.dbg_stop == 13) return;
            // (1d) desired_i (warp 0 of the group) and the A-order rank (warp 1, or 0)
            if (active && wg == 0) {
                const int des = p.topm ? min(p.n_max + (i < p.n_max_extra ? 1 : 0), nr)
                                       : slo_prefix_len(p, A_s[i], keyc + (off - i), nr);
                if (lane == 0) desired_s[k] = des;
            }
            if (active && p.topm) {
                if (wg == 0 && lane == 0) arank_s[k] = i;  // no A ordering: the caps never compete
            } else if (active && wg == (W > 1 ? 1 : 0)) {
                const double a = A_s[i];
                int rk = 0;
                for (int j = lane; j < n; j += 32) {
                    const double b = A_s[j];
                    rk += (b > a) || (b == a && j < i);
                }
                rk = warp_sum(rk);
                if (lane == 0) arank_s[k] = rk;
            }
        }
    } else {
        // large batches: one warp per request, candidates read from global memory
        for (int k = warp; k < nown; k += kSelWarps) {
            const int i = r0 + k;
            const int off = off_s[k];
            const int nr = nr_s[k];
            uint64_t* ko = keyc + (off - i);
            int des;
            if (nr <= 32) des = sort_request<1>(p, i, probc + off, parc + off, nr, ko);
            else if (nr <= 64) des = sort_request<2>(p, i, probc + off, parc + off, nr, ko);
            else if (nr <= 128) des = sort_request<4>(p, i, probc + off, parc + off, nr, ko);
            else des = sort_request<8>(p, i, probc + off, parc + off, nr, ko);
            int rk = i;
            if (!p.topm) {
                const double a = A_s[i];
                rk = 0;
                for (int j = lane; j < n; j += 32) {
                    const double b = A_s[j];
                    rk += (b > a) || (b == a && j < i);
                }
                rk = warp_sum(rk);
            }
            if (lane == 0) {
                desired_s[k] = des;
                arank_s[k] = rk;
            }
        }
    }
    __syncthreads();

    // ---- exchange 1: desired at rank position, per-CTA sum of nr, into every CTA ----
    if (p.dbg_stop == 2) return;
    cl_wait();  // every CTA of the cluster has started
    for (int x = tid; x < nown * CS; x += kSelThreads) {
        const int k = x / CS, dst = x - k * CS;
        cluster.map_shared_rank(des_all, dst)[arank_s[k]] = desired_s[k];
    }
    if (warp == kSelWarps - 1) {
        int v = 0;
        for (int k = lane; k < nown; k += 32) v += nr_s[k];
        v = warp_sum(v);
        if (lane < CS) cluster.map_shared_rank(part_nr, lane)[c] = v;
    }
    cl_sync();

    if (p.dbg_stop == 3) return;
    // ---- (3) budget sequencing, redundant in every CTA (warp 0) ----
    const int B0 = p.topm ? 0x3fffffff : p.budget - n;  // topm: the caps alone bound the trees
    if (warp == 0) {
        warp_exclusive_scan(des_all, exc_all, n);
        __syncwarp();
        int my_s = 0;
        for (int x = lane; x < n; x += 32) my_s += max(0, min(B0 - exc_all[x], des_all[x]));
        my_s = warp_sum(my_s);
        int sum_nr = 0;
        for (int q = 0; q < CS; ++q) sum_nr += part_nr[q];
        if (lane == 0) {
            s_bcast[4] = my_s;
            s_bcast[5] = sum_nr;
        }
    }
    __syncthreads();
    const int sum_s = s_bcast[4];
    const int sum_tail = s_bcast[5] - sum_s;
    const int R = p.topm ? 0 : min(B0 - sum_s, sum_tail);  // topm: no throughput stage
    for (int k = tid; k < nown; k += kSelThreads) {
        const int sv = max(0, min(B0 - exc_all[arank_s[k]], desired_s[k]));
        s_s[k] = sv;
        if (p.slo_count) p.slo_count[r0 + k] = sv;
    }
    __syncthreads();

    if (p.dbg_stop == 4) return;
    // ---- (4) global top-R of the tails: cluster radix select ----
    // Per digit: warp-aggregated shared histogram of this CTA's matching tails,
    // pushed into every CTA's hsum with DSMEM reductions, one cluster barrier,
    // then every CTA picks the same digit.  hsum is double-buffered by pass.
    int sh = 64;
    uint64_t prefix = 0;
    const bool select_all = (R >= sum_tail) && R > 0;
    const bool select_none = (R <= 0);
    if (!select_all && !select_none) {
        int need = R;
        bool done = false;
        int pass = 0;
        while (!done && sh > 0) {
            sh -= 8;
            for (int k = warp; k < nown; k += kSelWarps) {
                const int i = r0 + k;
                const int nr = nr_s[k], sk = s_s[k];
                const uint64_t* ks = keyc + (off_s[k] - i);
                for (int t0 = sk; t0 < nr; t0 += 32) {  // warp-uniform trip count
                    const int t = t0 + lane;
                    const bool valid = t < nr;
                    const uint64_t key = valid ? tail_key(ks[t], i) : 0ull;
                    const bool match = valid && (sh + 8 == 64 || (key >> (sh + 8)) == prefix);
                    const int dig = (int)((key >> sh) & 255ull);
                    const unsigned same = __match_any_sync(0xffffffffu, match ? dig : -1);
                    if (match && (__ffs(same) - 1) == lane) atomicAdd(&hist[dig], __popc(same));
                }
            }
            __syncthreads();
            int* hs = hsum[pass & 1];
            for (int x = tid; x < 256 * CS; x += kSelThreads) {
                const int bin = x & 255, q = x >> 8;
                const int v = hist[bin];
                if (v) red_add_cluster(&hs[bin], q, v);
            }
            __syncthreads();
            for (int x = tid; x < 256; x += kSelThreads) hist[x] = 0;
            if (p.dbg_stop == 40 + 2 * pass) return;
            cl_sync();  // every CTA's contribution to hs has landed
            if (p.dbg_stop == 41 + 2 * pass) return;
            if (warp == 0) {
                int loc[8];
                int lsum = 0;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    loc[q] = hs[255 - 8 * lane - q];
                    hs[255 - 8 * lane - q] = 0;  // reused two passes later
                    lsum += loc[q];
                }
                int incl = lsum;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += y;
                }
                const int excl = incl - lsum;
                const unsigned hit = __ballot_sync(0xffffffffu, excl < need && need <= incl);
                const int Lh = __ffs(hit) - 1;
                if (lane == Lh) {
                    int cc = excl;
                    for (int q = 0; q < 8; ++q) {
                        if (cc + loc[q] >= need) {
                            s_bcast[0] = 255 - 8 * lane - q;
                            s_bcast[1] = cc;
                            s_bcast[2] = loc[q];
                            break;
                        }
                        cc += loc[q];
                    }
                }
            }
            __syncthreads();
            const int b = s_bcast[0];
            need -= s_bcast[1];
            prefix = (prefix << 8) | (uint64_t)b;
            done = (s_bcast[2] == need);
            __syncthreads();
            ++pass;
        }
    }
    // m_i, take_i, tree size of own requests
    for (int k = warp; k < nown; k += kSelWarps) {
        const int i = r0 + k;
        const int nr = nr_s[k], sk = s_s[k];
        int m = 0;
        if (select_all) {
            m = nr - sk;
        } else if (!select_none) {
            const uint64_t* ks = keyc + (off_s[k] - i);
            for (int t0 = sk; t0 < nr; t0 += 32) {
                const int t = t0 + lane;
                const bool in = t < nr && (tail_key(ks[t], i) >> sh) >= prefix;
                m += __popc(__ballot_sync(0xffffffffu, in));
            }
        }
        if (lane == 0) {
            take_s[k] = sk + m;
            desired_s[k] = 1 + sk + m;  // tree size (desired no longer needed)
        }
    }
    __syncthreads();
    if (warp == 0) {
        const int tot = warp_exclusive_scan(desired_s, size_s, nown);
        // ---- exchange 2: per-CTA totals -> tree offsets ----
        if (lane < CS) cluster.map_shared_rank(part_tot, lane)[c] = tot;
    }
    if (p.dbg_stop == 5) return;
    cl_sync();
    int base = 0, used = 0;
    for (int q = 0; q < CS; ++q) {
        base += (q < c) ? part_tot[q] : 0;
        used += part_tot[q];
    }
    for (int k = tid; k < nown; k += kSelThreads) p.tree_offsets[r0 + k] = base + size_s[k];
    if (c == CS - 1 && tid == 0) p.tree_offsets[n] = used;

    if (p.dbg_stop == 6) return;
    // ---- (5) emit own trees: group of W warps per request ----
    uint16_t* remap = reinterpret_cast<uint16_t*>(smem + Lo.o_remap) + grp * kRemapWords;
    unsigned* bits = reinterpret_cast<unsigned*>(smem + Lo.o_bits) + grp * kBitmapWords;
    const int* tokc = staged ? tok_s - cbase : p.cand_token;
    for (int rd = 0; rd < rounds; ++rd) {
        const int k = rd * G + grp;
        const bool active = grp < G && k < nown;
        const int i = r0 + k;
        const int off = active ? off_s[k] : 0;
        const int nr = active ? nr_s[k] : 0;
        const int take = active ? take_s[k] : 0;
        const int tbase = active ? base + size_s[k] : 0;
        const uint64_t* ks = keyc + (off - i);
        const int nwords = (nr + 1 + 31) >> 5;  // local indices 0..nr
        if (active)
            for (int w = wg * 32 + lane; w < nwords; w += W * 32) bits[w] = 0u;
        __syncthreads();
        for (int t = wg * 32 + lane; t < take; t += W * 32) {
            const uint32_t idx = 0xFFFFFFFFu - (uint32_t)(ks[t] & 0xFFFFFFFFull);
            atomicOr(&bits[idx >> 5], 1u << (idx & 31));
        }
        __syncthreads();
        // compact index of candidate cc = 1 + #selected candidates before it
        for (int w = wg; w < nwords; w += W) {
            const int cc = w * 32 + lane;
            const unsigned word = bits[w];
            int before = 0;
            for (int x = 0; x < w; ++x) before += __popc(bits[x]);
            if ((word >> lane) & 1u) remap[cc] = (uint16_t)(1 + before + __popc(word & ((1u << lane) - 1u)));
        }
        __syncthreads();
        if (active && wg == 0 && lane == 0) {
            p.tree_src[tbase] = 0;
            p.tree_parent[tbase] = 0;
            if (p.tree_depth) p.tree_depth[tbase] = 0;
            if (want_tok) p.tree_token[tbase] = tokc[off];
        }
        for (int cc = 1 + wg * 32 + lane; cc <= nr; cc += W * 32) {
            if (!((bits[cc >> 5] >> (cc & 31)) & 1u)) continue;
            const int row = tbase + remap[cc];
            const int par = parc[off + cc];
            const bool ok = par >= 0 && par < cc;
            p.tree_src[row] = cc;
            p.tree_parent[row] = (ok && par > 0) ? remap[par] : 0;
            if (p.tree_depth) {
                int dep;
                if (staged) {
                    dep = dep_s[off - cbase + cc];
                } else {
                    dep = 1;
                    for (int u = par, guard = 0; u > 0 && guard <= AS_MAX_CAND; ++guard) {
                        const int pu = parc[off + u];
                        u = (pu >= 0 && pu < u) ? pu : 0;
                        ++dep;
                    }
                }
                p.tree_depth[row] = dep;
            }
            if (want_tok) p.tree_token[row] = tokc[off + cc];
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// Host side.
// ---------------------------------------------------------------------------
int pdl_enabled() {
#ifdef AS_DEBUG
    static const int v = [] {
        const char* e = getenv("AS_PDL");  // A/B switch (debug build): 0 = plain stream ordering
        return (e && e[0] == '0') ? 0 : 1;
    }();
    return v;
#else
    return 1;
#endif
}

static int cluster_size_for(int n) {
    int cs = n;  // as many CTAs as possible: more warps per request (latency-bound)
    if (cs < 1) cs = 1;
    int cap = kSelMaxCluster;
#ifdef AS_DEBUG
    static const int dbg_cap = [] {  // A/B: cluster size cap (debug build)
        const char* e = getenv("AS_SEL_CS");
        return e ? atoi(e) : 0;
    }();
    if (dbg_cap > 0) cap = dbg_cap;
#endif
    if (cs > cap) cs = cap;
    return cs;
}

static int cand_cap_for(int n, int rpc, int n_cand_total) {
    const SelLayout base(n, rpc, 0);
    const int avail = kSelSmemLimit - base.bytes;
    int cap = avail > 0 ? avail / kSelBytesPerCand : 0;
    int want = rpc * (AS_MAX_CAND + 1);
    if (n_cand_total < want) want = n_cand_total;  // no CTA holds more than all candidates
    return cap < want ? cap : want;
}

// Largest cluster size <= want that the device can co-schedule with this smem.
static int fit_cluster(int want, size_t smem) {
    while (want > 1) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(want);
        cfg.blockDim = dim3(kSelThreads);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = want;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int nc = 0;
        if (cudaOccupancyMaxActiveClusters(&nc, select_trees_kernel, &cfg) == cudaSuccess && nc >= 1) return want;
        cudaGetLastError();
        want = want > 8 ? 8 : want / 2;
    }
    return 1;
}

size_t select_ws_bytes(int n_req, int n_cand_total) {
    size_t b = kWsHeaderBytes;
    b += align_up((size_t)(n_cand_total > 0 ? n_cand_total : 1) * 8, 256);
    return b;
}

int launch_select(int n_req, int n_cand_total, const int32_t* cand_offsets, const int32_t* cand_parent,
                  const float* cand_prob, const int32_t* cand_token, const double* A, int depth_d,
                  int n_max, int budget, int32_t* tree_offsets, int32_t* tree_parent, int32_t* tree_src,
                  int32_t* tree_depth, int32_t* tree_token, int32_t* slo_count, void* ws,
                  cudaStream_t stream, int topm, int n_max_extra) {
    if (n_req > kSelMaxReq) return -1;
    SelectParams p;
    p.topm = topm;
    p.n_max_extra = n_max_extra;
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
    p.skey_g = reinterpret_cast<uint64_t*>(reinterpret_cast<unsigned char*>(ws) + kWsHeaderBytes);
    // kernel attributes are per device: set once per device, under a mutex (re-entrant ABI)
    {
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return -1;
        static std::mutex mu;
        static bool attrs_set[64] = {false};
        std::lock_guard<std::mutex> lk(mu);
        if (!attrs_set[dev]) {
            if (cudaFuncSetAttribute(select_trees_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     kSelSmemLimit + 16 * 1024) != cudaSuccess ||
                cudaFuncSetAttribute(select_trees_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) !=
                    cudaSuccess)
                return -1;
            attrs_set[dev] = true;
        }
    }
    int cs = cluster_size_for(n_req);
    for (;;) {
        p.rpc = (n_req + cs - 1) / cs;
        p.cand_cap = cand_cap_for(n_req, p.rpc, n_cand_total);
        const int fit = fit_cluster(cs, SelLayout(n_req, p.rpc, p.cand_cap).bytes);
        if (fit == cs) break;
        cs = fit;
    }
    const size_t smem = SelLayout(n_req, p.rpc, p.cand_cap).bytes;
#ifdef AS_DEBUG
    static const int dbg_stop = [] {  // phase-latency experiments only (early exit, wrong outputs)
        const char* e = getenv("AS_SEL_STOP");
        return e ? atoi(e) : 99;
    }();
#else
    constexpr int dbg_stop = 99;
#endif
    p.dbg_stop = dbg_stop;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(kSelThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1 + fill_launch_attrs(attr + 1);
    if (cudaLaunchKernelEx(&cfg, select_trees_kernel, p) != cudaSuccess) return -1;
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace as
