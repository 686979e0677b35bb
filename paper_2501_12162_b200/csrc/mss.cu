// mss.cu -- NEXT-3(b): as_mss_verify, SpecInfer multi-step speculative sampling
// (reading R25) -- the stochastic acceptance rule of "tree-based
// verification ... prior work" (Step 4) when the tree's children were
// drawn from the draft distribution.
//
// At tree node u with children c_1 < ... < c_k (draft tokens x_j, uniforms r_j),
// target row p = p_u and draft row q = q_u (fp32 inputs, fp64 arithmetic):
//   p~ = p, N = sum p~
//   for j: accept c_j iff p~(x_j) > 0 and (r_j * N) * q(x_j) <= p~(x_j);
//          else p~(v) <- max(0, p~(v) - N q(v)) (v != x_j), p~(x_j) <- 0,
//               N <- sum p~ (N == 0: keep the previous p~, stop trying)
//   no child accepted: bonus = first v with cum(v) >= r_b N and p~(v) > 0
//                      (else the last v with p~(v) > 0).
// Every residual element is the same sequence of fp64 operations the oracle
// performs (one __dmul_rn, one __dsub_rn, one max per rejection; no FMA), so
// element values are bit-identical to oracle/mss.py's; only the sums'
// association differs (last bits -- the oracle reports each decision's margin).
//
// One thread-block cluster of C CTAs (C = 8, or 16 for vocabularies past 147k)
// per task.  CTA c owns the slice [c S, (c+1) S) of the vocabulary (S = E * 512,
// E a multiple of 4 with E/4 odd so per-thread float4 chunks are bank-conflict
// free): the node's p slice lands in shared memory by bulk copy (TMA engine)
// once per node; a node with children widens p into an fp64 residual R in
// shared memory while summing it, then bulk-copies its q slice over p (from
// L2: prefetched when the node starts), so every rejection updates R in place
// from shared memory (O(1) work per entry per rejection); the children's
// q(x_j) are loaded when the node starts, and the CTA owning the next child's
// token pushes p~(x) to its peers with each mass exchange, so a decision is
// local arithmetic.  The cluster combines per-CTA fp64 partials
// through DSMEM (each CTA pushes its partial into every peer, one cluster
// barrier, all CTAs sum them in rank order -> identical N everywhere).
// Measured (c2): ~2 us per node to load + sum, ~4.3 us per
// rejection (an fp64 pass over the slice + one cluster barrier).
//   walk = 1: task = request; the cluster walks from the root, visiting only the
//             nodes on the accepted path (HBM traffic = path rows, not tree rows),
//             and writes the accept record {len, bonus, path} (the layout of
//             as_accept_tokens' *_RECORDS phases: AS_ACCEPT_COMMIT_RECORDS then
//             commits the path's K/V).
//   walk = 0: task = node; every node's emitted token (all-nodes mode).
// Persistent grid: as many clusters as fit (one 225 KB CTA per SM), tasks strided.
#include <cooperative_groups.h>
#include <mutex>
#include <map>

#include "params.cuh"
#include "tc_ptx.cuh"

namespace cg = cooperative_groups;

namespace as {

constexpr int kMssThreads = 512;
constexpr int kMssWarps = kMssThreads / 32;
constexpr int kMssMaxKids = AS_MAX_TREE;
constexpr int kMssMaxC = 16;

struct MssParams {
    int req_begin, req_end, n_tree_rows, vocab;
    const int32_t* tree_offsets;
    const int32_t* tree_parent;
    const int32_t* tree_tokens;
    const float* p;
    const float* q;
    const float* uni;
    const float* bonus_uni;
    int32_t* emitted;  // [n_tree_rows] or NULL
    int32_t* records;  // walk: [n_req][2 + max_path] or NULL
    int max_path;
    int walk;
    int E;      // floats per thread chunk
    int S;      // floats per CTA slice (E * kMssThreads)
    int vec4;   // rows 16-byte aligned (vocab % 4 == 0 and aligned bases)
    void* ws;
    unsigned long long* trace;  // debug build: cluster-0 per-node timeline [64][8] (globaltimer ns) or NULL
};

#ifdef AS_DEBUG
#define MSS_TRACE(k, e, v)                                                                                   \
    do {                                                                                                     \
        if (p.trace && blockIdx.x == 0 && t == 0 && (k) < 64 && (k) >= 0) p.trace[(k) * 8 + (e)] = (v);                  \
    } while (0)
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long x;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(x));
    return x;
}
#else
#define MSS_TRACE(k, e, v) \
    do {                   \
    } while (0)
__device__ __forceinline__ unsigned long long gtime() { return 0; }
#endif

struct MssShared {
    // (p slice P [S] f32 and residual R [S] f64 follow this struct in shared memory)
    double hN[kMssMaxKids];      // history: mass N_k before rejection k
    int hx[kMssMaxKids];         // history: rejected token x_k
    int kid[kMssMaxKids];        // children of the current node (local index)
    double part[2][kMssMaxC];    // cluster exchange of CTA partial sums (double-buffered)
    double nrx[2];               // p~(x) of the next child to try, pushed by the owning CTA
    float kid_q[kMssMaxKids];    // q(x_j) of the children's tokens (loaded when the node starts)
    int ipart[2][kMssMaxC][2];   // cluster exchange of (first crossing, last with mass)
    double wsum[kMssWarps];
    double wscan[kMssWarps];
    int wmin[kMssWarps], wmax[kMssWarps];
    int t_par[AS_MAX_TREE];      // the task's request: parents, draft tokens, uniforms
    int t_tok[AS_MAX_TREE];
    float t_uni[AS_MAX_TREE];
    int n_kids, node, K, o, flag;
    int path[AS_MAX_TREE];
    int plen, acc;
    uint64_t bar;                // row loads (bulk copies, complete_tx)
};

__device__ __forceinline__ double f2d(float f) { return (double)f; }

// p~ at entry i of this CTA's slice: mat == 0 -> p (P holds p), else R[i].
__device__ __forceinline__ double res_at(const float* P, const double* R, int mat, int i) {
    return mat ? R[i] : f2d(P[i]);
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Cluster mass from the per-thread chunk sums tau: warp xor trees, warp 0
// reduces the 16 warp sums and pushes the CTA total into every peer, one
// cluster barrier, every thread sums the C totals in rank order.  The CTA
// owning entry `x_off` (x_owner >= 0: the next child's token) also pushes
// p~ there, so the next decision reads it locally (*nrx).
__device__ double cluster_mass(cg::cluster_group& cl, MssShared& sh, double tau, int& xbuf, int C, int rank,
                               int x_owner, int x_off, const float* P, const double* R, int mat, double* nrx) {
    const int t = threadIdx.x;
    const double ws = warp_sum_d(tau);
    if ((t & 31) == 0) sh.wsum[t >> 5] = ws;
    __syncthreads();
    const int b = xbuf;
    xbuf ^= 1;
    if (t < 32) {
        const double cta = warp_sum_d(t < kMssWarps ? sh.wsum[t] : 0.0);
        if (t < C) {
            cl.map_shared_rank(&sh.part[b][0], t)[rank] = cta;
            if (x_owner == rank) cl.map_shared_rank(&sh.nrx[0], t)[b] = res_at(P, R, mat, x_off);
        }
    }
    cl.sync();
    if (nrx) *nrx = sh.nrx[b];
    double s = 0.0;
    for (int c = 0; c < C; ++c) s = __dadd_rn(s, sh.part[b][c]);
    return s;
}

// Chunk sums use four independent chains (element j of each float4 -> chain j),
// combined (c0 + c1) + (c2 + c3): a fixed order, short dependency chains.
__device__ __forceinline__ double comb4(const double c[4]) {
    return __dadd_rn(__dadd_rn(c[0], c[1]), __dadd_rn(c[2], c[3]));
}

// Sum of this thread's chunk of p, widened into R on the way (R = p in fp64).
__device__ __forceinline__ double widen_sum(const float* P, double* R, int E) {
    const int t = threadIdx.x;
    double c[4] = {0.0, 0.0, 0.0, 0.0};
    const float4* P4 = reinterpret_cast<const float4*>(P + t * E);
    double2* R2 = reinterpret_cast<double2*>(R + t * E);
    for (int k = 0; k < E / 4; ++k) {
        const float4 a = P4[k];
        const double d0 = f2d(a.x), d1 = f2d(a.y), d2 = f2d(a.z), d3 = f2d(a.w);
        R2[2 * k] = make_double2(d0, d1);
        R2[2 * k + 1] = make_double2(d2, d3);
        c[0] = __dadd_rn(c[0], d0);
        c[1] = __dadd_rn(c[1], d1);
        c[2] = __dadd_rn(c[2], d2);
        c[3] = __dadd_rn(c[3], d3);
    }
    return comb4(c);
}

// sum of this thread's chunk of p (mat == 0) or R
__device__ __forceinline__ double chunk_sum(const float* P, const double* R, int mat, int E) {
    const int t = threadIdx.x;
    double c[4] = {0.0, 0.0, 0.0, 0.0};
    if (!mat) {
        const float4* P4 = reinterpret_cast<const float4*>(P + t * E);
        for (int k = 0; k < E / 4; ++k) {
            const float4 a = P4[k];
            c[0] = __dadd_rn(c[0], f2d(a.x));
            c[1] = __dadd_rn(c[1], f2d(a.y));
            c[2] = __dadd_rn(c[2], f2d(a.z));
            c[3] = __dadd_rn(c[3], f2d(a.w));
        }
    } else {
        const double2* R2 = reinterpret_cast<const double2*>(R + t * E);
        for (int k = 0; k < E / 4; ++k) {
            const double2 a = R2[2 * k], b = R2[2 * k + 1];
            c[0] = __dadd_rn(c[0], a.x);
            c[1] = __dadd_rn(c[1], a.y);
            c[2] = __dadd_rn(c[2], b.x);
            c[3] = __dadd_rn(c[3], b.y);
        }
    }
    return comb4(c);
}

__device__ __forceinline__ double rej1(double old, double Nx, float q, bool is_x) {
    return is_x ? 0.0 : fmax(0.0, __dsub_rn(old, __dmul_rn(Nx, f2d(q))));
}

// One rejection: R (p~) and q (in P's place) from shared memory.
__device__ __forceinline__ double reject_next(const float* Qs, double* R, int base_v, int E, double Nx, int x) {
    const int t = threadIdx.x;
    const int i0 = t * E;
    double c[4] = {0.0, 0.0, 0.0, 0.0};
    for (int k = 0; k < E; k += 4) {
        const int i = i0 + k;
        const float4 q4 = *reinterpret_cast<const float4*>(Qs + i);
        const double2 a = *reinterpret_cast<const double2*>(R + i), b = *reinterpret_cast<const double2*>(R + i + 2);
        const double n0 = rej1(a.x, Nx, q4.x, base_v + i == x), n1 = rej1(a.y, Nx, q4.y, base_v + i + 1 == x);
        const double n2 = rej1(b.x, Nx, q4.z, base_v + i + 2 == x), n3 = rej1(b.y, Nx, q4.w, base_v + i + 3 == x);
        *reinterpret_cast<double2*>(R + i) = make_double2(n0, n1);
        *reinterpret_cast<double2*>(R + i + 2) = make_double2(n2, n3);
        c[0] = __dadd_rn(c[0], n0);
        c[1] = __dadd_rn(c[1], n1);
        c[2] = __dadd_rn(c[2], n2);
        c[3] = __dadd_rn(c[3], n3);
    }
    return comb4(c);
}

// Rebuild p~ after `h` rejections from p and q in global memory (the rare
// empty-residual case: the walk keeps the previous residual).
__device__ void rebuild(float* P, double* R, const float* pg, const float* qg, int base_v, int lim, int E,
                        const MssShared& sh, int h) {
    const int i0 = threadIdx.x * E;
    for (int k = 0; k < E; ++k) {
        const int i = i0 + k;
        const float pf = i < lim ? pg[base_v + i] : 0.f;
        const float qf = i < lim ? qg[base_v + i] : 0.f;
        double v = f2d(pf);
        for (int j = 0; j < h; ++j) v = rej1(v, sh.hN[j], qf, base_v + i == sh.hx[j]);
        R[i] = v;
        P[i] = pf;
    }
}

__global__ void __launch_bounds__(kMssThreads, 1) mss_kernel(const MssParams p) {
    cg::cluster_group cl = cg::this_cluster();
    const int C = (int)cl.num_blocks();
    const int rank = (int)cl.block_rank();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    MssShared& sh = *reinterpret_cast<MssShared*>(smem_raw);
    float* P = reinterpret_cast<float*>(smem_raw + align_up(sizeof(MssShared), 128));
    double* R = reinterpret_cast<double*>(P + p.S);  // S is a multiple of 4: 16-B aligned
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int S = p.S, E = p.E, V = p.vocab;
    const int base_v = rank * S;
    const int lim = min(S, max(0, V - base_v));  // valid entries of this slice
    int xbuf = 0;
    int trace_k = 0;
    uint32_t phase = 0;
    if (t == 0) {
        ptx::mbar_init(&sh.bar, 1);
        ptx::fence_mbar_init();
    }
    // the padding past the row end is zero for every node (bulk copies never write it)
    for (int i = lim + t; i < S; i += kMssThreads) P[i] = 0.f;
    __syncthreads();

    pdl_wait();
    const int row_begin = p.tree_offsets[p.req_begin];
    const int row_end = p.tree_offsets[p.req_end];
    const int n_tasks = p.walk ? (p.req_end - p.req_begin) : (row_end - row_begin);
    const int n_clusters = gridDim.x / C;
    const int cid = blockIdx.x / C;

    for (int task = cid; task < n_tasks; task += n_clusters) {
        // ---- task setup: request geometry (and, all-nodes mode, the node) ----
        if (t == 0) {
            int req, node;
            if (p.walk) {
                req = p.req_begin + task;
                node = 0;
            } else {  // the request owning row row_begin + task (binary search)
                const int row = row_begin + task;
                int lo = p.req_begin, hi = p.req_end - 1;
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if (p.tree_offsets[mid] <= row) lo = mid; else hi = mid - 1;
                }
                req = lo;
                node = row - p.tree_offsets[req];
            }
            sh.o = p.tree_offsets[req];
            sh.K = p.tree_offsets[req + 1] - sh.o;
            sh.node = node;
            sh.plen = 0;
            sh.flag = req;
            if (sh.K > AS_MAX_TREE || sh.o + sh.K > p.n_tree_rows || sh.K < 1) {
                if (rank == 0) set_dev_error(p.ws, sh.o + sh.K > p.n_tree_rows ? AS_DEV_ROWS_OVERFLOW : AS_DEV_TREE_TOO_BIG, req);
                sh.K = -1;
            }
        }
        __syncthreads();
        const int K = sh.K, o = sh.o, req = sh.flag;
        if (K < 0) {  // uniform over the cluster (same inputs); records/emitted left as they are
            cl.sync();
            continue;
        }
        for (int k = t; k < K; k += kMssThreads) {
            sh.t_par[k] = p.tree_parent[o + k];
            sh.t_tok[k] = p.tree_tokens[o + k];
            sh.t_uni[k] = p.uni[o + k];
        }
        __syncthreads();
        int bonus = -1;
        for (;;) {  // one node per iteration (all-nodes mode: exactly one)
            const int u = sh.node;
            const int tk = trace_k++;
            cl.sync();  // peers are done reading the previous node's slice from this CTA
            MSS_TRACE(tk, 0, gtime());
            MSS_TRACE(tk, 6, (unsigned long long)u);
            // ---- children of u (warp 0, in local index order) ----
            if (warp == 0) {
                int cnt = 0;
                for (int c0 = u + 1; c0 < K; c0 += 32) {
                    const int c = c0 + lane;
                    const bool is_kid = c < K && sh.t_par[c] == u;
                    const unsigned msk = __ballot_sync(0xffffffffu, is_kid);
                    if (is_kid) sh.kid[cnt + __popc(msk & ((1u << lane) - 1u))] = c;
                    cnt += __popc(msk);
                }
                if (lane == 0) sh.n_kids = cnt;
                __syncwarp();
                const float* qrow = p.q + (size_t)(o + u) * (size_t)V;
                for (int j = lane; j < cnt; j += 32) {  // q(x_j): the decisions read it locally
                    const int x = sh.t_tok[sh.kid[j]];
                    sh.kid_q[j] = (x >= 0 && x < V) ? __ldg(qrow + x) : 0.f;
                }
            }
            __syncthreads();
            const int n_kids = sh.n_kids;
            const size_t row = (size_t)(o + u) * (size_t)V;
            const float* pr = p.p + row;
            const float* qr = p.q + row;
            // ---- the p slice -> shared memory; q slice and the likely next rows -> L2 ----
            if (p.vec4) {
                const uint32_t bytes = (uint32_t)lim * 4u;
                constexpr uint32_t kPiece = 16384;
                const uint32_t pieces = (bytes + kPiece - 1) / kPiece;
                if (warp == 0) {
                    if (lane == 0) {
                        if (bytes) ptx::mbar_arrive_expect_tx(&sh.bar, bytes);
                        else ptx::mbar_arrive(&sh.bar);
                    }
                    __syncwarp();
                    for (uint32_t k = lane; k < pieces; k += 32) {
                        const uint32_t off = k * kPiece;
                        ptx::bulk_g2s(reinterpret_cast<unsigned char*>(P) + off,
                                      reinterpret_cast<const unsigned char*>(pr + base_v) + off,
                                      min(kPiece, bytes - off), &sh.bar);
                    }
                    if (bytes && n_kids > 0 && lane == 31) ptx::bulk_prefetch_l2(qr + base_v, bytes);
                    // walk: the first two children's rows (the likely next node)
                    if (p.walk && bytes && lane < 4 && lane / 2 < n_kids) {
                        const size_t crow = (size_t)(o + sh.kid[lane / 2]) * (size_t)V + base_v;
                        ptx::bulk_prefetch_l2((lane & 1) ? p.q + crow : p.p + crow, bytes);
                    }
                }
                ptx::mbar_wait(&sh.bar, phase);
                phase ^= 1;
            } else {
                for (int i = t; i < lim; i += kMssThreads) P[i] = __ldcs(pr + base_v + i);
            }
            __syncthreads();
            MSS_TRACE(tk, 1, gtime());
            MSS_TRACE(tk, 7, (unsigned long long)n_kids);
            int mat = 0;   // history entries materialised in R (0: p~ = p)
            int hlen = 0;  // rejections so far
            double N = 0.0, tau = 0.0;
            int accepted = -1;
            if (n_kids > 0) {
                // owner / offset of a child's token (owner -1: out of range)
                auto own = [&](int j, int* off) {
                    const int x = sh.t_tok[sh.kid[j]];
                    if (x < 0 || x >= V) {
                        *off = 0;
                        return -1;
                    }
                    *off = x - (x / S) * S;
                    return x / S;
                };
                int xo, xoff;
                xo = own(0, &xoff);
                double rx;  // p~(x_j) under the current residual (pushed by its owner)
                // p -> R (fp64) while summing; then the q slice replaces p in P by bulk
                // copy (from L2: prefetched at the node start), overlapping the mass
                // exchange and the first decision -- every rejection pass then runs
                // from shared memory
                tau = widen_sum(P, R, E);
                mat = 1;
                __syncthreads();  // P is read: the q copy may overwrite it
                const bool q_tma = p.vec4 && lim > 0;
                if (q_tma && warp == 0) {
                    ptx::fence_proxy_async_smem();
                    const uint32_t bytes = (uint32_t)lim * 4u;
                    constexpr uint32_t kPiece = 16384;
                    if (lane == 0) ptx::mbar_arrive_expect_tx(&sh.bar, bytes);
                    __syncwarp();
                    for (uint32_t k = lane; k < (bytes + kPiece - 1) / kPiece; k += 32)
                        ptx::bulk_g2s(reinterpret_cast<unsigned char*>(P) + k * kPiece,
                                      reinterpret_cast<const unsigned char*>(qr + base_v) + k * kPiece,
                                      min(kPiece, bytes - k * kPiece), &sh.bar);
                } else if (!q_tma) {
                    for (int i = t; i < lim; i += kMssThreads) P[i] = __ldg(qr + base_v + i);
                }
                bool q_ready = !q_tma;
                N = cluster_mass(cl, sh, tau, xbuf, C, rank, xo, xoff, P, R, 1, &rx);
                MSS_TRACE(tk, 2, gtime());
                for (int j = 0; j < n_kids; ++j) {
                    const int x = sh.t_tok[sh.kid[j]];
                    // the decision (every thread, identically): p~(x) and q(x) are local
                    bool acc = false;
                    if (x >= 0 && x < V) {
                        const double lhs = __dmul_rn(__dmul_rn((double)sh.t_uni[sh.kid[j]], N), f2d(sh.kid_q[j]));
                        acc = rx > 0.0 && lhs <= rx;
                    } else if (t == 0 && rank == 0) {
                        set_dev_error(p.ws, AS_DEV_BAD_TOKEN, req);
                    }
                    if (acc) {
                        accepted = j;
                        break;
                    }
                    // rejected: p~ <- max(0, p~ - N q), p~(x) <- 0, in place; its mass
                    if (t == 0) {  // history: read only by the rare rebuild below
                        sh.hN[hlen] = N;
                        sh.hx[hlen] = x;
                    }
                    if (!q_ready) {
                        ptx::mbar_wait(&sh.bar, phase);
                        phase ^= 1;
                        q_ready = true;
                    }
                    if (j < 8) MSS_TRACE(32 + tk, j, gtime());
                    tau = reject_next(P, R, base_v, E, N, x);  // R: p~, P: q
                    if (j < 8) MSS_TRACE(48 + tk, j, gtime());
                    if (j + 1 < n_kids) xo = own(j + 1, &xoff);
                    else xo = -1;
                    const double N2 = cluster_mass(cl, sh, tau, xbuf, C, rank, xo, xoff, P, R, 1, &rx);
                    if (N2 == 0.0) {
                        // empty residual: keep the previous p~ -- rebuilt from p and q in
                        // global memory by replaying the hlen earlier rejections (P <- p)
                        rebuild(P, R, pr, qr, base_v, lim, E, sh, hlen);
                        __syncthreads();
                        tau = chunk_sum(P, R, 1, E);
                        break;
                    }
                    ++hlen;
                    N = N2;
                }
                if (!q_ready) {  // accepted before any rejection: retire the q copy
                    ptx::mbar_wait(&sh.bar, phase);
                    phase ^= 1;
                }
            }
            MSS_TRACE(tk, 3, gtime());
            MSS_TRACE(tk, 4, (unsigned long long)hlen);
            int emit;
            if (accepted >= 0) {
                emit = sh.t_tok[sh.kid[accepted]];
            } else {
                // ---- bonus: inverse CDF of the current residual ----
                // (tau / N of the current p~: a leaf computes them now; a node whose
                // children were all rejected has them from its last pass)
                if (n_kids == 0) tau = chunk_sum(P, R, 0, E);
                N = cluster_mass(cl, sh, tau, xbuf, C, rank, -1, 0, P, R, mat, nullptr);
                const double thr = __dmul_rn((double)p.bonus_uni[o + u], N);
                // exclusive prefix of the per-thread chunk sums inside the CTA
                double inc = tau;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const double y = __shfl_up_sync(0xffffffffu, inc, d);
                    if (lane >= d) inc = __dadd_rn(inc, y);
                }
                if (lane == 31) sh.wscan[warp] = inc;
                const int b = xbuf ^ 1;  // the buffer cluster_mass just used
                double pc = 0.0;  // CTA totals before this CTA, in rank order
                for (int c = 0; c < rank; ++c) pc = __dadd_rn(pc, sh.part[b][c]);
                __syncthreads();
                double wpre = 0.0;
                for (int w = 0; w < warp; ++w) wpre = __dadd_rn(wpre, sh.wscan[w]);
                const double base = __dadd_rn(pc, __dadd_rn(wpre, __dsub_rn(inc, tau)));
                // cum(v) = fl(base + s_k), s_k = the sequential prefix of this thread's
                // chunk.  s_k <= s_E <= tau (1 + 2^-40) (tau sums the same non-negative
                // values in another order, E < 2^12 terms) and fl addition is monotone, so
                // a chunk whose fl(base + tau (1 + 2^-40)) < thr holds no crossing.
                int first = INT_MAX;
                if (__dadd_rn(base, __dmul_rn(tau, 1.0 + 0x1p-40)) >= thr) {
                    double s = 0.0;
                    for (int k = 0; k < E && first == INT_MAX; k += 2) {
                        const int i = t * E + k;
                        const double r0 = res_at(P, R, mat, i), r1 = res_at(P, R, mat, i + 1);
                        const double s0 = __dadd_rn(s, r0), s1 = __dadd_rn(s0, r1);
                        if (r0 > 0.0 && __dadd_rn(base, s0) >= thr) first = base_v + i;
                        else if (r1 > 0.0 && __dadd_rn(base, s1) >= thr) first = base_v + i + 1;
                        s = s1;
                    }
                }
                int wm = first;
#pragma unroll
                for (int d = 16; d > 0; d >>= 1) wm = min(wm, __shfl_xor_sync(0xffffffffu, wm, d));
                if (lane == 0) sh.wmin[warp] = wm;
                __syncthreads();
                const int ib = xbuf;
                xbuf ^= 1;
                if (t < 32) {
                    int bm = t < kMssWarps ? sh.wmin[t] : INT_MAX;
#pragma unroll
                    for (int d = 16; d > 0; d >>= 1) bm = min(bm, __shfl_xor_sync(0xffffffffu, bm, d));
                    if (t < C) cl.map_shared_rank(&sh.ipart[ib][0][0], t)[2 * rank] = bm;
                }
                cl.sync();
                int gm = INT_MAX, gl = -1;
                for (int c = 0; c < C; ++c) gm = min(gm, sh.ipart[ib][c][0]);
                if (gm == INT_MAX) {
                    // rounding left the threshold unreached: the last token with mass (rare)
                    int last = -1;
                    for (int k = 0; k < E; ++k)
                        if (res_at(P, R, mat, t * E + k) > 0.0) last = base_v + t * E + k;
#pragma unroll
                    for (int d = 16; d > 0; d >>= 1) last = max(last, __shfl_xor_sync(0xffffffffu, last, d));
                    if (lane == 0) sh.wmax[warp] = last;
                    __syncthreads();
                    const int ib2 = xbuf;
                    xbuf ^= 1;
                    if (t < 32) {
                        int bl = t < kMssWarps ? sh.wmax[t] : -1;
#pragma unroll
                        for (int d = 16; d > 0; d >>= 1) bl = max(bl, __shfl_xor_sync(0xffffffffu, bl, d));
                        if (t < C) cl.map_shared_rank(&sh.ipart[ib2][0][0], t)[2 * rank + 1] = bl;
                    }
                    cl.sync();
                    for (int c = 0; c < C; ++c) gl = max(gl, sh.ipart[ib2][c][1]);
                }
                emit = gm != INT_MAX ? gm : (gl >= 0 ? gl : 0);
                bonus = emit;
                MSS_TRACE(tk, 5, gtime());
            }
            if (t == 0 && rank == 0) {
                if (p.emitted) p.emitted[o + u] = emit;
                if (p.walk) sh.path[sh.plen] = u;
            }
            if (t == 0) {
                sh.plen += 1;
                if (accepted >= 0) sh.node = sh.kid[accepted];
            }
            __syncthreads();
            if (!p.walk || accepted < 0) break;
        }
        // ---- walk: the accept record; unvisited nodes' emitted = -1 ----
        if (p.walk && rank == 0) {
            const int len = sh.plen;
            if (p.records) {
                int32_t* rec = p.records + (size_t)req * (2 + p.max_path);
                for (int k = t; k < p.max_path; k += kMssThreads) rec[2 + k] = k < len ? sh.path[k] : -1;
                if (t == 0) {
                    rec[0] = min(len, p.max_path);
                    rec[1] = bonus;
                    if (len > p.max_path) set_dev_error(p.ws, AS_DEV_PATH_TOO_LONG, req);
                }
            }
            if (p.emitted) {
                __syncthreads();
                for (int k = t; k < K; k += kMssThreads) {
                    bool on = false;
                    for (int m2 = 0; m2 < len; ++m2) on |= sh.path[m2] == k;
                    if (!on) p.emitted[o + k] = -1;
                }
            }
        }
        __syncthreads();
    }
    cl.sync();  // no CTA exits while a peer may still read its shared memory
}

// ---------------------------------------------------------------------------
// Host side.
// ---------------------------------------------------------------------------
constexpr size_t kMssSmemMax = 227 * 1024;

static void mss_geometry(int vocab, int* C, int* E) {
    // smallest E (multiple of 4, E/4 odd) with C * 512 * E >= vocab, C = 8 first;
    // shared memory: p slice (4 B) + materialised residual (8 B) per entry
    for (int c : {8, 16}) {
        int e = 4;
        while ((long long)c * kMssThreads * e < vocab) e += 8;  // 4, 12, 20, ... keep E/4 odd
        if (12LL * e * kMssThreads + (long long)align_up(sizeof(MssShared), 128) <= (long long)kMssSmemMax) {
            *C = c;
            *E = e;
            return;
        }
    }
    *C = 0;
    *E = 0;
}

size_t mss_smem_bytes(int vocab) {
    int C, E;
    mss_geometry(vocab, &C, &E);
    if (!C) return 0;
    return align_up(sizeof(MssShared), 128) + 12 * (size_t)E * kMssThreads;
}

int launch_mss(int req_begin, int req_end, int n_tree_rows, int vocab, const int32_t* tree_offsets,
               const int32_t* tree_parent, const int32_t* tree_tokens, const float* p_rows, const float* q_rows,
               const float* uni, const float* bonus_uni, int32_t* emitted, int32_t* records, int max_path, int walk,
               void* ws, size_t ws_bytes, cudaStream_t stream) {
    int C, E;
    mss_geometry(vocab, &C, &E);
    if (!C) return 1;
    const size_t smem = mss_smem_bytes(vocab);
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return -1;
    int max_clusters = 0;
    {
        static std::mutex mu;
        static bool attrs_set[64] = {false};
        static std::map<std::pair<int, size_t>, int> fit;  // (device, smem) -> active clusters
        std::lock_guard<std::mutex> lk(mu);
        if (!attrs_set[dev]) {
            if (cudaFuncSetAttribute(mss_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMssSmemMax) !=
                    cudaSuccess ||
                cudaFuncSetAttribute(mss_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
                return -1;
            attrs_set[dev] = true;
        }
        auto key = std::make_pair(dev, smem + (size_t)C);
        auto it = fit.find(key);
        if (it == fit.end()) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(C);
            cfg.blockDim = dim3(kMssThreads);
            cfg.dynamicSmemBytes = smem;
            cudaLaunchAttribute a[1];
            a[0].id = cudaLaunchAttributeClusterDimension;
            a[0].val.clusterDim.x = C;
            a[0].val.clusterDim.y = 1;
            a[0].val.clusterDim.z = 1;
            cfg.attrs = a;
            cfg.numAttrs = 1;
            int nc = 0;
            if (cudaOccupancyMaxActiveClusters(&nc, mss_kernel, &cfg) != cudaSuccess || nc < 1) {
                cudaGetLastError();
                return -1;
            }
            it = fit.emplace(key, nc).first;
        }
        max_clusters = it->second;
    }
    const int n_req = req_end - req_begin;
    const long long tasks_hi = walk ? n_req : n_tree_rows;  // upper bound (rows are device-side)
    int n_clusters = (int)(tasks_hi < max_clusters ? tasks_hi : max_clusters);
    if (n_clusters < 1) n_clusters = 1;
    MssParams p;
    p.req_begin = req_begin;
    p.req_end = req_end;
    p.n_tree_rows = n_tree_rows;
    p.vocab = vocab;
    p.tree_offsets = tree_offsets;
    p.tree_parent = tree_parent;
    p.tree_tokens = tree_tokens;
    p.p = p_rows;
    p.q = q_rows;
    p.uni = uni;
    p.bonus_uni = bonus_uni;
    p.emitted = emitted;
    p.records = records;
    p.max_path = max_path;
    p.walk = walk;
    p.E = E;
    p.S = E * kMssThreads;
    p.vec4 = (vocab % 4 == 0) && ((reinterpret_cast<uintptr_t>(p_rows) | reinterpret_cast<uintptr_t>(q_rows)) % 16 == 0);
    p.ws = ws;
    p.trace = nullptr;
#ifdef AS_DEBUG
    if (ws_bytes >= kWsHeaderBytes + 64 * 8 * 8)
        p.trace = reinterpret_cast<unsigned long long*>(reinterpret_cast<unsigned char*>(ws) + kWsHeaderBytes);
#else
    (void)ws_bytes;
#endif
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(n_clusters * C);
    cfg.blockDim = dim3(kMssThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1 + fill_launch_attrs(attr + 1);
    if (cudaLaunchKernelEx(&cfg, mss_kernel, p) != cudaSuccess) return -1;
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace as
