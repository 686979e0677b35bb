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
// p~ after h rejections is never stored: residual() replays the h updates on
// the (p, q) pair -- the same sequence of fp64 operations the oracle performs
// (one __dmul_rn, one __dsub_rn, one max per rejection; no FMA), so every
// element value is bit-identical to oracle/mss.py's; only the sums' association
// differs (last bits -- the oracle reports each decision's margin).
//
// One thread-block cluster of C CTAs (C = 8, or 16 for vocabularies past 180k)
// per task.  CTA c holds the slice [c S, (c+1) S) of the node's p and q rows in
// shared memory (S = E * 512 floats, E a multiple of 4 with E/4 odd so the
// per-thread float4 chunks are bank-conflict free): the rows are read from HBM
// ONCE per node, every later pass (the residual mass after each rejection, the
// bonus inverse CDF) runs from shared memory, and the cluster combines per-CTA
// fp64 partials through DSMEM (each CTA writes its partial into every peer,
// one cluster barrier, all CTAs sum them in rank order -> identical N
// everywhere).  A decision reads p(x), q(x) straight from the owning CTA's
// shared memory (ld.shared::cluster).
//   walk = 1: task = request; the cluster walks from the root, visiting only the
//             nodes on the accepted path (HBM traffic = path rows, not tree rows),
//             and writes the accept record {len, bonus, path} (the layout of
//             as_accept_tokens' *_RECORDS phases: AS_ACCEPT_COMMIT_RECORDS then
//             commits the path's K/V).
//   walk = 0: task = node; every node's emitted token (all-nodes mode).
// Persistent grid: as many clusters as fit (one 150 KB CTA per SM), tasks strided.
#include <cooperative_groups.h>
#include <mutex>
#include <map>

#include "params.cuh"

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
};

struct MssShared {
    double hN[kMssMaxKids];      // history: mass N_k before rejection k
    int hx[kMssMaxKids];         // history: rejected token x_k
    int kid[kMssMaxKids];        // children of the current node (local index)
    double part[2][kMssMaxC];    // cluster exchange of CTA partial sums (double-buffered)
    int ipart[2][kMssMaxC][2];   // cluster exchange of (first crossing, last with mass)
    double wsum[kMssWarps];
    double wscan[kMssWarps];
    int wmin[kMssWarps], wmax[kMssWarps];
    int t_par[AS_MAX_TREE];      // the task's request: parents, draft tokens, uniforms
    int t_tok[AS_MAX_TREE];
    float t_uni[AS_MAX_TREE];
    int n_kids, hlen, node, K, o, flag;
    double N;
    int path[AS_MAX_TREE];
    int plen;
};

__device__ __forceinline__ double residual(float pf, float qf, int v, const MssShared& sh, int hlen) {
    double t = (double)pf;
    const double qd = (double)qf;
    for (int k = 0; k < hlen; ++k) t = (v == sh.hx[k]) ? 0.0 : fmax(0.0, __dsub_rn(t, __dmul_rn(sh.hN[k], qd)));
    return t;
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Cluster-wide sum of one fp64 value per CTA: written into every peer's slot,
// one cluster barrier, summed in rank order (identical result on every CTA).
__device__ double cluster_sum(cg::cluster_group& cl, MssShared& sh, double mine, int& xbuf, int C, int rank) {
    const int b = xbuf;
    xbuf ^= 1;
    if (threadIdx.x < (unsigned)C) cl.map_shared_rank(&sh.part[b][0], (int)threadIdx.x)[rank] = mine;
    cl.sync();
    double s = 0.0;
    for (int c = 0; c < C; ++c) s = __dadd_rn(s, sh.part[b][c]);
    return s;
}

// One pass over the CTA's slice: tau = this thread's sequential residual sum
// over its chunk; the CTA total (warp xor trees, warps in order); the cluster
// mass.  Returns N (every thread); *tau_out = tau; *cta_out = the CTA total.
__device__ double mass_pass(cg::cluster_group& cl, MssShared& sh, const float* P, const float* Q, int base_v,
                            int E, int hlen, int& xbuf, int C, int rank, double* tau_out, double* cta_out) {
    const int t = threadIdx.x;
    const float4* P4 = reinterpret_cast<const float4*>(P + t * E);
    const float4* Q4 = reinterpret_cast<const float4*>(Q + t * E);
    double tau = 0.0;
    const int v0 = base_v + t * E;
    if (hlen == 0) {
        for (int k = 0; k < E / 4; ++k) {
            const float4 a = P4[k];
            tau = __dadd_rn(tau, (double)a.x);
            tau = __dadd_rn(tau, (double)a.y);
            tau = __dadd_rn(tau, (double)a.z);
            tau = __dadd_rn(tau, (double)a.w);
        }
    } else {
        for (int k = 0; k < E / 4; ++k) {
            const float4 a = P4[k], b = Q4[k];
            const int v = v0 + 4 * k;
            tau = __dadd_rn(tau, residual(a.x, b.x, v, sh, hlen));
            tau = __dadd_rn(tau, residual(a.y, b.y, v + 1, sh, hlen));
            tau = __dadd_rn(tau, residual(a.z, b.z, v + 2, sh, hlen));
            tau = __dadd_rn(tau, residual(a.w, b.w, v + 3, sh, hlen));
        }
    }
    *tau_out = tau;
    const double ws = warp_sum_d(tau);
    if ((t & 31) == 0) sh.wsum[t >> 5] = ws;
    __syncthreads();
    double cta = 0.0;
    for (int w = 0; w < kMssWarps; ++w) cta = __dadd_rn(cta, sh.wsum[w]);
    *cta_out = cta;
    return cluster_sum(cl, sh, cta, xbuf, C, rank);
}

__global__ void __launch_bounds__(kMssThreads, 1) mss_kernel(const MssParams p) {
    cg::cluster_group cl = cg::this_cluster();
    const int C = (int)cl.num_blocks();
    const int rank = (int)cl.block_rank();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    MssShared& sh = *reinterpret_cast<MssShared*>(smem_raw);
    float* P = reinterpret_cast<float*>(smem_raw + align_up(sizeof(MssShared), 128));
    float* Q = P + p.S;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int S = p.S, E = p.E, V = p.vocab;
    const int base_v = rank * S;
    int xbuf = 0;

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
            cl.sync();  // peers are done reading the previous node's rows from this CTA
            // ---- children of u (warp 0, in local index order), then the rows ----
            if (warp == 0) {
                int cnt = 0;
                for (int c0 = u + 1; c0 < K; c0 += 32) {
                    const int c = c0 + lane;
                    const bool is_kid = c < K && sh.t_par[c] == u;
                    const unsigned m = __ballot_sync(0xffffffffu, is_kid);
                    if (is_kid) sh.kid[cnt + __popc(m & ((1u << lane) - 1u))] = c;
                    cnt += __popc(m);
                }
                if (lane == 0) sh.n_kids = cnt;
            }
            __syncthreads();
            const int n_kids = sh.n_kids;
            const bool need_q = n_kids > 0;  // a leaf only samples its bonus from p
            const size_t row = (size_t)(o + u) * (size_t)V;
            const float* pr = p.p + row;
            const float* qr = p.q + row;
            const int lim = min(S, max(0, V - base_v));  // valid floats of this slice
            if (p.vec4) {
                const float4* pr4 = reinterpret_cast<const float4*>(pr + base_v);
                const float4* qr4 = reinterpret_cast<const float4*>(qr + base_v);
                float4* P4 = reinterpret_cast<float4*>(P);
                float4* Q4 = reinterpret_cast<float4*>(Q);
                const int n4 = lim >> 2;
                const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
                int i = t;
                for (; i + 3 * kMssThreads < n4; i += 4 * kMssThreads) {
                    float4 a[4], b[4];
#pragma unroll
                    for (int k = 0; k < 4; ++k) a[k] = __ldcs(pr4 + i + k * kMssThreads);
                    if (need_q) {
#pragma unroll
                        for (int k = 0; k < 4; ++k) b[k] = __ldcs(qr4 + i + k * kMssThreads);
                    } else {
#pragma unroll
                        for (int k = 0; k < 4; ++k) b[k] = z;
                    }
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        P4[i + k * kMssThreads] = a[k];
                        Q4[i + k * kMssThreads] = b[k];
                    }
                }
                for (; i < n4; i += kMssThreads) {
                    P4[i] = __ldcs(pr4 + i);
                    Q4[i] = need_q ? __ldcs(qr4 + i) : z;
                }
                for (int j = n4 + t; j < (S >> 2); j += kMssThreads) {
                    P4[j] = z;
                    Q4[j] = z;
                }
            } else {
                for (int i = t; i < S; i += kMssThreads) {
                    P[i] = i < lim ? __ldcs(pr + base_v + i) : 0.f;
                    Q[i] = (i < lim && need_q) ? __ldcs(qr + base_v + i) : 0.f;
                }
            }
            __syncthreads();
            double tau = 0.0, cta = 0.0, N = 0.0;
            int accepted = -1;
            int hlen = 0;
            if (n_kids > 0) {
                N = mass_pass(cl, sh, P, Q, base_v, E, 0, xbuf, C, rank, &tau, &cta);
                for (int j = 0; j < n_kids; ++j) {
                    const int x = sh.t_tok[sh.kid[j]];
                    bool acc = false;
                    if (x >= 0 && x < V) {
                        const int owner = x / S, off = x - owner * S;
                        const float px = *cl.map_shared_rank(P + off, owner);
                        const float qx = *cl.map_shared_rank(Q + off, owner);
                        const double rx = residual(px, qx, x, sh, hlen);
                        const double lhs = __dmul_rn(__dmul_rn((double)sh.t_uni[sh.kid[j]], N), (double)qx);
                        acc = rx > 0.0 && lhs <= rx;
                    } else if (t == 0 && rank == 0) {
                        set_dev_error(p.ws, AS_DEV_BAD_TOKEN, req);
                    }
                    if (acc) {
                        accepted = j;
                        break;
                    }
                    // rejected: the residual after this rejection and its mass (entry
                    // hlen is read by nobody before the barrier below)
                    if (t == 0) {
                        sh.hN[hlen] = N;
                        sh.hx[hlen] = x;
                    }
                    __syncthreads();
                    const double N2 = mass_pass(cl, sh, P, Q, base_v, E, hlen + 1, xbuf, C, rank, &tau, &cta);
                    if (N2 == 0.0) break;  // empty residual: keep the previous p~
                    ++hlen;
                    N = N2;
                }
            }
            int emit;
            if (accepted >= 0) {
                emit = sh.t_tok[sh.kid[accepted]];
            } else {
                // ---- bonus: inverse CDF of the current residual ----
                N = mass_pass(cl, sh, P, Q, base_v, E, hlen, xbuf, C, rank, &tau, &cta);
                const double thr = __dmul_rn((double)p.bonus_uni[o + u], N);
                // exclusive prefix of the per-thread chunk sums inside the CTA
                double inc = tau;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const double y = __shfl_up_sync(0xffffffffu, inc, d);
                    if (lane >= d) inc = __dadd_rn(inc, y);
                }
                if (lane == 31) sh.wscan[warp] = inc;
                // prefix of the CTA totals before this CTA, in rank order
                const int b = xbuf ^ 1;  // the buffer mass_pass just used
                double pc = 0.0;
                for (int c = 0; c < rank; ++c) pc = __dadd_rn(pc, sh.part[b][c]);
                __syncthreads();
                double wpre = 0.0;
                for (int w = 0; w < warp; ++w) wpre = __dadd_rn(wpre, sh.wscan[w]);
                const double base = __dadd_rn(pc, __dadd_rn(wpre, __dsub_rn(inc, tau)));
                int first = INT_MAX, last = -1;
                double s = 0.0;
                const int v0 = base_v + t * E;
                for (int k = 0; k < E; ++k) {
                    const int v = v0 + k;
                    const double val = hlen ? residual(P[t * E + k], Q[t * E + k], v, sh, hlen) : (double)P[t * E + k];
                    if (val > 0.0) {
                        last = v;
                        s = __dadd_rn(s, val);
                        if (__dadd_rn(base, s) >= thr) {
                            first = v;
                            break;
                        }
                    }
                }
                int wm = first, wl = last;
#pragma unroll
                for (int d = 16; d > 0; d >>= 1) {
                    wm = min(wm, __shfl_xor_sync(0xffffffffu, wm, d));
                    wl = max(wl, __shfl_xor_sync(0xffffffffu, wl, d));
                }
                if (lane == 0) {
                    sh.wmin[warp] = wm;
                    sh.wmax[warp] = wl;
                }
                __syncthreads();
                if (t == 0) {
                    int bm = INT_MAX, bl = -1;
                    for (int w = 0; w < kMssWarps; ++w) {
                        bm = min(bm, sh.wmin[w]);
                        bl = max(bl, sh.wmax[w]);
                    }
                    sh.wmin[0] = bm;
                    sh.wmax[0] = bl;
                }
                __syncthreads();
                const int ib = xbuf;
                xbuf ^= 1;
                if (t < C) {
                    int* dst = cl.map_shared_rank(&sh.ipart[ib][0][0], t);
                    dst[2 * rank] = sh.wmin[0];
                    dst[2 * rank + 1] = sh.wmax[0];
                }
                cl.sync();
                int gm = INT_MAX, gl = -1;
                for (int c = 0; c < C; ++c) {
                    gm = min(gm, sh.ipart[ib][c][0]);
                    gl = max(gl, sh.ipart[ib][c][1]);
                }
                emit = gm != INT_MAX ? gm : (gl >= 0 ? gl : 0);
                bonus = emit;
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
                    for (int m = 0; m < len; ++m) on |= sh.path[m] == k;
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
static void mss_geometry(int vocab, int* C, int* E) {
    // smallest E (multiple of 4, E/4 odd) with C * 512 * E >= vocab, C = 8 first
    for (int c : {8, 16}) {
        int e = 4;
        while ((long long)c * kMssThreads * e < vocab) e += 8;  // 4, 12, 20, ... keep E/4 odd
        if (2LL * e * kMssThreads * 4 + (long long)align_up(sizeof(MssShared), 128) <= 200 * 1024) {
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
    return align_up(sizeof(MssShared), 128) + 2 * (size_t)E * kMssThreads * 4;
}

int launch_mss(int req_begin, int req_end, int n_tree_rows, int vocab, const int32_t* tree_offsets,
               const int32_t* tree_parent, const int32_t* tree_tokens, const float* p_rows, const float* q_rows,
               const float* uni, const float* bonus_uni, int32_t* emitted, int32_t* records, int max_path, int walk,
               void* ws, cudaStream_t stream) {
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
            if (cudaFuncSetAttribute(mss_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) !=
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
