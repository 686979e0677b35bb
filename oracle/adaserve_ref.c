/*
 * adaserve_ref.c -- CPU ORACLE for the AdaServe select -> verify -> accept hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2501_12162_b200/) never links, imports or executes anything under oracle/.
 * It shares no source, header, table or helper with the CUDA library: the layouts
 * below are restated from DESIGN.md, not included from include/adaserve.h.
 *
 * Plain, slow, obviously-correct C99.  Floating point in double unless the paper
 * fixes it.  Every function cites the PAPER.md passage it follows
 * ("P:Lnnn" = line nnn of the paper's LaTeX source) and the DESIGN.md reading
 * (R1..R20) used where the paper is silent or garbled.
 *
 * Pins (tests/test_oracle_*.py, all "-m 'not gpu'"):
 *   asref_select_literal : Fig. 4 golden, exhaustive enumeration vs Alg. 1
 *                          and brute force (App. C), closed-form O2 fuzz,
 *                          library special cases (np.lexsort GlobalGreedy), invariants.
 *   asref_tree_attn      : chain tree == causal attention computed independently with
 *                          torch SDPA / numpy (P-att-1), closed forms O = v_root,
 *                          O = const, uniform weights (P-att-3/4), star-tree permutation.
 *   asref_accept_walk    : Thm. 1 exact enumeration E[accept_len] = sum f,
 *                          chain == sequence speculative decoding, degenerate cases.
 *   asref_commit         : byte-exact cache diff (only path rows change).
 * Parity unpinned: none.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* status codes (restated, same numeric meaning as the library's) */
#define REF_OK 0
#define REF_ERR_INVALID_ARG 1
#define REF_ERR_BUDGET_TOO_SMALL 2
#define REF_ERR_PRECONDITION 6

/* ------------------------------------------------------------------------- */
/* Select: Alg. 2 executed literally, step by step.              */
/* ------------------------------------------------------------------------- */

/* Does candidate a rank before candidate b under "GetTop" inside one request?
 * Paper: GetTop picks "the node with the highest path probability" (P:L702,
 * P:L827).  No tie rule in the paper -> R8: f-hat descending, then lower local
 * index first. */
static int ref_better_local(float fa, int ia, float fb, int ib) {
    if (fa != fb) return fa > fb;
    return ia < ib;
}

/* Global GetTop over the union of requests: R8 order
 * (f-hat desc, request asc, local index asc). */
static int ref_better_global(float fa, int ra, int ia, float fb, int rb, int ib) {
    if (fa != fb) return fa > fb;
    if (ra != rb) return ra < rb;
    return ia < ib;
}

/*
 * asref_select_literal
 *   Inputs (host arrays, CSR forest):
 *     n_req; cand_offsets[n_req+1]; cand_parent[N] local parent (root: 0);
 *     cand_prob[N] f-hat, the draft path-probability product of P:L691-694 (root 1.0);
 *     slo_deficit[n_req] = A(r_i) of P:L549-550 (Eq. 2 rewritten);
 *     depth_d (the speculation depth d, R11), n_max (R6), budget B (R1).
 *   Outputs: tree_offsets[n_req+1], tree_parent[<=B], tree_src[<=B],
 *            tree_depth[<=B], slo_count[n_req] (non-root tokens added in the SLO stage).
 *   Returns REF_OK or REF_ERR_BUDGET_TOO_SMALL (R10: B < n).
 */
int asref_select_literal(int n_req, const int32_t* cand_offsets, const int32_t* cand_parent,
                         const float* cand_prob, const double* slo_deficit, int depth_d,
                         int n_max, int budget, int32_t* tree_offsets, int32_t* tree_parent,
                         int32_t* tree_src, int32_t* tree_depth, int32_t* slo_count) {
    if (n_req < 0 || depth_d < 0 || n_max < 0) return REF_ERR_INVALID_ARG;
    /* Initialization, Alg. 2: every root is in its tree, n_acc = 1.0, B -= 1. */
    if (budget < n_req) return REF_ERR_BUDGET_TOO_SMALL; /* R10 */
    int n_cand = cand_offsets[n_req];
    long B = (long)budget - n_req; /* R1: roots are charged */
    char* added = (char*)calloc((size_t)(n_cand > 0 ? n_cand : 1), 1); /* S_added */
    double* n_acc = (double*)malloc(sizeof(double) * (size_t)(n_req > 0 ? n_req : 1));
    int* order = (int*)malloc(sizeof(int) * (size_t)(n_req > 0 ? n_req : 1));
    for (int i = 0; i < n_req; ++i) {
        n_acc[i] = 1.0;
        added[cand_offsets[i]] = 1;       /* the root is already T(r_i)'s node */
        order[i] = i;
        slo_count[i] = 0;
    }

    /* SLO-customized selection.
     * Sort(requests, key = A(r)): R5 -> descending A ("prioritizes ... larger
     * A(r_i) ... descending order"), ties by ascending request index.  Insertion sort. */
    for (int a = 1; a < n_req; ++a) {
        int x = order[a];
        int b = a - 1;
        while (b >= 0 && (slo_deficit[order[b]] < slo_deficit[x] ||
                          (slo_deficit[order[b]] == slo_deficit[x] && order[b] > x))) {
            order[b + 1] = order[b];
            --b;
        }
        order[b + 1] = x;
    }
    for (int oi = 0; oi < n_req; ++oi) {
        int r = order[oi];
        /* A_cap(r) = min(A(r), d+1) */
        double a_cap = fmin(slo_deficit[r], (double)depth_d + 1.0);
        int added_here = 0;
        /* while n_acc < A_cap  and  |T(r)| < n_max  and  B >= 0
         * readings: R6 -> non-root tokens added in this stage < n_max;
         *           R2 -> B > 0 so that sum |T_i| <= B holds (Eq. 1). */
        while (n_acc[r] < a_cap && added_here < n_max && B > 0) {
            /* v <- GetTop(T_cand(r) - S_added) : linear scan */
            int best = -1;
            for (int j = cand_offsets[r] + 1; j < cand_offsets[r + 1]; ++j) {
                if (added[j]) continue;
                int lj = j - cand_offsets[r];
                if (best < 0 || ref_better_local(cand_prob[j], lj, cand_prob[best],
                                                 best - cand_offsets[r]))
                    best = j;
            }
            if (best < 0) break; /* R7: empty GetTop ends the stage */
            added[best] = 1;     /* T(r).Add(v); S_added.Add(v) */
            /* n_acc += ... : R3 -> the PATH probability f-hat(v) (Fig. 4 sum
             * "0.5 + 0.4", Thm. 1), accumulated in double (R9). */
            n_acc[r] += (double)cand_prob[best];
            B -= 1;
            ++added_here;
        }
        slo_count[r] = added_here;
    }

    /* Throughput-optimized selection: while B >= 0 (R2: B > 0),
     * v <- GetTop(union_i T_cand(r_i) - S_added), add v to its request's tree. */
    while (B > 0) {
        int best = -1, best_r = -1;
        for (int r = 0; r < n_req; ++r) {
            for (int j = cand_offsets[r] + 1; j < cand_offsets[r + 1]; ++j) {
                if (added[j]) continue;
                int lj = j - cand_offsets[r];
                if (best < 0 || ref_better_global(cand_prob[j], r, lj, cand_prob[best], best_r,
                                                  best - cand_offsets[best_r])) {
                    best = j;
                    best_r = r;
                }
            }
        }
        if (best < 0) break; /* R7 */
        added[best] = 1;
        B -= 1;
    }

    /* Emit: each tree lists its selected candidates in ascending local index
     * (topological, since parents precede children), root first; parents are
     * remapped to compact indices; root's parent is itself (R12). */
    int out = 0;
    int* remap = (int*)malloc(sizeof(int) * (size_t)(n_cand > 0 ? n_cand : 1));
    for (int r = 0; r < n_req; ++r) {
        tree_offsets[r] = out;
        int base = out;
        for (int j = cand_offsets[r]; j < cand_offsets[r + 1]; ++j) {
            if (!added[j]) { remap[j] = -1; continue; }
            int lj = j - cand_offsets[r];
            int k = out - base;
            remap[j] = k;
            tree_src[out] = lj;
            if (lj == 0) {
                tree_parent[out] = 0;
                if (tree_depth) tree_depth[out] = 0;
            } else {
                int pj = cand_offsets[r] + cand_parent[j];
                tree_parent[out] = remap[pj]; /* -1 would mean not ancestor-closed */
                if (tree_depth) tree_depth[out] = (remap[pj] >= 0) ? tree_depth[base + remap[pj]] + 1 : -1;
            }
            ++out;
        }
    }
    tree_offsets[n_req] = out;
    free(remap);
    free(order);
    free(n_acc);
    free(added);
    return REF_OK;
}

/* ------------------------------------------------------------------------- */
/* Verify: explicit-mask attention per tree node.                            */
/* ------------------------------------------------------------------------- */
/*
 * Step 4 "verification" verifies all tree tokens in one target
 * forward pass; the paper fixes no mask, so R15: node j of request i attends to
 * every committed prefix key t < L_i (read through the page table, D6/P:L935
 * PagedAttention) plus the tree nodes u with u in anc(j) U {j}.  GQA: q head h
 * uses kv head h / (n_q / n_kv).  softmax(sm_scale * q.k) with no cap/bias.
 *
 * Layouts (restated from DESIGN.md "HBM layout"):
 *   q, out       [n_tree_rows, n_q, d]        row = tree_offsets[i] + j
 *   k_tree,v_tree[n_tree_rows, n_kv, d]
 *   k_cache,v_cache [num_pages, n_kv, page_size, d]
 *   page_table   [n_req, max_pages]           key t of request i lives in
 *                page page_table[i][t / page_size], slot t % page_size
 *   lse          [n_tree_rows, n_q]  natural log of the softmax denominator
 *                (including the max), or NULL.
 * All float inputs are fp32 values (bf16 inputs are widened exactly by the
 * caller).  Arithmetic: fp64; two passes (max, then exp/sum); no tiling.
 * n_threads > 1 parallelises over (request, head) with OpenMP (timing only).
 */
int asref_tree_attn(int n_req, int n_q, int n_kv, int d, const float* q, const float* k_tree,
                    const float* v_tree, const float* k_cache, const float* v_cache,
                    int page_size, const int32_t* page_table, int max_pages,
                    const int32_t* kv_len, const int32_t* tree_offsets,
                    const int32_t* tree_parent, float sm_scale, float* out, float* lse,
                    int n_threads) {
    if (n_req < 0 || n_q <= 0 || n_kv <= 0 || d <= 0 || n_q % n_kv != 0 || page_size <= 0)
        return REF_ERR_INVALID_ARG;
    int G = n_q / n_kv;
    int bad = 0;
#ifdef _OPENMP
    if (n_threads < 1) n_threads = 1;
#pragma omp parallel for schedule(dynamic, 1) num_threads(n_threads) reduction(| : bad)
#endif
    for (long unit = 0; unit < (long)n_req * n_q; ++unit) {
        int i = (int)(unit / n_q);
        int h = (int)(unit % n_q);
        int kvh = h / G;
        int off = tree_offsets[i];
        int K = tree_offsets[i + 1] - off;
        int L = kv_len[i];
        if (K <= 0) continue;
        /* explicit mask: mask[j*K + u] = 1 iff u is an ancestor-or-self of j */
        char* mask = (char*)calloc((size_t)K * K, 1);
        double* s = (double*)malloc(sizeof(double) * (size_t)(L + K));
        double* acc = (double*)malloc(sizeof(double) * (size_t)d);
        for (int j = 0; j < K; ++j) {
            int u = j, steps = 0;
            for (;;) {
                mask[(size_t)j * K + u] = 1;
                if (u == 0) break;
                int p = tree_parent[off + u];
                if (p < 0 || p >= u || ++steps > K) { bad = 1; break; } /* not a forest in topological order */
                u = p;
            }
        }
        for (int j = 0; j < K; ++j) {
            const float* qrow = q + ((size_t)(off + j) * n_q + h) * d;
            int nk = 0;
            /* pass 1: scores over the allowed key list, and their max */
            double m = -INFINITY;
            for (int t = 0; t < L; ++t) {
                int page = page_table[(size_t)i * max_pages + t / page_size];
                const float* krow = k_cache + (((size_t)page * n_kv + kvh) * page_size + t % page_size) * d;
                double dot = 0.0;
                for (int e = 0; e < d; ++e) dot += (double)qrow[e] * (double)krow[e];
                s[nk] = (double)sm_scale * dot;
                if (s[nk] > m) m = s[nk];
                ++nk;
            }
            for (int u = 0; u < K; ++u) {
                if (!mask[(size_t)j * K + u]) continue;
                const float* krow = k_tree + ((size_t)(off + u) * n_kv + kvh) * d;
                double dot = 0.0;
                for (int e = 0; e < d; ++e) dot += (double)qrow[e] * (double)krow[e];
                s[nk] = (double)sm_scale * dot;
                if (s[nk] > m) m = s[nk];
                ++nk;
            }
            /* pass 2: p = exp(s - m), O = sum p v / sum p */
            double denom = 0.0;
            for (int e = 0; e < d; ++e) acc[e] = 0.0;
            nk = 0;
            for (int t = 0; t < L; ++t) {
                int page = page_table[(size_t)i * max_pages + t / page_size];
                const float* vrow = v_cache + (((size_t)page * n_kv + kvh) * page_size + t % page_size) * d;
                double p = exp(s[nk++] - m);
                denom += p;
                for (int e = 0; e < d; ++e) acc[e] += p * (double)vrow[e];
            }
            for (int u = 0; u < K; ++u) {
                if (!mask[(size_t)j * K + u]) continue;
                const float* vrow = v_tree + ((size_t)(off + u) * n_kv + kvh) * d;
                double p = exp(s[nk++] - m);
                denom += p;
                for (int e = 0; e < d; ++e) acc[e] += p * (double)vrow[e];
            }
            float* orow = out + ((size_t)(off + j) * n_q + h) * d;
            for (int e = 0; e < d; ++e) orow[e] = (float)(acc[e] / denom);
            if (lse) lse[(size_t)(off + j) * n_q + h] = (float)(m + log(denom));
        }
        free(acc);
        free(s);
        free(mask);
    }
    return bad ? REF_ERR_PRECONDITION : REF_OK;
}

/* ------------------------------------------------------------------------- */
/* Accept: the sequential acceptance walk and the KV commit.         */
/* ------------------------------------------------------------------------- */
/*
 * "The scheduler uses these logits to identify the verified tokens for each
 * request"; the verification rule is "tree-based verification ... as
 * introduced in prior work".  R13: starting at the root, t* = the
 * target token at the current node (greedy: argmax of that node's logits with
 * the lowest index winning ties; stochastic: a per-node target sample supplied
 * by the caller); move to the lowest-index child whose draft token equals t*,
 * else stop.  R14: accept_len counts the root; bonus = t* at the last accepted
 * node.  accept_path[i][k] = local index of the k-th node on the path, -1 after.
 *
 * target_tokens may be NULL, then target_logits [n_tree_rows, vocab] (fp32
 * values) is used greedily.  Returns REF_ERR_PRECONDITION on a NaN logit or a
 * path longer than max_path (the path is then truncated).
 */
int asref_accept_walk(int n_req, const int32_t* tree_offsets, const int32_t* tree_parent,
                      const int32_t* tree_tokens, const int32_t* target_tokens,
                      const float* target_logits, int vocab, int max_path,
                      int32_t* accept_len, int32_t* accept_path, int32_t* bonus_token) {
    int status = REF_OK;
    for (int i = 0; i < n_req; ++i) {
        int off = tree_offsets[i];
        int K = tree_offsets[i + 1] - off;
        for (int k = 0; k < max_path; ++k) accept_path[(size_t)i * max_path + k] = -1;
        if (K <= 0) { accept_len[i] = 0; bonus_token[i] = -1; continue; }
        int v = 0, len = 1;
        accept_path[(size_t)i * max_path] = 0;
        int tstar;
        for (;;) {
            if (target_tokens) {
                tstar = target_tokens[off + v];
            } else {
                const float* row = target_logits + (size_t)(off + v) * vocab;
                int arg = 0;
                for (int t = 0; t < vocab; ++t) {
                    if (row[t] != row[t]) { status = REF_ERR_PRECONDITION; }
                    if (row[t] > row[arg]) arg = t; /* strict > : lowest index wins ties */
                }
                tstar = arg;
            }
            int next = -1;
            for (int c = v + 1; c < K; ++c) {
                if (tree_parent[off + c] == v && tree_tokens[off + c] == tstar) { next = c; break; }
            }
            if (next < 0) break;
            if (len >= max_path) { status = REF_ERR_PRECONDITION; break; }
            accept_path[(size_t)i * max_path + len] = next;
            ++len;
            v = next;
        }
        accept_len[i] = len;
        bonus_token[i] = tstar;
    }
    return status;
}

/*
 * asref_commit: copy the accepted path rows of k_tree/v_tree (R16: the tree's
 * K/V live in dense per-node arrays) into cache slots [L_i, L_i + accept_len)
 * through the page table, then kv_len[i] += accept_len (R14: the root and the
 * accepted drafts are committed; the bonus becomes the next root).
 * elem_bytes = 2 (bf16) or 4 (fp32); copies are byte-exact.
 * Returns REF_ERR_PRECONDITION if a slot falls outside max_pages pages.
 */
int asref_commit(int n_req, const int32_t* tree_offsets, const int32_t* accept_len,
                 const int32_t* accept_path, int max_path, const void* k_tree,
                 const void* v_tree, int elem_bytes, int n_kv, int d, void* k_cache,
                 void* v_cache, int page_size, const int32_t* page_table, int max_pages,
                 int32_t* kv_len) {
    int status = REF_OK;
    size_t row_bytes = (size_t)d * elem_bytes;
    for (int i = 0; i < n_req; ++i) {
        int L = kv_len[i];
        int len = accept_len[i];
        for (int k = 0; k < len; ++k) {
            int node = tree_offsets[i] + accept_path[(size_t)i * max_path + k];
            int slot = L + k;
            if (slot / page_size >= max_pages) { status = REF_ERR_PRECONDITION; break; }
            int page = page_table[(size_t)i * max_pages + slot / page_size];
            for (int h = 0; h < n_kv; ++h) {
                size_t src = ((size_t)node * n_kv + h) * row_bytes;
                size_t dst = (((size_t)page * n_kv + h) * page_size + slot % page_size) * row_bytes;
                memcpy((char*)k_cache + dst, (const char*)k_tree + src, row_bytes);
                memcpy((char*)v_cache + dst, (const char*)v_tree + src, row_bytes);
            }
        }
        kv_len[i] = L + len;
    }
    return status;
}
