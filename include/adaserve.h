/*
 * adaserve.h -- C ABI of the B200-native AdaServe hot path (libadaserve.so).
 *
 * The three calls are the data-parallel hot path of one speculate-select-verify
 * iteration of AdaServe (arXiv 2501.12162, "SLO-Customized LLM Serving with
 * Fine-Grained Speculative Decoding").  Citations "P:Lnnn" are lines of the
 * paper's LaTeX source; "Rnn" are the readings listed in DESIGN.md
 * where the paper is silent or ambiguous.
 *
 *   as_select_trees      Alg. 2 SLO-customized + throughput-optimized selection
 *                         on the GPU.
 *   as_tree_verify_attn  Step 4 verification attention:
 *                        every tree node attends to its request's paged KV
 *                        prefix plus its tree ancestors.
 *   as_accept_tokens     "uses these logits to identify the verified tokens"
 *                        (P:L860): greedy/stochastic acceptance walk and the
 *                        KV commit of the accepted path.
 *   as_mss_verify        SpecInfer multi-step speculative sampling for trees
 *                        of drawn drafts (reading R25).
 *
 * Conventions (all calls):
 *  - Every pointer argument is a DEVICE pointer unless stated otherwise; all
 *    arrays are dense, row-major, naturally aligned; tensors of bf16/fp32
 *    elements additionally need 16-byte aligned base pointers and row strides.
 *  - Calls are asynchronous and ordered on `stream` (a cudaStream_t passed as
 *    void*; NULL = legacy default stream).  The library never allocates or frees
 *    device memory and never synchronises the host (except as_check_device_error).
 *  - Scratch memory is caller-owned `workspace` of at least as_*_workspace_size()
 *    bytes, 256-byte aligned, ZERO-FILLED ONCE before its first use (the library
 *    leaves it reusable after every call).  One workspace must not be used by two
 *    calls that may run concurrently.
 *  - Host-checkable errors return a status and launch nothing.  Data-dependent
 *    precondition violations (listed per call) are detected on the device: the
 *    kernel records a sticky {code, request} pair in the workspace header and
 *    still finishes with defined-but-unspecified outputs; read it with
 *    as_check_device_error().  Launch failures return AS_ERR_CUDA.  No C++
 *    exception crosses this ABI.  Thread-safe and re-entrant.
 */
#ifndef ADASERVE_H_
#define ADASERVE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    AS_OK = 0,
    AS_ERR_INVALID_ARG = 1,      /* null pointer, negative size, inconsistent shape  */
    AS_ERR_BUDGET_TOO_SMALL = 2, /* budget < n_req (R10)                             */
    AS_ERR_UNSUPPORTED = 3,      /* head_dim / page_size / dtype / GQA ratio        */
    AS_ERR_WORKSPACE = 4,        /* workspace too small or misaligned                */
    AS_ERR_CUDA = 5              /* a CUDA runtime/driver call failed               */
} as_status;

typedef enum { AS_F32 = 0, AS_BF16 = 1 } as_dtype;

/* Device-side precondition codes (workspace header, see as_check_device_error). */
enum {
    AS_DEV_OK = 0,
    AS_DEV_BAD_PARENT = 1,     /* parent not in [0, j) for node j > 0 (not topological)   */
    AS_DEV_BAD_PROB = 2,       /* f-hat NaN, <= 0, or > f-hat(parent)                     */
    AS_DEV_TOO_MANY_CAND = 3,  /* a request has more than AS_MAX_CAND non-root candidates */
    AS_DEV_TREE_TOO_BIG = 4,   /* a tree exceeds AS_MAX_TREE nodes in attention          */
    AS_DEV_ROWS_OVERFLOW = 5,  /* tree_offsets[n_req] > n_tree_rows                       */
    AS_DEV_PAGE_OVERFLOW = 6,  /* a KV slot falls outside the request's page-table row    */
    AS_DEV_NAN_LOGIT = 7,      /* NaN in target_logits                                    */
    AS_DEV_PATH_TOO_LONG = 8,  /* accepted path longer than max_path (truncated)          */
    AS_DEV_BAD_PAGE = 9,       /* page id outside [0, num_pages)                          */
    AS_DEV_BAD_TOKEN = 10,     /* draft token outside [0, vocab) (as_mss_verify)          */
    AS_DEV_NOT_RESIDENT = 11   /* split-KV pieces not co-resident (SMs held elsewhere): gave up */
};

#define AS_MAX_TREE 256 /* nodes per tree (incl. root) accepted by as_tree_verify_attn */
#define AS_MAX_CAND 256 /* non-root candidates per request accepted by as_select_trees */
#define AS_MAX_BEAM 16  /* beam width accepted by as_beam_step */

/* ------------------------------------------------------------------------- */
/* Speculation: one beam-search layer (Step 1)                    */
/* ------------------------------------------------------------------------- */
/*
 * Builds layer `layer` (1..d) of every request's candidate tree (the input of
 * as_select_trees) from the draft model's distributions at the kept nodes of
 * layer-1.  Every expansion (parent k, token t) gets the approximated path
 * probability f-hat = fl32(f-hat(k) * draft_probs[i][k][t]) (the product of
 * draft conditionals along the path); the layer keeps the `width`
 * largest by (f-hat desc, parent rank asc, token asc) (R8).
 *
 * Forest layout (the one as_select_trees reads): request i owns candidates
 * [i*cand_stride, (i+1)*cand_stride), cand_stride >= 1 + layer*width; local
 * node 0 is the root (caller-initialised: parent 0, prob 1.0, its token);
 * layer l occupies local nodes 1 + (l-1)*width + r, r = rank (0 = best), so the
 * kept nodes of layer l-1 are the w_in = (l == 1 ? 1 : width) nodes before it.
 * Inputs (device):
 *   draft_probs [n_req][w_in][vocab] fp32  M_q(t | X, Path(node)) of the kept
 *                nodes of layer-1 in rank order; finite and >= 0.
 *   cand_prob    read: f-hat of the layer-1 nodes.
 * Outputs (device): cand_parent / cand_prob / cand_token of the layer's
 *   `width` nodes (parent = local index of the kept parent).
 * Scalars: 1 <= width <= AS_MAX_BEAM, width <= vocab (every layer then keeps
 *   exactly `width` nodes), layer >= 1, w_in*vocab < 2^32.
 * Workspace >= as_beam_workspace_size(n_req, width, vocab) (chunk top-w lists).
 * Device preconditions: AS_DEV_BAD_PROB (a negative probability); a NaN
 *   probability is treated as 0 (never preferred to a real one).
 */
size_t as_beam_workspace_size(int32_t n_req, int32_t width, int32_t vocab);
as_status as_beam_step(int32_t n_req, int32_t layer, int32_t width, int32_t vocab,
                       const float* draft_probs, int32_t cand_stride, int32_t* cand_parent,
                       float* cand_prob, int32_t* cand_token, void* workspace,
                       size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------------------- */
/* Select: Alg. 2                                                */
/* ------------------------------------------------------------------------- */
/*
 * Builds each request's draft token tree from its candidate tree (the beam of
 * Step 1) under the global budget B (Eq. 1) and the
 * per-request SLO threshold A_cap(r) = min(A(r), d+1):
 *   roots are charged first (B0 = B - n, R1);
 *   SLO stage: requests in descending A (ties: lower id, R5) take their best
 *     remaining candidates (f-hat desc, then lower local index, R8) while
 *     1.0 + sum f-hat (fp64, R3/R9) < A_cap, at most n_max each (R6), and while
 *     budget remains (R2);
 *   throughput stage: the remaining budget goes to the global best candidates
 *     (f-hat desc, request asc, index asc, R8).
 * The result is bit-identical to the sequential algorithm (the oracle).
 *
 * Inputs (device):
 *   cand_offsets [n_req+1]  CSR offsets; request i owns candidates
 *                           [cand_offsets[i], cand_offsets[i+1]); local index 0
 *                           is the root; 1 <= C_i, C_i - 1 <= AS_MAX_CAND.
 *   cand_parent  [N]        local parent; parent of root = 0; 0 <= parent[j] < j.
 *   cand_prob    [N] f32    f-hat = product of draft conditionals on the path
 *                           (P:L691-694); root 1.0; 0 < f[j] <= f[parent[j]].
 *   cand_token   [N] i32    draft token id per candidate, or NULL.
 *   slo_deficit  [n_req] f64  A(r_i) = (l_i + t_spec)/t_TPOT_i - o_i, finite.
 * Scalars (host): n_req >= 0; n_cand_total = cand_offsets[n_req] (host copy,
 *   used only to size/check the workspace); depth_d >= 0 (R11); n_max >= 0;
 *   budget >= n_req.
 * Outputs (device):
 *   tree_offsets [n_req+1]  tree_offsets[n_req] = nodes used <= budget.
 *   tree_parent  [budget]   compact local parent (root -> 0), topological.
 *   tree_src     [budget]   local candidate index, ascending within a tree.
 *   tree_depth   [budget]   or NULL.
 *   tree_token   [budget]   cand_token[src] or NULL (requires cand_token).
 *   slo_count    [n_req]    non-root nodes taken in the SLO stage, or NULL.
 *   Entries beyond tree_offsets[n_req] are left untouched.
 * Device preconditions: AS_DEV_BAD_PARENT, AS_DEV_BAD_PROB, AS_DEV_TOO_MANY_CAND.
 */
size_t as_select_workspace_size(int32_t n_req, int32_t n_cand_total);
as_status as_select_trees(int32_t n_req, int32_t n_cand_total, const int32_t* cand_offsets,
                          const int32_t* cand_parent, const float* cand_prob,
                          const int32_t* cand_token, const double* slo_deficit, int32_t depth_d,
                          int32_t n_max, int32_t budget, int32_t* tree_offsets,
                          int32_t* tree_parent, int32_t* tree_src, int32_t* tree_depth,
                          int32_t* tree_token, int32_t* slo_count, void* workspace,
                          size_t workspace_bytes, void* stream);

/*
 * Selection variants without SLO awareness (NEXT-4; reading R24 in DESIGN.md):
 * request i keeps its root plus its best m_i candidates, chosen greedily by
 * (f-hat desc, lower local index) (R8) -- the first m_i entries of pi_i, an
 * ancestor-closed set (App. B) -- with
 *   m_i = min(m_base + (i < m_extra ? 1 : 0), C_i - 1).
 *   EqualGreedy (dead-text ablation "evenly distributes the budget among
 *   requests and greedily selects tokens ... for each request"): budget B split
 *   evenly, m_base = floor(B / n) - 1, m_extra = B mod n (a share a request
 *   cannot fill stays unused); Eagle-2 top-m: m_base = m, m_extra = 0.
 * Same inputs/outputs as as_select_trees (no slo_deficit, depth_d or budget;
 * tree_parent / tree_src / tree_depth / tree_token need sum_i (1 + m_i) rows);
 * kept [n_req] (or NULL) receives m_i.  Requires 0 <= m_extra <= n_req,
 * m_base >= 0.  Same kernel, device preconditions and workspace as
 * as_select_trees; bit-identical to the per-request greedy loop (the oracle).
 */
as_status as_select_topm(int32_t n_req, int32_t n_cand_total, const int32_t* cand_offsets,
                         const int32_t* cand_parent, const float* cand_prob, const int32_t* cand_token,
                         int32_t m_base, int32_t m_extra, int32_t* tree_offsets, int32_t* tree_parent,
                         int32_t* tree_src, int32_t* tree_depth, int32_t* tree_token, int32_t* kept,
                         void* workspace, size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------------------- */
/* Verify: tree-masked attention over the paged KV cache */
/* ------------------------------------------------------------------------- */
/*
 * For request i, tree node j (global row r = tree_offsets[i] + j) and query
 * head h (kv head h / (n_q_heads / n_kv_heads)):
 *   out[r, h] = softmax_k(sm_scale * q[r,h] . key_k) value_k
 * over the keys k = committed prefix positions t < kv_len[i] (key/value at page
 * page_table[i][t / page_size], slot t % page_size of k_cache / v_cache) and the
 * tree nodes u that are ancestors of j or j itself (k_tree/v_tree rows
 * tree_offsets[i] + u) (R15, R16).  A chain tree is exactly causal decoding.
 * lse[r, h] = natural log of sum_k exp(sm_scale q.key_k) (optional).
 *
 * dtype AS_BF16: q, k_tree, v_tree, caches, out are bf16; tcgen05 tensor-core
 *   path (fp32 accumulation in TMEM, fp32 softmax, P rounded to bf16).
 * dtype AS_F32: all fp32; CUDA-core path (the 1e-5 parity configuration).
 * Layouts:
 *   q, out        [n_tree_rows, n_q_heads, head_dim]
 *   k_tree,v_tree [n_tree_rows, n_kv_heads, head_dim]   (RoPE already applied)
 *   k_cache,v_cache [num_pages, n_kv_heads, page_size, head_dim]
 *   page_table    [n_req, max_pages_per_req] i32
 *   kv_len        [n_req] i32, 0 <= kv_len[i] <= max_pages_per_req * page_size
 *   tree_offsets  [n_req+1], tree_parent [n_tree_rows] (compact local parents,
 *                 as produced by as_select_trees); rows >= tree_offsets[n_req]
 *                 of out/lse are not written.
 *   lse           [n_tree_rows, n_q_heads] f32, or NULL.
 * Supported: head_dim in {64, 128}; page_size in {16, 32, 64, 128};
 *   n_q_heads % n_kv_heads == 0; for AS_BF16 the group size n_q/n_kv must be
 *   a power of two <= 16.  Heads are the caller's LOCAL heads (KV-head sharding).
 * Device preconditions: AS_DEV_TREE_TOO_BIG, AS_DEV_BAD_PARENT,
 *   AS_DEV_ROWS_OVERFLOW, AS_DEV_BAD_PAGE; AS_DEV_NOT_RESIDENT if the split-KV
 *   pieces of a unit cannot all be resident (the device shared with another
 *   tenant): the call returns after 0.5 s with that unit's output unspecified.
 */
size_t as_attn_workspace_size(as_dtype dtype, int32_t n_req, int32_t n_tree_rows,
                              int32_t n_q_heads, int32_t head_dim, int32_t max_kv_len);
as_status as_tree_verify_attn(as_dtype dtype, int32_t n_req, int32_t n_tree_rows,
                              int32_t n_q_heads, int32_t n_kv_heads, int32_t head_dim,
                              const void* q, const void* k_tree, const void* v_tree,
                              const void* k_cache, const void* v_cache, int32_t num_pages,
                              int32_t page_size, const int32_t* page_table,
                              int32_t max_pages_per_req, const int32_t* kv_len,
                              const int32_t* tree_offsets, const int32_t* tree_parent,
                              float sm_scale, void* out, float* lse, void* workspace,
                              size_t workspace_bytes, void* stream);

/*
 * Schedule override of the bf16 path (A/B tests and tuning; every choice gives
 * bit-identical results).  NULL or zero fields = the library's choice.
 *   q_tiles_per_cta  1: one 128-row q-tile per CTA (2 CTAs / SM); 2: the two
 *                    q-tiles of a (request, kv head) in one CTA sharing every
 *                    K/V tile (1 CTA / SM); 0: auto (2 when trees span > 1 q-tile)
 *   cluster_ctas     2 or 4: clusters of one-q-tile CTAs, each K/V tile fetched
 *                    once and multicast (measured slower); 0/1: none
 *   split            0: whole units only; 1 or -1/auto: split-KV / tail pieces allowed
 *   cta_pair         1: CTA pairs -- one tcgen05.mma.cta_group::2 (M = 256) per q-tile
 *                    pair of a 2-CTA cluster, each CTA loading half of every K/V tile
 *                    (head_dim 128, page_size >= 64, >= 2 q-tiles per (request, kv
 *                    head), else AS_ERR_UNSUPPORTED); 0 / -1: not used
 * Unknown values return AS_ERR_INVALID_ARG.
 */
typedef struct {
    int32_t q_tiles_per_cta;
    int32_t cluster_ctas;
    int32_t split;
    int32_t cta_pair;
} as_attn_schedule;

as_status as_tree_verify_attn_sched(as_dtype dtype, int32_t n_req, int32_t n_tree_rows,
                                    int32_t n_q_heads, int32_t n_kv_heads, int32_t head_dim,
                                    const void* q, const void* k_tree, const void* v_tree,
                                    const void* k_cache, const void* v_cache, int32_t num_pages,
                                    int32_t page_size, const int32_t* page_table,
                                    int32_t max_pages_per_req, const int32_t* kv_len,
                                    const int32_t* tree_offsets, const int32_t* tree_parent,
                                    float sm_scale, void* out, float* lse, void* workspace,
                                    size_t workspace_bytes, void* stream,
                                    const as_attn_schedule* schedule);

/* ------------------------------------------------------------------------- */
/* Accept: acceptance walk + KV commit                               */
/* ------------------------------------------------------------------------- */
/*
 * Walk (R13/R14): for each request in [req_begin, req_end): v = root; repeat
 *   t* = target token at v (target_tokens[row] if target_tokens != NULL, else
 *   the argmax of target_logits[row, :] with the lowest index winning ties);
 *   move to the lowest-index child c of v with tree_tokens[c] == t*, else stop.
 *   accept_len[i] = nodes on the path including the root; accept_path[i][k] =
 *   local index of the k-th path node (-1 padded to max_path); bonus_token[i] = t*
 *   at the last accepted node.  With target_tokens holding per-node samples of
 *   the target distribution this is the lossless stochastic walk for which
 *   E[accept_len] = sum_v f(v) (Thm. 1).
 * Commit (R14/R16): rows accept_path[i][0..len) of k_tree/v_tree are copied
 *   into cache slots [kv_len[i], kv_len[i] + len) through the page table, then
 *   kv_len_out[i] = kv_len[i] + len (kv_len_out == NULL or == kv_len: in place;
 *   a separate kv_len_out keeps kv_len unchanged, e.g. for a replayed graph
 *   whose next iteration swaps the two buffers).  COMMIT covers ALL requests [0, n_req) (for KV-head
 *   sharding every rank commits every request's path for its own heads).
 * Phases: AS_ACCEPT_FUSED = walk [begin,end) + commit of the same requests;
 *   AS_ACCEPT_WALK_ONLY = walk only; AS_ACCEPT_COMMIT_ONLY = commit from
 *   accept_len/accept_path given as inputs (e.g. after an all-gather).
 *   *_RECORDS: the walk result of request i is ONE contiguous int32 row
 *   accept_path[i*(max_path+2) ..] = {len, bonus, path[max_path]} (accept_len
 *   and bonus_token unused, may be NULL) -- a request shard's rows are then a
 *   contiguous slice, all-gathered in place with no packing (multi-GPU).
 * Inputs: tree_offsets [n_req+1], tree_parent/tree_tokens [n_tree_rows];
 *   target_tokens [n_tree_rows] or NULL; target_logits [n_tree_rows, vocab] of
 *   logits_dtype or NULL (one of the two is required for the walk);
 *   k_tree/v_tree [n_tree_rows, n_kv_heads, head_dim] of kv_dtype;
 *   caches [num_pages, n_kv_heads, page_size, head_dim]; page_table
 *   [n_req, max_pages_per_req]; kv_len [n_req] (in; also the output when
 *   kv_len_out is NULL); kv_len_out [n_req] or NULL.
 * For WALK_ONLY the KV arguments may be NULL.
 * Device preconditions: AS_DEV_NAN_LOGIT, AS_DEV_PATH_TOO_LONG,
 *   AS_DEV_PAGE_OVERFLOW, AS_DEV_BAD_PAGE.
 */
typedef enum {
    AS_ACCEPT_FUSED = 0,
    AS_ACCEPT_WALK_ONLY = 1,
    AS_ACCEPT_COMMIT_ONLY = 2,
    AS_ACCEPT_WALK_RECORDS = 3,   /* walk [begin,end) into records (see below)        */
    AS_ACCEPT_COMMIT_RECORDS = 4  /* commit all requests from records                 */
} as_accept_phase;

size_t as_accept_workspace_size(int32_t n_tree_rows);
as_status as_accept_tokens(as_accept_phase phase, int32_t n_req, int32_t req_begin,
                           int32_t req_end, int32_t n_tree_rows, const int32_t* tree_offsets,
                           const int32_t* tree_parent, const int32_t* tree_tokens,
                           const int32_t* target_tokens, const void* target_logits,
                           as_dtype logits_dtype, int32_t vocab, int32_t max_path,
                           int32_t* accept_len, int32_t* accept_path, int32_t* bonus_token,
                           const void* k_tree, const void* v_tree, as_dtype kv_dtype,
                           int32_t n_kv_heads, int32_t head_dim, void* k_cache, void* v_cache,
                           int32_t num_pages, int32_t page_size, const int32_t* page_table,
                           int32_t max_pages_per_req, int32_t* kv_len, int32_t* kv_len_out,
                           void* workspace, size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------------------- */
/* Target samples for the stochastic walk: Gumbel-max (NEXT-3(a), reading R23) */
/* ------------------------------------------------------------------------- */
/*
 * out_tokens[r] = argmax_t fl32(fl32(logits[r, t] * inv_temperature) + g(r, t)),
 * lowest t on ties, for r in [0, n_rows): one sample of softmax(logits / T)
 * per tree node (T = 1 / inv_temperature), the per-node target samples R13's
 * lossless stochastic walk takes as target_tokens of as_accept_tokens
 * (E[accept_len] = sum_v f(v), Thm. 1).  g(r, t) is R23's
 * Gumbel draw: Philox4x32-10 with key (seed lo, seed hi) and counter
 * (t / 4, r, offset lo, offset hi), word t % 4 -> x; u = fl32((x >> 9)*2 + 1)
 * * 2^-24; g = -ln(-ln u) with R23's fp32 logarithm, so the
 * result is bit-identical to oracle/sampling.py.  A new (seed, offset) pair per
 * iteration gives fresh samples.
 * Inputs (device): logits [n_rows, vocab] of logits_dtype (AS_F32 or AS_BF16),
 *   finite (NaN sets AS_DEV_NAN_LOGIT; +-inf rows follow IEEE arithmetic).
 * Output (device): out_tokens [n_rows] int32.
 * Workspace: >= 256 bytes (device error word), 256-byte aligned.
 */
as_status as_sample_tokens(int32_t n_rows, int32_t vocab, const void* logits, as_dtype logits_dtype,
                           float inv_temperature, unsigned long long seed, unsigned long long offset,
                           int32_t* out_tokens, void* workspace, size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------------------- */
/* Stochastic verification: SpecInfer multi-step speculative sampling         */
/* (NEXT-3(b), reading R25)                                                   */
/* ------------------------------------------------------------------------- */
/*
 * The lossless acceptance rule for trees whose children were DRAWN from the
 * draft distribution ("tree-based verification ... prior work", Step 4;
 * R25 in DESIGN.md).  At node u of request i (row r = tree_offsets[i] + u) with
 * children c_1 < ... < c_k (local index order), draft tokens x_j =
 * tree_tokens[c_j], target row p = target_probs[r, :], draft row q =
 * draft_probs[r, :] (fp32 in, fp64 arithmetic):
 *   p~ = p; N = sum_v p~(v)
 *   for j = 1..k: accept c_j iff p~(x_j) > 0 and (r_j * N) * q(x_j) <= p~(x_j),
 *     r_j = uniforms[row of c_j]; else p~(v) <- max(0, p~(v) - N q(v)) for
 *     v != x_j, p~(x_j) <- 0, N <- sum p~ (if that is 0: keep the previous p~
 *     and stop trying);
 *   no child accepted: u emits the bonus token b = the first v (index order)
 *     with sum_{w <= v} p~(w) >= r_b * N and p~(v) > 0 (else the last v with
 *     p~(v) > 0), r_b = bonus_uniforms[r].
 * Element values follow the oracle's fp64 operation sequence exactly; the
 * masses N and the prefix sums are fp64 sums in a fixed blocked order (not the
 * oracle's exactly rounded / sequential sums), so a decision can differ from
 * the oracle's only when it lies within ~1e-13 (relative) of its threshold.
 *
 * mode AS_MSS_WALK: for each request in [req_begin, req_end) walk from the
 *   root through the accepted children, evaluating only the nodes on the path
 *   (rows of p and q are read once per VISITED node); writes the accept record
 *   records[i * (max_path + 2) ..] = {len, bonus, path[max_path] (-1 padded)}
 *   (the layout of as_accept_tokens' *_RECORDS phases: commit with
 *   AS_ACCEPT_COMMIT_RECORDS, or all-gather first for KV-head sharding) and,
 *   if emitted != NULL, emitted[r] = the token node r emitted on the path
 *   (accepted child's token or the bonus), -1 for nodes not visited.
 * mode AS_MSS_ALL_NODES: emitted[r] for every node of [req_begin, req_end)
 *   (records unused, may be NULL).  emitted is then a valid target_tokens
 *   input of as_accept_tokens (the walk moves to the lowest-index child with
 *   the emitted token: a rejected token gets p~ = 0, so it identifies the
 *   accepted child), except where a residual mass became exactly 0.
 * Layouts: tree_offsets [n_req+1], tree_parent / tree_tokens / uniforms /
 *   bonus_uniforms [n_tree_rows] (uniforms in (0, 1]); target_probs,
 *   draft_probs [n_tree_rows, vocab] f32 (rows of leaves of draft_probs are
 *   not read); records int32 [n_req, max_path + 2]; emitted int32 [n_tree_rows].
 * Supported: vocab <= 294912, trees <= AS_MAX_TREE nodes, max_path >= 1.
 * Device preconditions: AS_DEV_TREE_TOO_BIG, AS_DEV_ROWS_OVERFLOW,
 *   AS_DEV_BAD_TOKEN, AS_DEV_PATH_TOO_LONG.
 * Workspace: >= 256 bytes (device error word), 256-byte aligned.
 */
typedef enum { AS_MSS_WALK = 0, AS_MSS_ALL_NODES = 1 } as_mss_mode;

as_status as_mss_verify(as_mss_mode mode, int32_t n_req, int32_t req_begin, int32_t req_end,
                        int32_t n_tree_rows, int32_t vocab, const int32_t* tree_offsets,
                        const int32_t* tree_parent, const int32_t* tree_tokens,
                        const float* target_probs, const float* draft_probs, const float* uniforms,
                        const float* bonus_uniforms, int32_t max_path, int32_t* records,
                        int32_t* emitted, void* workspace, size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------------------- */
/* Utilities                                                                 */
/* ------------------------------------------------------------------------- */
const char* as_status_string(as_status s);
const char* as_version(void);
/* Synchronises `stream`, then copies the workspace header's sticky device error
 * {code, request} to the HOST pointers (either may be NULL).  Tests/debug only. */
as_status as_check_device_error(const void* workspace, int32_t* code, int32_t* request,
                                void* stream);
/* Zero-fills a workspace (async on stream); equivalent to cudaMemsetAsync(ws, 0, bytes). */
as_status as_reset_workspace(void* workspace, size_t workspace_bytes, void* stream);
/* Self-test of the tcgen05/TMA building blocks used by the bf16 attention:
 * D[M=128, N] = A[128, K] . B[N, K]^T with bf16 A/B (device, K-major rows) and
 * fp32 D (device), N in {64,128}, K in {64,128}; bit 0 of b_mn_major treats B
 * as [K, N] (N contiguous), as the PV product does with V; bit 1 stages A in
 * tensor memory (the A-from-TMEM form used for P); bit 2 runs the CTA-pair form
 * (a 2-CTA cluster, tcgen05.mma.cta_group::2 with M = 256: A and D have 256
 * rows, each CTA holds 128 A rows and half of B along N; MN-major needs N =
 * 128).  Debug/tests only. */
as_status as_selftest_umma(const void* a, const void* b, float* d, int32_t n, int32_t k,
                           int32_t b_mn_major, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* ADASERVE_H_ */
