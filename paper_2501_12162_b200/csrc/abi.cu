// abi.cu -- the extern "C" boundary of libadaserve.so (see include/adaserve.h).
// Host-side argument checking, workspace carving, TMA tensor-map encoding and
// kernel launches.  No exception crosses this file's functions.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <mutex>

#include "params.cuh"
#ifdef AS_DEBUG
#include "../../include/adaserve_debug.h"
#endif


using namespace as;

namespace {

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

// bf16 tensor map, SWIZZLE_128B, zero OOB fill.  dims/box innermost first;
// strides_bytes has rank-1 entries (dims 1..rank-1).
bool make_map(CUtensorMap* m, const void* base, int rank, const uint64_t* dims, const uint64_t* strides_bytes,
              const uint32_t* box) {
    auto enc = get_encode();
    if (!enc) return false;
    cuuint64_t gd[5], gs[4];
    cuuint32_t bd[5], es[5];
    for (int r = 0; r < rank; ++r) {
        gd[r] = dims[r];
        bd[r] = box[r];
        es[r] = 1;
    }
    for (int r = 0; r < rank - 1; ++r) gs[r] = strides_bytes[r];
    CUresult res = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, (cuuint32_t)rank, const_cast<void*>(base), gd, gs, bd, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return res == CUDA_SUCCESS;
}

constexpr int kMaxKLead = 1;  // must stay < the K ring depth (2)

int sm_count() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 148;
    static std::atomic<int> cache[64];  // per device (zero-initialised statics; re-entrant)
    if (dev < 64) {
        const int c = cache[dev].load(std::memory_order_relaxed);
        if (c) return c;
    }
    int n = 148;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (dev < 64) cache[dev].store(n, std::memory_order_relaxed);
    return n;
}

inline bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
inline bool al256(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 255u) == 0; }
inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

}  // namespace

extern "C" {

const char* as_version(void) { return "adaserve-b200 0.1 (sm_100a)"; }

const char* as_status_string(as_status s) {
    switch (s) {
        case AS_OK: return "ok";
        case AS_ERR_INVALID_ARG: return "invalid argument";
        case AS_ERR_BUDGET_TOO_SMALL: return "budget smaller than the number of requests";
        case AS_ERR_UNSUPPORTED: return "unsupported shape or dtype";
        case AS_ERR_WORKSPACE: return "workspace too small or misaligned";
        case AS_ERR_CUDA: return "CUDA error";
    }
    return "unknown status";
}

as_status as_check_device_error(const void* workspace, int32_t* code, int32_t* request, void* stream) {
    if (!workspace) return AS_ERR_INVALID_ARG;
    int32_t h[2] = {0, 0};
    if (cudaStreamSynchronize(S(stream)) != cudaSuccess) return AS_ERR_CUDA;
    if (cudaMemcpy(h, workspace, sizeof(h), cudaMemcpyDeviceToHost) != cudaSuccess) return AS_ERR_CUDA;
    if (code) *code = h[0];
    if (request) *request = h[1];
    return AS_OK;
}

as_status as_reset_workspace(void* workspace, size_t workspace_bytes, void* stream) {
    if (!workspace) return AS_ERR_INVALID_ARG;
    return cudaMemsetAsync(workspace, 0, workspace_bytes, S(stream)) == cudaSuccess ? AS_OK : AS_ERR_CUDA;
}

// ----------------------------------------------------------------- speculation (beam layer)
size_t as_beam_workspace_size(int32_t n_req, int32_t width, int32_t vocab) {
    if (n_req < 0 || width < 1 || width > AS_MAX_BEAM || vocab < 1) return 0;
    return beam_ws_bytes(n_req, width, vocab);
}

as_status as_beam_step(int32_t n_req, int32_t layer, int32_t width, int32_t vocab, const float* draft_probs,
                       int32_t cand_stride, int32_t* cand_parent, float* cand_prob, int32_t* cand_token,
                       void* workspace, size_t workspace_bytes, void* stream) {
    if (n_req < 0 || layer < 1 || vocab < 1) return AS_ERR_INVALID_ARG;
    if (width < 1 || width > AS_MAX_BEAM || vocab < width) return AS_ERR_UNSUPPORTED;
    const long long w_in = layer == 1 ? 1 : width;
    if (w_in * (long long)vocab >= (1ll << 32) - 1) return AS_ERR_UNSUPPORTED;
    if ((long long)cand_stride < 1 + (long long)layer * width) return AS_ERR_INVALID_ARG;
    if (n_req == 0) return AS_OK;
    if (!draft_probs || !cand_parent || !cand_prob || !cand_token) return AS_ERR_INVALID_ARG;
    if (!workspace || !al256(workspace) || workspace_bytes < beam_ws_bytes(n_req, width, vocab))
        return AS_ERR_WORKSPACE;
    return launch_beam(n_req, layer, width, vocab, draft_probs, cand_stride, cand_parent, cand_prob, cand_token,
                       workspace, S(stream)) == 0 ? AS_OK : AS_ERR_CUDA;
}

// ----------------------------------------------------------------- sample (NEXT-3a)
as_status as_sample_tokens(int32_t n_rows, int32_t vocab, const void* logits, as_dtype logits_dtype,
                           float inv_temperature, unsigned long long seed, unsigned long long offset,
                           int32_t* out_tokens, void* workspace, size_t workspace_bytes, void* stream) {
    if (n_rows < 0 || vocab < 1) return AS_ERR_INVALID_ARG;
    if (logits_dtype != AS_F32 && logits_dtype != AS_BF16) return AS_ERR_UNSUPPORTED;
    if (!(inv_temperature >= 0.f) || isinf(inv_temperature)) return AS_ERR_INVALID_ARG;
    if (n_rows == 0) return AS_OK;
    if (!logits || !out_tokens) return AS_ERR_INVALID_ARG;
    if (!workspace || !al256(workspace) || workspace_bytes < kWsHeaderBytes) return AS_ERR_WORKSPACE;
    return launch_sample(logits, logits_dtype == AS_BF16, n_rows, vocab, inv_temperature, seed, offset, out_tokens,
                         workspace, S(stream)) == 0 ? AS_OK : AS_ERR_CUDA;
}

// ----------------------------------------------------------------- MSS (NEXT-3(b))
as_status as_mss_verify(as_mss_mode mode, int32_t n_req, int32_t req_begin, int32_t req_end, int32_t n_tree_rows,
                        int32_t vocab, const int32_t* tree_offsets, const int32_t* tree_parent,
                        const int32_t* tree_tokens, const float* target_probs, const float* draft_probs,
                        const float* uniforms, const float* bonus_uniforms, int32_t max_path, int32_t* records,
                        int32_t* emitted, void* workspace, size_t workspace_bytes, void* stream) {
    if (mode != AS_MSS_WALK && mode != AS_MSS_ALL_NODES) return AS_ERR_INVALID_ARG;
    if (n_req < 0 || req_begin < 0 || req_end < req_begin || req_end > n_req || n_tree_rows < 0 || vocab < 1)
        return AS_ERR_INVALID_ARG;
    if (mss_smem_bytes(vocab) == 0) return AS_ERR_UNSUPPORTED;
    if (req_end == req_begin) return AS_OK;
    if (!tree_offsets || !tree_parent || !tree_tokens || !target_probs || !draft_probs || !uniforms ||
        !bonus_uniforms)
        return AS_ERR_INVALID_ARG;
    if (mode == AS_MSS_WALK && (max_path < 1 || (!records && !emitted))) return AS_ERR_INVALID_ARG;
    if (mode == AS_MSS_ALL_NODES && !emitted) return AS_ERR_INVALID_ARG;
    if (!workspace || !al256(workspace) || workspace_bytes < kWsHeaderBytes) return AS_ERR_WORKSPACE;
    return launch_mss(req_begin, req_end, n_tree_rows, vocab, tree_offsets, tree_parent, tree_tokens, target_probs,
                      draft_probs, uniforms, bonus_uniforms, emitted, mode == AS_MSS_WALK ? records : nullptr,
                      max_path, mode == AS_MSS_WALK ? 1 : 0, workspace, workspace_bytes, S(stream)) == 0 ? AS_OK
                                                                                                    : AS_ERR_CUDA;
}

// ----------------------------------------------------------------- select
size_t as_select_workspace_size(int32_t n_req, int32_t n_cand_total) {
    if (n_req < 0 || n_cand_total < 0) return 0;
    return select_ws_bytes(n_req, n_cand_total);
}

as_status as_select_trees(int32_t n_req, int32_t n_cand_total, const int32_t* cand_offsets, const int32_t* cand_parent,
                          const float* cand_prob, const int32_t* cand_token, const double* slo_deficit,
                          int32_t depth_d, int32_t n_max, int32_t budget, int32_t* tree_offsets, int32_t* tree_parent,
                          int32_t* tree_src, int32_t* tree_depth, int32_t* tree_token, int32_t* slo_count,
                          void* workspace, size_t workspace_bytes, void* stream) {
    if (n_req < 0 || n_cand_total < n_req || depth_d < 0 || n_max < 0 || !tree_offsets) return AS_ERR_INVALID_ARG;
    if (budget < n_req) return AS_ERR_BUDGET_TOO_SMALL;
    if (n_req > 4096) return AS_ERR_UNSUPPORTED;
    if (n_req == 0) {
        return cudaMemsetAsync(tree_offsets, 0, sizeof(int32_t), S(stream)) == cudaSuccess ? AS_OK : AS_ERR_CUDA;
    }
    if (!cand_offsets || !cand_parent || !cand_prob || !slo_deficit || !tree_parent || !tree_src)
        return AS_ERR_INVALID_ARG;
    if (tree_token && !cand_token) return AS_ERR_INVALID_ARG;
    if (!workspace || !al256(workspace) || workspace_bytes < select_ws_bytes(n_req, n_cand_total))
        return AS_ERR_WORKSPACE;
    int rc = launch_select(n_req, n_cand_total, cand_offsets, cand_parent, cand_prob, cand_token, slo_deficit, depth_d,
                           n_max, budget, tree_offsets, tree_parent, tree_src, tree_depth, tree_token, slo_count,
                           workspace, S(stream));
    return rc == 0 ? AS_OK : AS_ERR_CUDA;
}

as_status as_select_topm(int32_t n_req, int32_t n_cand_total, const int32_t* cand_offsets, const int32_t* cand_parent,
                         const float* cand_prob, const int32_t* cand_token, int32_t m_base, int32_t m_extra,
                         int32_t* tree_offsets, int32_t* tree_parent, int32_t* tree_src, int32_t* tree_depth,
                         int32_t* tree_token, int32_t* kept, void* workspace, size_t workspace_bytes, void* stream) {
    if (n_req < 0 || n_cand_total < n_req || m_base < 0 || m_extra < 0 || m_extra > n_req || !tree_offsets)
        return AS_ERR_INVALID_ARG;
    if (n_req > 4096) return AS_ERR_UNSUPPORTED;
    if (n_req == 0) {
        return cudaMemsetAsync(tree_offsets, 0, sizeof(int32_t), S(stream)) == cudaSuccess ? AS_OK : AS_ERR_CUDA;
    }
    if (!cand_offsets || !cand_parent || !cand_prob || !tree_parent || !tree_src) return AS_ERR_INVALID_ARG;
    if (tree_token && !cand_token) return AS_ERR_INVALID_ARG;
    if (!workspace || !al256(workspace) || workspace_bytes < select_ws_bytes(n_req, n_cand_total))
        return AS_ERR_WORKSPACE;
    int rc = launch_select(n_req, n_cand_total, cand_offsets, cand_parent, cand_prob, cand_token, nullptr, 0, m_base,
                           0, tree_offsets, tree_parent, tree_src, tree_depth, tree_token, kept, workspace, S(stream),
                           1, m_extra);
    return rc == 0 ? AS_OK : AS_ERR_CUDA;
}

// ----------------------------------------------------------------- attention
size_t as_attn_workspace_size(as_dtype dtype, int32_t n_req, int32_t n_tree_rows, int32_t n_q_heads,
                              int32_t head_dim, int32_t max_kv_len) {
    (void)dtype; (void)n_tree_rows; (void)max_kv_len;
    if (n_req < 0 || n_q_heads < 0 || head_dim <= 0) return 0;
    // header + debug trace + split-KV counters (two per unit: n_units = n_q * n_req
    // for every GQA ratio) + 2 partial-state slots per resident CTA
    // mt_max * n_kv = ceil(AS_MAX_TREE * G / 128) * n_kv = n_q * AS_MAX_TREE / 128 (G >= 1)
    const size_t units = (size_t)n_q_heads * (size_t)n_req * (AS_MAX_TREE / 128);
    const size_t slot = ((size_t)128 * head_dim + 256) * 4;
    return kWsHeaderBytes + kAttnTraceBytes + align_up(2 * units * 4, 256) +
           2 * (size_t)sm_count() * (size_t)tc_ctas_per_sm() * slot;
}

as_status as_tree_verify_attn(as_dtype dtype, int32_t n_req, int32_t n_tree_rows, int32_t n_q_heads,
                              int32_t n_kv_heads, int32_t head_dim, const void* q, const void* k_tree,
                              const void* v_tree, const void* k_cache, const void* v_cache, int32_t num_pages,
                              int32_t page_size, const int32_t* page_table, int32_t max_pages_per_req,
                              const int32_t* kv_len, const int32_t* tree_offsets, const int32_t* tree_parent,
                              float sm_scale, void* out, float* lse, void* workspace, size_t workspace_bytes,
                              void* stream) {
    return as_tree_verify_attn_sched(dtype, n_req, n_tree_rows, n_q_heads, n_kv_heads, head_dim, q, k_tree, v_tree,
                                     k_cache, v_cache, num_pages, page_size, page_table, max_pages_per_req, kv_len,
                                     tree_offsets, tree_parent, sm_scale, out, lse, workspace, workspace_bytes, stream,
                                     nullptr);
}

as_status as_tree_verify_attn_sched(as_dtype dtype, int32_t n_req, int32_t n_tree_rows, int32_t n_q_heads,
                                    int32_t n_kv_heads, int32_t head_dim, const void* q, const void* k_tree,
                                    const void* v_tree, const void* k_cache, const void* v_cache, int32_t num_pages,
                                    int32_t page_size, const int32_t* page_table, int32_t max_pages_per_req,
                                    const int32_t* kv_len, const int32_t* tree_offsets, const int32_t* tree_parent,
                                    float sm_scale, void* out, float* lse, void* workspace, size_t workspace_bytes,
                                    void* stream, const as_attn_schedule* schedule) {
    if (schedule && (schedule->q_tiles_per_cta < 0 || schedule->q_tiles_per_cta > 2 ||
                     !(schedule->cluster_ctas == 0 || schedule->cluster_ctas == 1 || schedule->cluster_ctas == 2 ||
                       schedule->cluster_ctas == 4) ||
                     schedule->split < -1 || schedule->split > 1 || schedule->cta_pair < -1 || schedule->cta_pair > 1))
        return AS_ERR_INVALID_ARG;
    if (n_req < 0 || n_tree_rows < 0 || n_q_heads <= 0 || n_kv_heads <= 0 || num_pages < 0 || max_pages_per_req < 0)
        return AS_ERR_INVALID_ARG;
    if (n_q_heads % n_kv_heads != 0) return AS_ERR_UNSUPPORTED;
    if (head_dim != 64 && head_dim != 128) return AS_ERR_UNSUPPORTED;
    if (page_size != 16 && page_size != 32 && page_size != 64 && page_size != 128) return AS_ERR_UNSUPPORTED;
    if (dtype != AS_F32 && dtype != AS_BF16) return AS_ERR_UNSUPPORTED;
    if (!workspace || !al256(workspace) || workspace_bytes < kWsHeaderBytes) return AS_ERR_WORKSPACE;
    if (n_req == 0 || n_tree_rows == 0) return AS_OK;
    if (!q || !k_tree || !v_tree || !out || !kv_len || !tree_offsets || !tree_parent) return AS_ERR_INVALID_ARG;
    if (num_pages > 0 && max_pages_per_req > 0 && (!k_cache || !v_cache || !page_table)) return AS_ERR_INVALID_ARG;
    const int G = n_q_heads / n_kv_heads;
    if (!al16(q) || !al16(k_tree) || !al16(v_tree) || !al16(out) || (k_cache && !al16(k_cache)) ||
        (v_cache && !al16(v_cache)))
        return AS_ERR_INVALID_ARG;  // 16-byte vector / TMA access (both paths)
    if (dtype == AS_F32) {
        SimtParams p;
        p.n_req = n_req; p.n_tree_rows = n_tree_rows; p.n_q = n_q_heads; p.n_kv = n_kv_heads; p.G = G;
        p.q = (const float*)q; p.k_tree = (const float*)k_tree; p.v_tree = (const float*)v_tree;
        p.k_cache = (const float*)k_cache; p.v_cache = (const float*)v_cache;
        p.num_pages = num_pages; p.page_size = page_size; p.page_table = page_table; p.max_pages = max_pages_per_req;
        p.kv_len = kv_len; p.tree_offsets = tree_offsets; p.tree_parent = tree_parent; p.sm_scale = sm_scale;
        p.out = (float*)out; p.lse = lse; p.ws = workspace;
        return launch_attn_simt(p, head_dim, S(stream)) == 0 ? AS_OK : AS_ERR_CUDA;
    }
    // bf16 tcgen05 path
    if ((G & (G - 1)) != 0 || G > 16) return AS_ERR_UNSUPPORTED;
    const uint64_t D = (uint64_t)head_dim;
    CUtensorMap maps[5];
    const uint64_t NCH = D / 64;
    // Every map carries the 64-element d-chunk index as its own dimension so one
    // TMA box fills all chunks of a tile ([chunk][row][64] in smem, SW128): half
    // the TMA issues of per-chunk boxes (the producer's issue rate bounded the
    // per-SM streaming rate).
    {
        uint64_t dims[4] = {64, (uint64_t)n_q_heads, (uint64_t)n_tree_rows, NCH};
        uint64_t str[3] = {D * 2, (uint64_t)n_q_heads * D * 2, 128};
        uint32_t box[4] = {64, (uint32_t)G, (uint32_t)(128 / G), (uint32_t)NCH};
        if (!make_map(&maps[0], q, 4, dims, str, box)) return AS_ERR_CUDA;
    }
    const int box_rows = page_size < 64 ? page_size : 64;
    const int kv_split_d = page_size >= 64 ? 1 : 0;  // one box covers a whole 64-key tile
    // CTA pair (cta_group::2): trees spanning >= 2 q-tiles per (request, kv head),
    // head_dim 128, whole-tile boxes; each CTA loads half of every K/V tile
    const long long qt_req = n_req > 0 ? ((long long)G * (n_tree_rows / n_req) + 127) / 128 : 0;
    int pair = 0;
    if (schedule && schedule->cta_pair == 1) pair = 1;
    if (pair && !(head_dim == 128 && kv_split_d && qt_req >= 2)) return AS_ERR_UNSUPPORTED;
    {
        const uint64_t np = (uint64_t)(num_pages > 0 ? num_pages : 1);
        const void* kc = k_cache ? k_cache : k_tree;  // never dereferenced when there are no pages
        const void* vc = v_cache ? v_cache : v_tree;
        if (kv_split_d) {
            uint64_t dims[5] = {64, (uint64_t)page_size, NCH, (uint64_t)n_kv_heads, np};
            uint64_t str[4] = {D * 2, 128, (uint64_t)page_size * D * 2, (uint64_t)n_kv_heads * page_size * D * 2};
            uint32_t box[5] = {64, (uint32_t)box_rows, (uint32_t)NCH, 1, 1};
            uint32_t kbox[5] = {64, 32, (uint32_t)NCH, 1, 1};  // pair: 32 of the tile's keys
            uint32_t vbox[5] = {64, 64, 1, 1, 1};              // pair: one d-chunk of all 64 keys
            if (!make_map(&maps[1], kc, 5, dims, str, pair ? kbox : box)) return AS_ERR_CUDA;
            if (!make_map(&maps[2], vc, 5, dims, str, pair ? vbox : box)) return AS_ERR_CUDA;
        } else {
            uint64_t dims[4] = {D, (uint64_t)page_size, (uint64_t)n_kv_heads, np};
            uint64_t str[3] = {D * 2, (uint64_t)page_size * D * 2, (uint64_t)n_kv_heads * page_size * D * 2};
            uint32_t box[4] = {64, (uint32_t)box_rows, 1, 1};
            if (!make_map(&maps[1], kc, 4, dims, str, box)) return AS_ERR_CUDA;
            if (!make_map(&maps[2], vc, 4, dims, str, box)) return AS_ERR_CUDA;
        }
    }
    {
        uint64_t dims[4] = {64, (uint64_t)n_tree_rows, NCH, (uint64_t)n_kv_heads};
        uint64_t str[3] = {(uint64_t)n_kv_heads * D * 2, 128, D * 2};
        uint32_t box[4] = {64, 64, (uint32_t)NCH, 1};
        uint32_t kbox[4] = {64, 32, (uint32_t)NCH, 1};
        uint32_t vbox[4] = {64, 64, 1, 1};
        if (!make_map(&maps[3], k_tree, 4, dims, str, pair ? kbox : box)) return AS_ERR_CUDA;
        if (!make_map(&maps[4], v_tree, 4, dims, str, pair ? vbox : box)) return AS_ERR_CUDA;
    }
    TcParams p;
    p.n_req = n_req; p.n_tree_rows = n_tree_rows; p.n_q = n_q_heads; p.n_kv = n_kv_heads; p.G = G;
    p.page_size = page_size; p.box_rows = box_rows; p.kv_split_d = kv_split_d; p.max_pages = max_pages_per_req; p.num_pages = num_pages;
    p.page_table = page_table; p.kv_len = kv_len; p.tree_offsets = tree_offsets; p.tree_parent = tree_parent;
    p.scale_log2 = sm_scale * 1.4426950408889634f;
    p.out = (__nv_bfloat16*)out; p.lse = lse; p.ws = workspace;
    const int mt_max = (AS_MAX_TREE * G + 127) / 128;
    p.n_units = mt_max * n_req * n_kv_heads;
    p.mt_max = mt_max;
    // CTA shape, from the trees' q-tiles per (request, kv head) -- n_tree_rows / n_req
    // is the caller's row allocation per request: one q-tile -> one-q-tile CTAs, two
    // per SM; more -> the q-tiles of a head share every K/V tile fetch (NQ = 2: two
    // q-tiles in one CTA; cs: a cluster of one-q-tile CTAs with multicast).
    // as_tree_verify_attn_sched overrides the choice (A/B; results identical).
    {
        const long long rows_per_req = n_req > 0 ? (long long)n_tree_rows / n_req : 0;
        const long long qt = (G * rows_per_req + 127) / 128;
        // 1 q-tile: one-q-tile CTAs, 2 per SM; 2: both q-tiles in one CTA; 3-4 (c4: 4):
        // a 2-CTA cluster of NQ = 2 CTAs, each K/V tile fetched once for all four q-tiles
        // (multicast) -- measured 3-6 % faster than NQ = 2 alone and no re-read of the
        // head's KV
        p.nq = qt > 1 ? 2 : 1;
        p.cs = qt >= 3 ? 2 : 1;
        if (schedule && schedule->q_tiles_per_cta > 0) {
            p.nq = schedule->q_tiles_per_cta;
            p.cs = 1;
        }
        if (schedule && schedule->cluster_ctas == 1) p.cs = 1;
        if (schedule && schedule->cluster_ctas > 1) {
            p.cs = schedule->cluster_ctas;
            if (!(schedule->q_tiles_per_cta == 2 && p.cs == 2)) p.nq = 1;  // (2, 2): two NQ=2 CTAs
        }
        p.pair = pair;
        if (pair) {  // q-tiles per CTA: 2 when the head spans > 2 q-tiles, else 1 (the pair covers 2)
            p.nq = (schedule && schedule->q_tiles_per_cta > 0) ? schedule->q_tiles_per_cta : (qt > 2 ? 2 : 1);
            p.cs = 2;
        }
    }
    {
        const int nsm = sm_count();
        const size_t slot = ((size_t)128 * head_dim + 256) * 4;
        const size_t cnt_bytes = align_up((size_t)p.n_units * 8, 256);  // tile counters + merge counters
        const size_t need = kWsHeaderBytes + kAttnTraceBytes + cnt_bytes + 2 * (size_t)nsm * tc_ctas_per_sm() * slot;
        unsigned char* base = reinterpret_cast<unsigned char*>(workspace) + kWsHeaderBytes + kAttnTraceBytes;
        // split-KV / tail pieces need the counters and partial slots in the workspace
        p.stream_k = (workspace_bytes >= need && !(schedule && schedule->split == 0)) ? 1 : 0;
        p.cnt = reinterpret_cast<int*>(base);
        p.cnt2 = p.cnt + p.n_units;
        p.partial = reinterpret_cast<float*>(base + cnt_bytes);
        p.slot_floats = 128 * head_dim + 256;
    }
    p.req_base = 0;
    p.tail_mode = 1;
    p.debug_mode = 0;
    p.evict_first = 1;
    p.k_lead = 1;
    p.trace = nullptr;
    p.trace_cap = 0;
#ifdef AS_DEBUG
    // Experiment switches, compiled only into the debug build (AS_DEBUG=1 build.py):
    // the product library reads no environment variable on this path.
    if (const char* dbg = getenv("AS_ATTN_DEBUG_MODE")) p.debug_mode = atoi(dbg);  // timing only (wrong outputs)
    if (const char* tm = getenv("AS_ATTN_TAIL")) p.tail_mode = atoi(tm);           // schedule A/B
    if (const char* ef = getenv("AS_ATTN_EVICT_FIRST")) p.evict_first = atoi(ef);  // L2 evict-first hint A/B
    if (const char* kl = getenv("AS_ATTN_KLEAD")) p.k_lead = atoi(kl);             // K stream lead over V
    if (p.k_lead < 0) p.k_lead = 0;
    if (p.k_lead > kMaxKLead) p.k_lead = kMaxKLead;
    const char* tr = getenv("AS_ATTN_TRACE");  // CTA-0 pipeline timestamps into the workspace
    if (tr && atoi(tr) && workspace_bytes >= kWsHeaderBytes + kAttnTraceBytes) {
        p.trace = reinterpret_cast<unsigned long long*>(reinterpret_cast<unsigned char*>(workspace) + kWsHeaderBytes);
        p.trace_cap = (int)(kAttnTraceBytes / 64) - 512;  // last 512 records: per-CTA timeline
    }
#endif
    return launch_attn_tc(maps, p, head_dim, sm_count(), S(stream)) == 0 ? AS_OK : AS_ERR_CUDA;
}

// ----------------------------------------------------------------- accept
size_t as_accept_workspace_size(int32_t n_tree_rows) {
    return kWsHeaderBytes + align_up((size_t)(n_tree_rows > 0 ? n_tree_rows : 1) * 4, 256);
}

as_status as_accept_tokens(as_accept_phase phase, int32_t n_req, int32_t req_begin, int32_t req_end,
                           int32_t n_tree_rows, const int32_t* tree_offsets, const int32_t* tree_parent,
                           const int32_t* tree_tokens, const int32_t* target_tokens, const void* target_logits,
                           as_dtype logits_dtype, int32_t vocab, int32_t max_path, int32_t* accept_len,
                           int32_t* accept_path, int32_t* bonus_token, const void* k_tree, const void* v_tree,
                           as_dtype kv_dtype, int32_t n_kv_heads, int32_t head_dim, void* k_cache, void* v_cache,
                           int32_t num_pages, int32_t page_size, const int32_t* page_table, int32_t max_pages_per_req,
                           int32_t* kv_len, int32_t* kv_len_out, void* workspace, size_t workspace_bytes,
                           void* stream) {
    if (phase != AS_ACCEPT_FUSED && phase != AS_ACCEPT_WALK_ONLY && phase != AS_ACCEPT_COMMIT_ONLY &&
        phase != AS_ACCEPT_WALK_RECORDS && phase != AS_ACCEPT_COMMIT_RECORDS)
        return AS_ERR_INVALID_ARG;
    const bool records = phase == AS_ACCEPT_WALK_RECORDS || phase == AS_ACCEPT_COMMIT_RECORDS;
    if (n_req < 0 || req_begin < 0 || req_end < req_begin || req_end > n_req || n_tree_rows < 0) return AS_ERR_INVALID_ARG;
    if (max_path < 1 || max_path > 64) return AS_ERR_UNSUPPORTED;
    if (!workspace || !al256(workspace) || workspace_bytes < as_accept_workspace_size(n_tree_rows))
        return AS_ERR_WORKSPACE;
    if (!tree_offsets || !accept_path || (!records && !accept_len)) return AS_ERR_INVALID_ARG;
    const bool walk = phase == AS_ACCEPT_FUSED || phase == AS_ACCEPT_WALK_ONLY || phase == AS_ACCEPT_WALK_RECORDS;
    const bool commit = phase == AS_ACCEPT_FUSED || phase == AS_ACCEPT_COMMIT_ONLY || phase == AS_ACCEPT_COMMIT_RECORDS;
    if (walk) {
        if (!tree_parent || !tree_tokens || (!records && !bonus_token)) return AS_ERR_INVALID_ARG;
        if (!target_tokens && !target_logits) return AS_ERR_INVALID_ARG;
        if (!target_tokens && (vocab <= 0 || (logits_dtype != AS_F32 && logits_dtype != AS_BF16)))
            return AS_ERR_INVALID_ARG;
    }
    if (commit) {
        if (!k_tree || !v_tree || !k_cache || !v_cache || !page_table || !kv_len) return AS_ERR_INVALID_ARG;
        if (kv_dtype != AS_F32 && kv_dtype != AS_BF16) return AS_ERR_UNSUPPORTED;
        if (head_dim <= 0 || n_kv_heads <= 0 || page_size <= 0) return AS_ERR_INVALID_ARG;
        const int eb = kv_dtype == AS_BF16 ? 2 : 4;
        if ((head_dim * eb) % 16 != 0) return AS_ERR_UNSUPPORTED;
        if (!al16(k_tree) || !al16(v_tree) || !al16(k_cache) || !al16(v_cache)) return AS_ERR_INVALID_ARG;
    }
    AcceptParams p;
    p.n_req = n_req; p.req_begin = req_begin; p.req_end = req_end; p.n_tree_rows = n_tree_rows;
    p.tree_offsets = tree_offsets; p.tree_parent = tree_parent; p.tree_tokens = tree_tokens;
    p.target_tokens = target_tokens; p.max_path = max_path;
    p.accept_len = accept_len; p.accept_path = accept_path; p.bonus_token = bonus_token;
    p.k_tree = (const unsigned char*)k_tree; p.v_tree = (const unsigned char*)v_tree;
    p.elem_bytes = kv_dtype == AS_BF16 ? 2 : 4; p.n_kv = n_kv_heads; p.head_dim = head_dim;
    p.k_cache = (unsigned char*)k_cache; p.v_cache = (unsigned char*)v_cache;
    p.num_pages = num_pages; p.page_size = page_size; p.page_table = page_table; p.max_pages = max_pages_per_req;
    p.kv_len = kv_len; p.kv_len_out = kv_len_out ? kv_len_out : kv_len; p.ws = workspace;
    p.do_walk = walk ? 1 : 0;
    p.do_commit = commit ? 1 : 0;
    p.records = records ? 1 : 0;
    int32_t* argmax_buf = reinterpret_cast<int32_t*>(reinterpret_cast<unsigned char*>(workspace) + kWsHeaderBytes);
    return launch_accept(p, target_logits, logits_dtype == AS_BF16, vocab, argmax_buf, S(stream)) == 0 ? AS_OK
                                                                                                      : AS_ERR_CUDA;
}

#ifdef AS_DEBUG
// ----------------------------------------------------------------- debug
as_status as_debug_stream_bw(const void* src, const int32_t* order, int32_t n_chunks, int32_t chunk_bytes,
                             int32_t stages, int32_t mode, unsigned long long* sink, int32_t grid, void* stream) {
    if (!src || !order || !sink || n_chunks <= 0 || chunk_bytes <= 0 || chunk_bytes % 16 || stages <= 0 || grid <= 0)
        return AS_ERR_INVALID_ARG;
    if ((size_t)stages * chunk_bytes > 200 * 1024) return AS_ERR_UNSUPPORTED;
    CUtensorMap tm;
    memset(&tm, 0, sizeof(tm));
    if (mode >= 3) {  // [rows][128] bf16 view, box {64, rows_per_chunk, 2}, SW128
        const uint64_t rows = (uint64_t)n_chunks * (chunk_bytes / 256);
        uint64_t dims[3] = {64, rows, 2};
        uint64_t str[2] = {256, 128};
        uint32_t box[3] = {64, (uint32_t)(chunk_bytes / 256), 2};
        if (chunk_bytes / 256 > 256 || !make_map(&tm, src, 3, dims, str, box)) return AS_ERR_UNSUPPORTED;
    }
    return launch_stream_bw(src, order, n_chunks, chunk_bytes, stages, mode, sink, grid, &tm, S(stream)) == 0
               ? AS_OK
               : AS_ERR_CUDA;
}

#endif  // AS_DEBUG

// ----------------------------------------------------------------- selftest
as_status as_selftest_umma(const void* a, const void* b, float* d, int32_t n, int32_t k, int32_t b_mn_major,
                           void* stream) {
    if (!a || !b || !d) return AS_ERR_INVALID_ARG;
    if ((n != 64 && n != 128) || (k != 64 && k != 128)) return AS_ERR_UNSUPPORTED;
    const bool pair = (b_mn_major & 4) != 0;  // bit 2: CTA pair, M = 256 (cta_group::2)
    if (pair && (b_mn_major & 1) && n != 128) return AS_ERR_UNSUPPORTED;  // MN-major halves are 64-wide chunks
    const int m = pair ? 256 : 128;
    CUtensorMap ma, mb;
    {
        uint64_t dims[2] = {(uint64_t)k, (uint64_t)m};
        uint64_t str[1] = {(uint64_t)k * 2};
        uint32_t box[2] = {64, 128};
        if (!make_map(&ma, a, 2, dims, str, box)) return AS_ERR_CUDA;
    }
    if (!(b_mn_major & 1)) {  // bit 0: B MN-major; bit 1: A staged in TMEM
        uint64_t dims[2] = {(uint64_t)k, (uint64_t)n};
        uint64_t str[1] = {(uint64_t)k * 2};
        uint32_t box[2] = {64, (uint32_t)(pair ? n / 2 : n)};
        if (!make_map(&mb, b, 2, dims, str, box)) return AS_ERR_CUDA;
    } else {
        uint64_t dims[2] = {(uint64_t)n, (uint64_t)k};
        uint64_t str[1] = {(uint64_t)n * 2};
        uint32_t box[2] = {64, (uint32_t)k};
        if (!make_map(&mb, b, 2, dims, str, box)) return AS_ERR_CUDA;
    }
    const int rc = pair ? launch_umma2_selftest(&ma, &mb, d, n, k, b_mn_major & 1, a, (b_mn_major & 2) ? 1 : 0, S(stream))
                        : launch_umma_selftest(&ma, &mb, d, n, k, (b_mn_major & 1) ? 1 : 0, a, (b_mn_major & 2) ? 1 : 0,
                                               S(stream));
    return rc == 0 ? AS_OK : AS_ERR_CUDA;
}

}  // extern "C"
