// params.cuh -- launch parameter blocks shared by abi.cu and the kernels.
#pragma once
#include <cuda.h>
#include "common.cuh"

namespace as {

struct AcceptParams {
    int n_req, req_begin, req_end, n_tree_rows;
    const int32_t* tree_offsets;
    const int32_t* tree_parent;
    const int32_t* tree_tokens;
    const int32_t* target_tokens;
    int max_path;
    int32_t* accept_len;
    int32_t* accept_path;
    int32_t* bonus_token;
    const unsigned char* k_tree;
    const unsigned char* v_tree;
    int elem_bytes, n_kv, head_dim;
    unsigned char* k_cache;
    unsigned char* v_cache;
    int num_pages, page_size;
    const int32_t* page_table;
    int max_pages;
    const int32_t* kv_len;
    int32_t* kv_len_out;  // == kv_len for in-place updates
    void* ws;
    int do_walk, do_commit;
    int records;  // 1: accept_path is int32 [rows][2 + max_path] records {len, bonus, path}
};

struct SimtParams {
    int n_req, n_tree_rows, n_q, n_kv, G;
    const float* q;
    const float* k_tree;
    const float* v_tree;
    const float* k_cache;
    const float* v_cache;
    int num_pages, page_size;
    const int32_t* page_table;
    int max_pages;
    const int32_t* kv_len;
    const int32_t* tree_offsets;
    const int32_t* tree_parent;
    float sm_scale;
    float* out;
    float* lse;
    void* ws;
};

struct TcParams {
    int n_req, n_tree_rows, n_q, n_kv, G;
    int page_size, box_rows, max_pages, num_pages;
    int kv_split_d;  // 1: cache maps are 5-D (d-chunk dim), one box per 64-key tile
    const int32_t* page_table;
    const int32_t* kv_len;
    const int32_t* tree_offsets;
    const int32_t* tree_parent;
    float scale_log2;
    __nv_bfloat16* out;
    float* lse;
    void* ws;
    int n_units;
    int req_base;         // caller's index of request 0 of this launch (device-error reports)
    int nq;               // host in: CTA shape (1 or 2 q-tiles per CTA); kernel: q-tiles per unit (nq * cs)
    int cs;               // thread-block cluster size (1, 2, 4; one-q-tile CTAs sharing K/V by multicast)
    int pair;             // 1: CTA pairs (cs = 2, tcgen05.mma.cta_group::2, half K/V tiles per CTA)
    int mt_max;           // q-tiles per (request, kv head) upper bound (unit id stride)
    int stream_k;         // 1: split-KV allowed (needs cnt/cnt2/partial in the workspace), 0: whole units only
    int tail_mode;        // 1: tail stream-K for a partial last wave; 0: balanced whole-unit waves; 2: tail even when balanced waves fit (debug A/B)
    int* cnt;             // [n_units] tiles completed per split unit (zeroed, self-resetting)
    int* cnt2;            // [n_units] pieces that finished merging (zeroed, self-resetting)
    float* partial;       // [2 * gridDim.x][slot_floats] partial (O, m, l) of split units
    int slot_floats;      // 128 * D + 256
    int evict_first;
    int k_lead;           // tiles by which the K stream leads the V stream in the producer
    int debug_mode;  // 0 = normal; 1 = skip softmax math; 2 = also skip MMAs (timing experiments only)
    unsigned long long* trace;  // CTA-0 pipeline timestamps [trace_cap][8] (clock64) or NULL
    int trace_cap;
};

size_t select_ws_bytes(int n_req, int n_cand_total);
int launch_select(int, int, const int32_t*, const int32_t*, const float*, const int32_t*, const double*, int, int,
                  int, int32_t*, int32_t*, int32_t*, int32_t*, int32_t*, int32_t*, void*, cudaStream_t,
                  int topm = 0, int n_max_extra = 0);
int launch_accept(const AcceptParams& p, const void* target_logits, int logits_bf16, int vocab, int32_t* argmax_buf,
                  cudaStream_t stream);
int launch_attn_simt(const SimtParams& p, int head_dim, cudaStream_t stream);
int launch_sample(const void* logits, int logits_bf16, int n_rows, int vocab, float inv_t, unsigned long long seed,
                  unsigned long long offset, int32_t* out, void* ws, cudaStream_t stream);
size_t mss_smem_bytes(int vocab);
int launch_mss(int req_begin, int req_end, int n_tree_rows, int vocab, const int32_t* tree_offsets,
               const int32_t* tree_parent, const int32_t* tree_tokens, const float* p_rows, const float* q_rows,
               const float* uni, const float* bonus_uni, int32_t* emitted, int32_t* records, int max_path, int walk,
               void* ws, size_t ws_bytes, cudaStream_t stream);
int launch_attn_tc(const CUtensorMap* maps, const TcParams& p, int head_dim, int n_sms, cudaStream_t stream);
int tc_ctas_per_sm();
size_t beam_ws_bytes(int n_req, int width, int vocab);
int launch_beam(int n_req, int layer, int width, int vocab, const float* probs, int stride, int32_t* cand_parent,
                float* cand_prob, int32_t* cand_token, void* ws, cudaStream_t stream);
#ifdef AS_DEBUG
int launch_stream_bw(const void* src, const int* order, int n_chunks, int chunk_bytes, int stages, int mode,
                     unsigned long long* sink, int grid, const CUtensorMap* tmap, cudaStream_t stream);
#endif
int launch_umma2_selftest(const CUtensorMap* ma, const CUtensorMap* mb, float* d, int N, int K, int b_mn,
                          const void* a_g, int a_tmem, cudaStream_t stream);
int launch_umma_selftest(const CUtensorMap* ma, const CUtensorMap* mb, float* d, int N, int K, int b_mn,
                         const void* a_g, int a_tmem, cudaStream_t stream);

}  // namespace as
