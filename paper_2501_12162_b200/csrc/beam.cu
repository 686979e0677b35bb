// beam.cu -- NEXT-1: as_beam_step, one layer of Step 1 speculation.
//
// For every request, the kept nodes of the previous layer (w_in = 1 at layer 1,
// else w) each get the draft model's distribution over the vocabulary; every
// expansion (parent k, token t) has the approximated path probability
// f-hat = fl32(f-hat(parent k) * M_q(t | X, Path(k))), and the layer
// keeps the w largest by (f-hat desc, parent asc, token asc) (R8).  The w x |V|
// scan is HBM-bound (|V| = 128 256: 513 KB of fp32 per row):
//
//   beam_scan_kernel   one CTA per row: 16-byte streaming loads; each warp keeps
//                      a shared-memory buffer of the 64-bit keys (f-hat bits
//                      << 32 | ~(k*|V| + t)) -- the key order IS the tie order
//                      and keys are unique -- that beat its threshold (the w-th
//                      best so far), compacted to its top w when full; a
//                      max-of-float4 prefilter on the raw probability keeps the
//                      common path at a few instructions per element; the 8
//                      warps' top-w merged into the row's slot.
//   beam_merge_kernel  one warp per request: top-w of its rows' lists; writes
//                      the new layer's nodes into the candidate forest.
#include "params.cuh"

namespace as {

constexpr int kBeamW = 16;                                             // list capacity (lanes) >= width

__device__ __forceinline__ uint64_t beam_key(float f, uint32_t idx) {
    const uint32_t fb = (f > 0.f) ? __float_as_uint(f) : 0u;  // NaN / negative / zero -> 0
    return ((uint64_t)fb << 32) | (uint64_t)(0xFFFFFFFFu - idx);
}

// A warp-distributed top-w list: lane j < w holds the j-th largest key (desc),
// the other lanes hold 0.  thr = the w-th largest (0 while the list fills up).
struct WarpList {
    uint64_t v;
    uint64_t thr;   // the list's w-th key
    uint64_t filt;  // >= thr: also a lower bound shared by the CTA's other warps (their w-th keys)
    float thr_f;    // f-hat of filt (prefilter: a key can beat filt only if f >= thr_f)
};

__device__ __forceinline__ void wl_init(WarpList& L) {
    L.v = 0ull;
    L.thr = 0ull;
    L.filt = 0ull;
    L.thr_f = 0.f;
}

// Raise the filter to a bound published by another warp of the same CTA: a key
// below some warp's w-th key cannot be among the CTA's top w.
__device__ __forceinline__ void wl_raise(WarpList& L, uint64_t bound) {
    if (bound > L.filt) {
        L.filt = bound;
        L.thr_f = __uint_as_float((uint32_t)(bound >> 32));
    }
}

// Warp-uniform insert of `key` (all lanes pass the same key).
__device__ __forceinline__ void wl_insert(WarpList& L, uint64_t key, int w) {
    if (key <= L.filt) return;
    const int lane = lane_id();
    const int pos = __popc(__ballot_sync(0xffffffffu, lane < w && L.v > key));  // entries above key
    const uint64_t up = __shfl_up_sync(0xffffffffu, L.v, 1);
    if (lane < w) L.v = lane < pos ? L.v : (lane == pos ? key : up);
    L.thr = __shfl_sync(0xffffffffu, L.v, w - 1);
    wl_raise(L, L.thr);
}

// Offer one candidate per lane (valid lanes only); the warp inserts every
// offered key that beats the threshold, lane order.
__device__ __forceinline__ void wl_offer(WarpList& L, bool valid, float f, uint32_t idx, int w) {
    unsigned b = __ballot_sync(0xffffffffu, valid && f >= L.thr_f);
    while (b) {
        const int src = __ffs(b) - 1;
        b &= b - 1;
        const float fs = __shfl_sync(0xffffffffu, f, src);
        const uint32_t is = __shfl_sync(0xffffffffu, idx, src);
        if (fs >= L.thr_f) wl_insert(L, beam_key(fs, is), w);
    }
}

struct BeamParams {
    int n_req, w_in, width, w_out, vocab, stride, base_prev, base_new;
    long long total, seg;  // elements of all rows, elements per CTA (multiple of 1024)
    int pieces;            // max list slots per row
    const float* probs;
    int32_t* cand_parent;
    float* cand_prob;
    int32_t* cand_token;
    uint64_t* lists;  // [rows][pieces][kBeamW]
    void* ws;
};

__device__ __forceinline__ int first_cta(const BeamParams& p, long long row) {
    return (int)((row * p.vocab) / p.seg);
}

// Scan: one CTA per row (request, kept parent); 8 warps each stream a
// contiguous 1/8 of the row with 8 float4 loads in flight per lane, keep a
// warp top-w list behind a max-of-float4 prefilter, and merge the 8 lists into
// the row's slot.  (Measured against a persistent TMA-ring variant with
// CTA-shared filters: this simple form streams faster -- DESIGN.md §NEXT-1.)
constexpr int kCandCap = 512;  // per-warp candidate buffer (keys above the warp's threshold)

// The warp's buffered candidates cbuf[0..n) -> their top-w in cbuf[0..min(n,w))
// (warp-distributed list insertion); returns the new count and sets thr to
// the w-th key (0 while fewer than w).
__device__ __forceinline__ int compact_cands(uint64_t* cbuf, int n, int w, uint64_t& thr) {
    WarpList M;
    wl_init(M);
    const int lane = lane_id();
    for (int x0 = 0; x0 < n; x0 += 32) {
        const uint64_t k = x0 + lane < n ? cbuf[x0 + lane] : 0ull;
        unsigned bb = __ballot_sync(0xffffffffu, k > M.thr);
        while (bb) {
            const int src = __ffs(bb) - 1;
            bb &= bb - 1;
            wl_insert(M, __shfl_sync(0xffffffffu, k, src), w);
        }
    }
    __syncwarp();
    if (lane < w) cbuf[lane] = M.v;
    __syncwarp();
    thr = M.thr;
    return min(n, w);
}

__global__ void __launch_bounds__(256) beam_scan_kernel(BeamParams p) {
    __shared__ uint64_t cbuf_all[8][kCandCap];
    pdl_launch_dependents();
    pdl_wait();
    const long long row = blockIdx.x;
    const int i = (int)(row / p.w_in), kpar = (int)(row - (long long)i * p.w_in);
    const float fpar = p.cand_prob[(size_t)i * p.stride + p.base_prev + kpar];
    const float* r = p.probs + (size_t)row * p.vocab;
    const uint32_t ibase = (uint32_t)kpar * (uint32_t)p.vocab;
    const int w = p.w_out, warp = warp_id(), lane = lane_id();
    uint64_t* cbuf = cbuf_all[warp];
    int nc = 0;          // buffered candidates (warp-uniform)
    uint64_t thr = 0ull;  // keys <= thr cannot be in the row's top w (warp-uniform)
    // prefilter on the raw probability: fl32(fpar * e) > thr needs e >= f(thr) / fpar up to
    // 2^-24 rounding; the 2^-18 margin keeps it conservative (exact keys decide)
    const float inv_fpar = fpar > 0.f ? 1.f / fpar : 0.f;
    float e_thr = 0.f;
    auto set_thr = [&](uint64_t t) {
        thr = t;
        const float tf = __uint_as_float((uint32_t)(t >> 32));
        e_thr = fpar > 0.f ? tf * inv_fpar * (1.f - 3.814697265625e-06f) : 0.f;
    };
    // push the elements of this lane that beat thr (warp-aggregated slots)
    auto push = [&](bool ok, float f, uint32_t idx) {
        const uint64_t key = beam_key(f, idx);
        const bool c = ok && key > thr;
        const unsigned bb = __ballot_sync(0xffffffffu, c);
        if (c) cbuf[nc + __popc(bb & ((1u << lane) - 1u))] = key;
        nc += __popc(bb);
    };
    float emin = 0.f;
    const int part = (((p.vocab + 7) / 8) + 3) & ~3;
    const int w0 = min(p.vocab, warp * part), w1 = min(p.vocab, w0 + part);
    const bool vec = ((reinterpret_cast<uintptr_t>(r) & 15u) == 0) && ((p.vocab & 3) == 0);
    if (vec) {
        constexpr int U = 8;
        for (int base = w0; base < w1; base += 32 * 4 * U) {
            float4 x[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int t = base + (u * 32 + lane) * 4;
                x[u] = t < w1 ? __ldcs(reinterpret_cast<const float4*>(r + t)) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int t = base + (u * 32 + lane) * 4;
                const bool ok = t < w1;
                const float mx = fmaxf(fmaxf(x[u].x, x[u].y), fmaxf(x[u].z, x[u].w));
                emin = fminf(emin, fminf(fminf(x[u].x, x[u].y), fminf(x[u].z, x[u].w)));
                if (__any_sync(0xffffffffu, ok && mx >= e_thr)) {  // rare once thr is established
                    if (nc + 128 > kCandCap) {
                        uint64_t t2;
                        nc = compact_cands(cbuf, nc, w, t2);
                        set_thr(t2);
                    }
                    push(ok, __fmul_rn(fpar, x[u].x), ibase + t);
                    push(ok, __fmul_rn(fpar, x[u].y), ibase + t + 1);
                    push(ok, __fmul_rn(fpar, x[u].z), ibase + t + 2);
                    push(ok, __fmul_rn(fpar, x[u].w), ibase + t + 3);
                }
            }
        }
    } else {
        for (int t0 = w0; t0 < w1; t0 += 32) {
            const int t = t0 + lane;
            const bool ok = t < w1;
            const float ev = ok ? r[t] : 0.f;
            emin = fminf(emin, ev);
            if (nc + 32 > kCandCap) {
                uint64_t t2;
                nc = compact_cands(cbuf, nc, w, t2);
                set_thr(t2);
            }
            push(ok, __fmul_rn(fpar, ev), ibase + (uint32_t)t);
        }
    }
    if (emin < 0.f) set_dev_error(p.ws, AS_DEV_BAD_PROB, i);
    __syncwarp();
    {
        uint64_t t2;
        nc = compact_cands(cbuf, nc, w, t2);
        if (lane < kBeamW && lane >= nc) cbuf[lane] = 0ull;  // fewer than w: empty keys
    }
    __syncthreads();
    if (warp == 0) {
        WarpList M;
        wl_init(M);
        for (int x = lane; x < 8 * kBeamW; x += 32) {
            const int wv = x / kBeamW, j = x % kBeamW;
            const uint64_t k = j < w ? cbuf_all[wv][j] : 0ull;
            unsigned bb = __ballot_sync(0xffffffffu, k > M.thr);
            while (bb) {
                const int src = __ffs(bb) - 1;
                bb &= bb - 1;
                wl_insert(M, __shfl_sync(0xffffffffu, k, src), w);
            }
        }
        if (lane < kBeamW) p.lists[(size_t)row * p.pieces * kBeamW + lane] = M.v;
    }
}

__global__ void __launch_bounds__(128) beam_merge_kernel(BeamParams p) {
    pdl_launch_dependents();
    pdl_wait();
    const int i = blockIdx.x * 4 + warp_id();
    if (i >= p.n_req) return;
    const int lane = lane_id();
    const int w = p.w_out;
    WarpList M;
    wl_init(M);
    constexpr int PF = 8;  // keys prefetched per lane (loads in flight before the serial inserts)
    for (int k = 0; k < p.w_in; ++k) {
        const long long row = (long long)i * p.w_in + k;
        const int np = (int)((row * p.vocab + p.vocab - 1) / p.seg) - first_cta(p, row) + 1;
        const uint64_t* K = p.lists + (size_t)row * p.pieces * kBeamW;
        const int nk = np * kBeamW;
        for (int x00 = 0; x00 < nk; x00 += 32 * PF) {
            uint64_t kk[PF];
#pragma unroll
            for (int u = 0; u < PF; ++u) {
                const int x = x00 + u * 32 + lane;
                kk[u] = x < nk ? __ldcg(K + x) : 0ull;
            }
#pragma unroll
            for (int u = 0; u < PF; ++u) {
                const uint64_t key = kk[u];
                unsigned b = __ballot_sync(0xffffffffu, key > M.thr);
                while (b) {
                    const int src = __ffs(b) - 1;
                    b &= b - 1;
                    wl_insert(M, __shfl_sync(0xffffffffu, key, src), w);
                }
            }
        }
    }
    if (lane < w) {
        const uint64_t key = M.v;
        const uint32_t idx = 0xFFFFFFFFu - (uint32_t)(key & 0xFFFFFFFFull);
        const int kpar = (int)(idx / (uint32_t)p.vocab);
        const int t = (int)(idx - (uint32_t)kpar * (uint32_t)p.vocab);
        const size_t node = (size_t)i * p.stride + p.base_new + lane;
        p.cand_parent[node] = p.base_prev + kpar;
        p.cand_token[node] = t;
        p.cand_prob[node] = __uint_as_float((uint32_t)(key >> 32));
    }
}

static void beam_geometry(int n_req, int w_in, int vocab, long long* total, long long* seg, int* grid, int* pieces) {
    *total = (long long)n_req * w_in * vocab;
    *seg = vocab;  // one row per CTA
    *grid = n_req * w_in;
    *pieces = 1;
}

size_t beam_ws_bytes(int n_req, int width, int vocab) {
    long long total, seg;
    int grid, pieces;
    beam_geometry(n_req, width, vocab, &total, &seg, &grid, &pieces);  // w_in <= width
    long long t1, s1;
    int g1, p1;
    beam_geometry(n_req, 1, vocab, &t1, &s1, &g1, &p1);  // layer 1 may cut rows finer
    const int pmax = pieces > p1 ? pieces : p1;
    return kWsHeaderBytes + align_up((size_t)n_req * width * pmax * kBeamW * 8, 256);
}

int launch_beam(int n_req, int layer, int width, int vocab, const float* probs, int stride, int32_t* cand_parent,
                float* cand_prob, int32_t* cand_token, void* ws, cudaStream_t stream) {
    BeamParams p;
    p.n_req = n_req;
    p.w_in = layer == 1 ? 1 : width;
    p.width = width;
    p.w_out = width;  // vocab >= width (checked by the ABI)
    p.vocab = vocab;
    int grid;
    beam_geometry(n_req, p.w_in, vocab, &p.total, &p.seg, &grid, &p.pieces);
    p.stride = stride;
    p.base_prev = layer == 1 ? 0 : 1 + (layer - 2) * width;
    p.base_new = 1 + (layer - 1) * width;
    p.probs = probs;
    p.cand_parent = cand_parent;
    p.cand_prob = cand_prob;
    p.cand_token = cand_token;
    p.lists = reinterpret_cast<uint64_t*>(reinterpret_cast<unsigned char*>(ws) + kWsHeaderBytes);
    p.ws = ws;
    cudaLaunchAttribute attr[1];
    cudaLaunchConfig_t c1 = {};
    c1.gridDim = dim3(grid);
    c1.blockDim = dim3(256);
    c1.dynamicSmemBytes = 0;
    c1.stream = stream;
    c1.attrs = attr;
    c1.numAttrs = fill_launch_attrs(attr);
    cudaLaunchConfig_t c2 = c1;
    c2.gridDim = dim3((n_req + 3) / 4);
    c2.blockDim = dim3(128);
    c2.dynamicSmemBytes = 0;
    cudaError_t e = cudaLaunchKernelEx(&c1, beam_scan_kernel, p);
    if (e == cudaSuccess) e = cudaLaunchKernelEx(&c2, beam_merge_kernel, p);
    if (e != cudaSuccess) return -1;
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace as
