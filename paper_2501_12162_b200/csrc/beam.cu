// beam.cu -- NEXT-1: as_beam_step, one layer of Step 1 speculation.
//
// For every request, the kept nodes of the previous layer (w_in = 1 at layer 1,
// else w) each get the draft model's distribution over the vocabulary; every
// expansion (parent k, token t) has the approximated path probability
// f-hat = fl32(f-hat(parent k) * M_q(t | X, Path(k))), and the layer
// keeps the w largest by (f-hat desc, parent asc, token asc) (R8).  The w x |V|
// scan is HBM-bound (|V| = 128 256: 513 KB of fp32 per row):
//
//   beam_scan_kernel   one CTA per row: 16-byte streaming loads, a warp-wide
//                      top-w list of the 64-bit keys (f-hat bits << 32 |
//                      ~(k*|V| + t)) -- the key order IS the tie order and keys
//                      are unique -- behind a cheap max-of-float4 prefilter,
//                      the 8 warp lists merged into the row's slot.
//   beam_merge_kernel  one warp per request: top-w of its rows' lists; writes
//                      the new layer's nodes into the candidate forest.
#include <mutex>

#include "params.cuh"

namespace as {

// Scan staging: each warp streams its chunk through a ring of kBeamStages batches of
// kBeamUA float4 per lane in shared memory (LDGSTS, no registers held by loads in
// flight): kBeamStages - 1 batches stay in flight while one is filtered.
#ifndef AS_BEAM_STAGES
#define AS_BEAM_STAGES 3
#endif
constexpr int kBeamUA = 4, kBeamStages = AS_BEAM_STAGES;
constexpr int kBeamRingBytes = 8 * kBeamStages * kBeamUA * 32 * 16;  // 8 warps (48 KB at 3 stages)

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(smem_dst)),
                 "l"(gsrc)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

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


// Scan: one CTA per row (request, kept parent); 8 warps each stream a
// contiguous 1/8 of the row with 8 float4 loads in flight per lane, keep a
// warp top-w list behind a max-of-float4 prefilter, and merge the 8 lists into
// the row's slot.  (Measured against a persistent TMA-ring variant with
// CTA-shared filters: this simple form streams faster -- DESIGN.md §NEXT-1.)
template <bool RING>
__global__ void __launch_bounds__(256) beam_scan_kernel(BeamParams p) {
    __shared__ uint64_t wls[8][kBeamW];
    __shared__ unsigned long long s_bound;  // max over the 8 warps of their w-th key
    if (threadIdx.x == 0) s_bound = 0ull;
    __syncthreads();
    pdl_launch_dependents();
    pdl_wait();
    const long long row = blockIdx.x / p.pieces;   // small batches: each row split into `pieces` CTAs
    const int pc = (int)(blockIdx.x - row * p.pieces);
    const int a = (int)min((long long)p.vocab, (long long)pc * p.seg), e = (int)min((long long)p.vocab, a + p.seg);
    const int i = (int)(row / p.w_in), kpar = (int)(row - (long long)i * p.w_in);
    const float fpar = p.cand_prob[(size_t)i * p.stride + p.base_prev + kpar];
    const float* r = p.probs + (size_t)row * p.vocab;
    const uint32_t ibase = (uint32_t)kpar * (uint32_t)p.vocab;
    const int w = p.w_out, warp = warp_id(), lane = lane_id();
    WarpList L;
    wl_init(L);
    float emin = 0.f;
    const int part = ((((e - a) + 7) / 8) + 3) & ~3;
    const int w0 = min(e, a + warp * part), w1 = min(e, w0 + part);
    const bool vec = ((reinterpret_cast<uintptr_t>(r) & 15u) == 0) && ((p.vocab & 3) == 0);
    if (vec && RING) {
        // grids of more than one wave: batches staged through the LDGSTS ring
        constexpr int U = kBeamUA, BATCH = 32 * 4 * U;  // floats per batch
        extern __shared__ __align__(16) float4 ring_all[];
        float4* ring = ring_all + (size_t)warp * kBeamStages * U * 32;
        const int nb = w1 > w0 ? (w1 - w0 + BATCH - 1) / BATCH : 0;
        // each lane copies and later reads only its own 16-byte slots: a thread's
        // wait_group makes its own copies visible, no warp barrier needed
        auto issue = [&](int bi) {
            if (bi < nb) {
                float4* st = ring + (bi % kBeamStages) * U * 32;
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int t = w0 + bi * BATCH + (u * 32 + lane) * 4;
                    if (t < w1) cp_async16(st + u * 32 + lane, r + t);
                }
            }
            cp_async_commit();  // (empty groups keep the count uniform)
        };
#pragma unroll
        for (int s = 0; s < kBeamStages - 1; ++s) issue(s);
        uint64_t published = 0ull;
        for (int bi = 0; bi < nb; ++bi) {
            const int base = w0 + bi * BATCH;
            issue(bi + kBeamStages - 1);
            cp_async_wait<kBeamStages - 1>();
            // a key below any warp's w-th key is out of the row's top w: share the best bound
            if (L.thr > published) {
                if (lane == 0) atomicMax(&s_bound, (unsigned long long)L.thr);
                published = L.thr;
            }
            uint64_t sb = 0ull;
            if (lane == 0) sb = *reinterpret_cast<volatile unsigned long long*>(&s_bound);
            wl_raise(L, __shfl_sync(0xffffffffu, sb, 0));
            float4 x[U];
            const float4* st = ring + (bi % kBeamStages) * U * 32;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int t = base + (u * 32 + lane) * 4;
                x[u] = t < w1 ? st[u * 32 + lane] : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int t = base + (u * 32 + lane) * 4;
                const bool ok = t < w1;
                const float f0 = __fmul_rn(fpar, x[u].x), f1 = __fmul_rn(fpar, x[u].y);
                const float f2 = __fmul_rn(fpar, x[u].z), f3 = __fmul_rn(fpar, x[u].w);
                emin = fminf(emin, fminf(fminf(x[u].x, x[u].y), fminf(x[u].z, x[u].w)));
                const bool any = ok && fmaxf(fmaxf(f0, f1), fmaxf(f2, f3)) >= L.thr_f;
                if (__any_sync(0xffffffffu, any)) {
                    wl_offer(L, ok, f0, ibase + t, w);
                    wl_offer(L, ok, f1, ibase + t + 1, w);
                    wl_offer(L, ok, f2, ibase + t + 2, w);
                    wl_offer(L, ok, f3, ibase + t + 3, w);
                }
            }
        }
    } else if (vec) {
        constexpr int U = 8;
        uint64_t published = 0ull;
        for (int base = w0; base < w1; base += 32 * 4 * U) {
            // a key below any warp's w-th key is out of the row's top w: share the best bound
            if (L.thr > published) {
                if (lane == 0) atomicMax(&s_bound, (unsigned long long)L.thr);
                published = L.thr;
            }
            uint64_t sb = 0ull;
            if (lane == 0) sb = *reinterpret_cast<volatile unsigned long long*>(&s_bound);
            wl_raise(L, __shfl_sync(0xffffffffu, sb, 0));
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
                const float f0 = __fmul_rn(fpar, x[u].x), f1 = __fmul_rn(fpar, x[u].y);
                const float f2 = __fmul_rn(fpar, x[u].z), f3 = __fmul_rn(fpar, x[u].w);
                emin = fminf(emin, fminf(fminf(x[u].x, x[u].y), fminf(x[u].z, x[u].w)));
                const bool any = ok && fmaxf(fmaxf(f0, f1), fmaxf(f2, f3)) >= L.thr_f;
                if (__any_sync(0xffffffffu, any)) {
                    wl_offer(L, ok, f0, ibase + t, w);
                    wl_offer(L, ok, f1, ibase + t + 1, w);
                    wl_offer(L, ok, f2, ibase + t + 2, w);
                    wl_offer(L, ok, f3, ibase + t + 3, w);
                }
            }
        }
    } else {
        for (int t0 = w0; t0 < w1; t0 += 32) {
            const int t = t0 + lane;
            const bool ok = t < w1;
            const float ev = ok ? r[t] : 0.f;
            emin = fminf(emin, ev);
            wl_offer(L, ok, __fmul_rn(fpar, ev), ibase + (uint32_t)t, w);
        }
    }
    if (RING && vec) cp_async_wait<0>();  // (only empty groups can still be pending)
    if (emin < 0.f) set_dev_error(p.ws, AS_DEV_BAD_PROB, i);
    if (lane < kBeamW) wls[warp][lane] = L.v;
    __syncthreads();
    if (warp == 0) {
        WarpList M;
        wl_init(M);
        for (int x = lane; x < 8 * kBeamW; x += 32) {
            const uint64_t k = wls[x / kBeamW][x % kBeamW];
            unsigned bb = __ballot_sync(0xffffffffu, k > M.thr);
            while (bb) {
                const int src = __ffs(bb) - 1;
                bb &= bb - 1;
                wl_insert(M, __shfl_sync(0xffffffffu, k, src), w);
            }
        }
        if (lane < kBeamW) p.lists[((size_t)row * p.pieces + pc) * kBeamW + lane] = M.v;
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
    // the request's rows' lists are contiguous ([w_in][pieces][kBeamW] keys):
    // one pass, PF keys per lane in flight before the serial inserts
    constexpr int PF = 8;
    const int nk = p.w_in * p.pieces * kBeamW;
    const uint64_t* K = p.lists + (size_t)i * nk;
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

// One CTA per row; batches too small to fill the GPU (fewer rows than ~half the
// resident CTA slots, 148 SMs x 4) split each row into `pieces` (>= 8192
// elements each, 16-byte aligned), merged by the merge kernel.
static void beam_geometry(int n_req, int w_in, int vocab, long long* total, long long* seg, int* grid, int* pieces) {
    const long long rows = (long long)n_req * w_in;
    *total = rows * vocab;
    int k = 1;
    if (rows > 0 && rows < 296) k = (int)(592 / rows);
    k = max(1, min(k, max(1, vocab / 8192)));
    long long sg = (vocab + k - 1) / k;
    sg = (sg + 3) / 4 * 4;
    k = (int)((vocab + sg - 1) / sg);
    *seg = sg;
    *pieces = k;
    *grid = (int)(rows * k);
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
    int n_sms = 148;
    {
        // the ring exceeds the 48 KB default: set once per device, under a mutex (re-entrant ABI)
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return -1;
        static std::mutex mu;
        static bool attr_set[64] = {false};
        static int sms[64] = {0};
        std::lock_guard<std::mutex> lk(mu);
        if (!attr_set[dev]) {
            if (cudaFuncSetAttribute(beam_scan_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     kBeamRingBytes) != cudaSuccess ||
                cudaDeviceGetAttribute(&sms[dev], cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
                return -1;
            attr_set[dev] = true;
        }
        n_sms = sms[dev];
    }
    cudaLaunchAttribute attr[1];
    cudaLaunchConfig_t c1 = {};
    c1.gridDim = dim3(grid);
    c1.blockDim = dim3(256);
    // the ring pays when the rows take more than one wave (4 CTAs per SM): c3 229 -> 203 us;
    // within one wave the register loads are faster (c2 68.4 vs 70.6 us)
    const bool ring = grid > 4 * n_sms;
    c1.dynamicSmemBytes = ring ? kBeamRingBytes : 0;
    c1.stream = stream;
    c1.attrs = attr;
    c1.numAttrs = fill_launch_attrs(attr);
    cudaLaunchConfig_t c2 = c1;
    c2.gridDim = dim3((n_req + 3) / 4);
    c2.blockDim = dim3(128);
    c2.dynamicSmemBytes = 0;
    cudaError_t e = ring ? cudaLaunchKernelEx(&c1, beam_scan_kernel<true>, p)
                         : cudaLaunchKernelEx(&c1, beam_scan_kernel<false>, p);
    if (e == cudaSuccess) e = cudaLaunchKernelEx(&c2, beam_merge_kernel, p);
    if (e != cudaSuccess) return -1;
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace as
