// attn_tc.cu -- K2: as_tree_verify_attn for dtype AS_BF16 on sm_100a.
//
// Step 4 verification: every tree node of request i attends to
// the request's committed prefix (paged KV cache, D6/P:L935) and to its tree
// ancestors-or-self (R15).  Per (request i, kv head g) the G query heads of
// all K_i nodes form Q rows r = node*G + hh, so one kv head's keys are read
// from HBM once for all G*K_i rows (c2: 4*32 = 128 rows = one UMMA M tile).
//
// Structure: persistent, TWO 192-thread CTAs per SM (measured: one CTA's TMA
// stream tops out near 4.7 TB/s chip-wide with 16 KB operations, two CTAs per
// SM reach 6.5-6.9 TB/s -- DESIGN.md §5); static or split-KV schedule.
//   warp 0      TMA producer: Q tile (4-D map, box 64 x G x 128/G x 2 chunks,
//               SW128) and 64-key K/V tiles (5-D map over [page][head][row]
//               [chunk][64] -> one 16 KB box per tile, coordinates from the
//               page-table row staged in shared memory; k_tree/v_tree for the
//               tree tiles).  K_{t+1} and V_t are issued by two lanes of the
//               same instructions (consumption order).
//   warp 1      TMEM owner + single-thread tcgen05.mma issuer:
//               S_t = Q K_t^T (M=128, N=64, K=d; SS, both K-major SW128) into
//               TMEM S buffer t&1; O += P_t V_t (M=128, N=d, K=64; A = P_t read
//               from TMEM where the softmax wrote it over S_t, V MN-major SW128).
//               Issue order QK_0 QK_1 PV_0 QK_2 PV_1 ...: S is double-buffered,
//               so S_{t+1} is computed while the softmax works on S_t, and
//               QK_{t+2} may overwrite buffer t&1 right after PV_t is issued
//               (tcgen05.mma of one thread execute in issue order).
//   warps 2-5   softmax + epilogue, one TMEM lane (= Q row) per thread:
//               tcgen05.ld S -> mask (prefix length / ancestor bit words) ->
//               online softmax in the log2 domain with lazy O rescaling
//               (only when the running max grows by > 8, i.e. 256x) ->
//               P (bf16 pairs) tcgen05.st over S_t -> PV.  Epilogue:
//               tcgen05.ld O, * 1/l, bf16 store, optional natural-log LSE; or,
//               for a unit split across CTAs (split-KV), the fp32 partial
//               (O, m, l), then a share of the unit's cooperative merge.
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "params.cuh"
#include "tc_ptx.cuh"

namespace as {

constexpr int kBM = 128;          // query rows per tile (UMMA M)
constexpr int kBN = 64;           // keys per tile
// Two CTA shapes (template NQ = q-tiles processed per CTA):
//  NQ = 1: 192 threads (TMA producer, MMA, 4 softmax warps), 2 CTAs per SM,
//          256 TMEM columns, 2+2-stage K/V rings -- every unit its own K/V stream;
//  NQ = 2: 384 threads (producer, 2 MMA warps, 1 idle, 2 x 4 softmax warps), 1 CTA/SM, all
//          512 TMEM columns, 4+5-stage rings -- the two q-tiles of a (request,
//          kv head) share every K/V tile (loaded once for both), chosen when the
//          trees span more than one 128-row q-tile (c4/c5 shapes).
// TMEM columns of q-tile q (base q * (128 + D)): S/P buffers b = 0, 1 at
// base + 64 b (S_t fp32 in 64 columns; P_t bf16 pairs over its first 32), O at
// base + 128.
template <int NQ> struct TcCfg;
template <> struct TcCfg<1> {
    static constexpr int THREADS = 192, CTAS = 2, TMEM = 256, KST = 2, VST = 2;
};
// NQ = 2: warps 0-3 = producer, 2 MMA issuers, one idle warp (warpgroup 0);
// softmax groups = warps 4-7 and 8-11 (warpgroups 1, 2), so setmaxnreg moves
// registers from warpgroup 0 to the softmax warpgroups.
template <> struct TcCfg<2> {
    static constexpr int THREADS = 384, CTAS = 1, TMEM = 512, KST = 4, VST = 5;
};
constexpr int kRegLow = 56, kRegHigh = 224;  // 128 * 56 + 256 * 224 = 384 * 168 (the launch allocation)
constexpr int kCtasPerSm = 2;     // max over the shapes (workspace sizing)
constexpr int kPtChunk = 256;     // page-table entries staged per refill
constexpr float kRescaleThresh = 8.0f;  // log2 units
constexpr int kMaxRec = 64;       // pieces per CTA precomputed in the prologue
constexpr int kMaxSplit = 8;      // split-KV: pieces per unit when units are fewer than CTAs
constexpr int kTraceCtas = 512;   // per-CTA timeline records after the CTA-0 tile trace (debug)
constexpr int kAncWords = AS_MAX_TREE / 64;  // 64-bit ancestor words per row (one per tree tile)
#ifdef AS_DEBUG
constexpr bool kDebug = true;     // timing-experiment switches (p.debug_mode, trace) compiled in
#else
constexpr bool kDebug = false;
#endif

// A piece precomputed in the prologue (shared memory): no global load and no
// request walk at a unit boundary.
struct PieceRec {
    int i, j, tb, te;  // request, unit within request (g*MT + mt), tile range
    int off, K, L, x;  // request geometry, piece kind (Piece::x)
    int x0, tr;        // tail pieces only (Piece::x0, Piece::tr)
};

// PR (CTA pair, cta_group::2): each CTA holds HALF of every K/V tile (K: 32 of
// the 64 keys; V: its 64-column d-chunk), so a stage is 8 KB and the rings are
// twice as deep in the same shared memory.
template <int D, int NQ, bool PR = false>
struct TcSmem {
    static constexpr int KST = TcCfg<NQ>::KST * (PR ? 2 : 1), VST = TcCfg<NQ>::VST * (PR ? 2 : 1);
    static constexpr int NCH = D / 64;                        // 128-byte swizzle chunks along d
    static constexpr int Q_BYTES = NCH * kBM * 128;           // 16 KB per chunk (one q-tile)
    static constexpr int KV_BYTES = NCH * kBN * 128 / (PR ? 2 : 1);  // 8 KB per chunk (PR: per half tile)
    static constexpr int KH_ROWS = PR ? kBN / 2 : kBN;        // K rows held per CTA
    static constexpr int OFF_Q = 0;                           // [NQ] q-tiles
    static constexpr int OFF_K = OFF_Q + NQ * Q_BYTES;
    static constexpr int OFF_V = OFF_K + KST * KV_BYTES;
    static constexpr int OFF_PT = OFF_V + VST * KV_BYTES;     // [kPtChunk] staged page-table row
    static constexpr int OFF_ANC = OFF_PT + kPtChunk * 4;     // [NQ][kAncWords][128] ancestor words per row
    static constexpr int OFF_TP = OFF_ANC + NQ * kAncWords * kBM * 8;  // [NQ][2][AS_MAX_TREE] staged tree parents
    static constexpr int OFF_REC = OFF_TP + NQ * 2 * AS_MAX_TREE * 4;  // [kMaxRec] this CTA's pieces
    static constexpr int OFF_BAR = OFF_REC + kMaxRec * (int)sizeof(PieceRec);
    // q_full q_empty, K/V rings, and per q-tile: s_full[2] p_full[2] pv_done[2] o_full o_empty
    static constexpr int N_BAR = 2 + 2 * KST + 2 * VST + NQ * 8;
    static constexpr int OFF_TMEM = OFF_BAR + N_BAR * 8;
    static constexpr int BYTES = OFF_TMEM + 16;
    static constexpr int ALLOC = BYTES + 1024;  // alignment slack
    // schedule-plan scratch (long long per request) aliases the K+V rings before any TMA
    // per request: tile prefix (8 B), unit prefix (8 B), geometry {off, K, L} (16 B)
    static constexpr int PLAN_N = (KST + VST) * KV_BYTES / 32;
    static constexpr int TM_QT = 128 + D;           // TMEM columns per q-tile (2 S/P buffers + O)
    static_assert(NQ * TM_QT <= TcCfg<NQ>::TMEM, "TMEM columns");
    static_assert(TcCfg<NQ>::CTAS * (ALLOC + 1024) <= 233472, "shared memory per SM");
};

// CTA-0 pipeline trace (debug): event e of CTA-local tile index idx.
#define AS_TRACE(e, idx)                                                                       \
    do {                                                                                       \
        if (kDebug && p.trace != nullptr && blockIdx.x == 0 && (int)(idx) < p.trace_cap)      \
            p.trace[(size_t)(idx) * 8 + (e)] = clock64();                                      \
        else if (kDebug && PR && p.trace != nullptr && blockIdx.x == 1 && (int)(idx) < 500)    \
            p.trace[(size_t)(2500 + (idx)) * 8 + (e)] = clock64();                             \
    } while (0)

// CTA-0 epilogue trace (debug): event e of the CTA's piece k (rows 3000.. of the tile trace).
#define AS_EPI_TRACE(e, k)                                                                        \
    do {                                                                                          \
        if (kDebug && p.trace != nullptr && blockIdx.x == 0 && gtid == 0 && grp == 0 && (k) < 64) { \
            unsigned long long tn_;                                                               \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tn_));                               \
            p.trace[(size_t)(3000 + (k)) * 8 + (e)] = tn_;                                        \
        }                                                                                         \
    } while (0)

// CTA pair, peer side: the 4 warps of a softmax group count themselves on a
// shared counter (acq_rel: the last one sees the others' TMEM writes) and the
// last forwards ONE cluster-scope arrive to the leader's barrier -- one remote
// release per group and tile instead of four.
__device__ __forceinline__ void peer_group_arrive(int* cnt, uint64_t* bar) {
    int old;
    asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;" : "=r"(old) : "r"(ptx::smem_u32(cnt)) : "memory");
    if (old == 3) {
        *reinterpret_cast<volatile int*>(cnt) = 0;  // next use of this counter is two tiles later
        ptx::mbar_arrive_remote(bar, 0);
    }
}

// Named barrier of one softmax warp group (128 threads; ids 1 and 2, constant
// operands so the kernel claims only the barriers it uses).
__device__ __forceinline__ void group_bar(int grp) {
    if (grp == 0) asm volatile("bar.sync 1, 128;" ::: "memory");
    else asm volatile("bar.sync 2, 128;" ::: "memory");
}

struct Unit {
    int i, g, mt, nq, off, K, L, nt, n_prefix;  // mt = first q-tile, nq = q-tiles in this unit
};

// Per-request geometry: QT q-tiles of 128 rows (rows = node*G + hh) per kv head,
// grouped p.nq at a time into MT units per head; nt KV tiles.
struct Req {
    int off, K, L, QT, MT, nt, n_prefix;
};

// Request geometry from {tree offset, tree size, kv_len} (the plan caches the
// triple in shared memory: the prologue's later steps make no global loads).
__device__ __forceinline__ void req_from(const TcParams& p, int off, int K, int L, Req& r) {
    r.off = off;
    r.K = K;
    r.L = L;
    if (r.L < 0) r.L = 0;
    if (r.L > p.max_pages * p.page_size) r.L = p.max_pages * p.page_size;
    r.n_prefix = (r.L + kBN - 1) / kBN;
    const bool ok = r.K > 0 && r.K <= AS_MAX_TREE && r.off + r.K <= p.n_tree_rows;
    r.QT = ok ? (r.K * p.G + kBM - 1) / kBM : 0;
    r.MT = (r.QT + p.nq - 1) / p.nq;
    r.nt = r.n_prefix + (r.K + kBN - 1) / kBN;
}

__device__ __forceinline__ void req_geo(const TcParams& p, const int4* geo, int i, Req& r) {
    const int4 g = geo[i];
    req_from(p, g.x, g.y, g.z, r);
}

__device__ __forceinline__ void make_unit(const TcParams& p, const Req& r, int i, int j, Unit& u) {
    u.i = i;
    u.g = j / r.MT;
    u.mt = (j - u.g * r.MT) * p.nq;
    u.nq = min(p.nq, r.QT - u.mt);
    u.off = r.off;
    u.K = r.K;
    u.L = r.L;
    u.nt = r.nt;
    u.n_prefix = r.n_prefix;
}

// ---------------------------------------------------------------------------
// Work schedule.  Units are (request i, kv head g, q-tile mt) in that order --
// the q-tiles of one (i, g) are adjacent, so CTAs running them side by side
// read that head's KV from L2 the second time.  A "piece" is a contiguous tile
// range [tb, te) of one unit.
//  static mode: non-empty unit k goes to CTA k mod G (whole units);
//  split-KV mode (units <= CTAs / 2): unit k's tiles are cut into S pieces,
//   piece s on CTA k*S + s; the co-resident pieces publish fp32 (O, m, l),
//   wait for each other and each merges 1/S of the columns.
// ---------------------------------------------------------------------------
struct Piece {
    Unit u;
    int w;         // unit id (i, g, mt) -> counter index
    int tb, te;    // tile range of this piece
    int x;         // >= 0: co-resident split-KV piece index; -1: whole unit; -2 - e: tail piece (e = 0
                   // the CTA's first tail piece, 1 its last), merged by the last finisher
    int x0, tr;    // tail pieces: the unit's first tile in the remainder stream, the stream's length
};

// The roles (producer, MMA, softmax) only replay the CTA's records.
struct RecCursor {
    int nrec, q;
    const PieceRec* rec;
};

__device__ __forceinline__ bool rec_next(const TcParams& p, RecCursor& cur, Piece& pc) {
    if (cur.q >= cur.nrec) return false;
    const PieceRec rc = cur.rec[cur.q++];
    Req r;
    r.off = rc.off;
    r.K = rc.K;
    r.L = rc.L;
    r.n_prefix = (r.L + kBN - 1) / kBN;
    r.QT = (r.K * p.G + kBM - 1) / kBM;
    r.MT = (r.QT + p.nq - 1) / p.nq;
    r.nt = r.n_prefix + (r.K + kBN - 1) / kBN;
    make_unit(p, r, rc.i, rc.j, pc.u);
    pc.w = (rc.i * p.n_kv + pc.u.g) * p.mt_max + pc.u.mt;
    pc.tb = rc.tb;
    pc.te = rc.te;
    pc.x = rc.x;
    pc.x0 = rc.x0;
    pc.tr = rc.tr;
    return true;
}

// Split-KV merge of one row (DESIGN.md §5 "Schedule"): the unit's live pieces each left an
// unnormalised fp32 (O, m, l) in their slot; this thread combines columns
// [c_lo, c_hi) of row r (its share among the n_live pieces) into bf16 out_row,
// out_row[c] = sum_s 2^(m_s - M) O_s[c] / sum_s 2^(m_s - M) l_s, M = max_s m_s.
// Kept out of line so its registers do not count against the tile loop's.
template <int D>
__device__ __noinline__ void split_merge(const float* __restrict__ slot0, size_t slot_stride, int Sx, int nt, int r,
                                         int my_rank, int n_live, __nv_bfloat16* out_row, float* lse_out) {
    float mb[kMaxSplit], lb[kMaxSplit];
    float M = -INFINITY;
#pragma unroll
    for (int s2 = 0; s2 < kMaxSplit; ++s2) {  // all (m, l) loads in flight at once
        mb[s2] = -INFINITY;
        lb[s2] = 0.f;
        if (s2 < Sx && nt * (s2 + 1) / Sx > nt * s2 / Sx) {
            mb[s2] = __ldcg(slot0 + s2 * slot_stride + 128 * D + r);
            lb[s2] = __ldcg(slot0 + s2 * slot_stride + 128 * D + 128 + r);
        }
    }
#pragma unroll
    for (int s2 = 0; s2 < kMaxSplit; ++s2) M = fmaxf(M, mb[s2]);
    float Ltot = 0.f;
#pragma unroll
    for (int s2 = 0; s2 < kMaxSplit; ++s2) {
        mb[s2] = mb[s2] == -INFINITY ? 0.f : ptx::ex2(mb[s2] - M);  // piece weight
        Ltot += lb[s2] * mb[s2];
    }
    const float invL = 1.f / Ltot;
#pragma unroll
    for (int s2 = 0; s2 < kMaxSplit; ++s2) mb[s2] *= invL;
    if (out_row != nullptr) {
        // this piece's columns: a multiple of 8 (16-byte bf16 stores)
        const int c_lo = my_rank * (D / 8) / n_live * 8, c_hi = (my_rank + 1) * (D / 8) / n_live * 8;
#pragma unroll 2
        for (int c0 = c_lo; c0 < c_hi; c0 += 8) {
            float acc[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[j] = 0.f;
            float4 qa[kMaxSplit], qb[kMaxSplit];
#pragma unroll
            for (int s2 = 0; s2 < kMaxSplit; ++s2) {  // every piece's 8 columns in flight
                qa[s2] = qb[s2] = make_float4(0.f, 0.f, 0.f, 0.f);
                if (s2 < Sx && mb[s2] != 0.f) {
                    const float4* src = reinterpret_cast<const float4*>(slot0 + s2 * slot_stride) + (c0 / 4) * 128 + r;
                    qa[s2] = __ldcg(src);
                    qb[s2] = __ldcg(src + 128);
                }
            }
#pragma unroll
            for (int s2 = 0; s2 < kMaxSplit; ++s2) {
                const float fb = mb[s2];
                acc[0] = fmaf(qa[s2].x, fb, acc[0]);
                acc[1] = fmaf(qa[s2].y, fb, acc[1]);
                acc[2] = fmaf(qa[s2].z, fb, acc[2]);
                acc[3] = fmaf(qa[s2].w, fb, acc[3]);
                acc[4] = fmaf(qb[s2].x, fb, acc[4]);
                acc[5] = fmaf(qb[s2].y, fb, acc[5]);
                acc[6] = fmaf(qb[s2].z, fb, acc[6]);
                acc[7] = fmaf(qb[s2].w, fb, acc[7]);
            }
            uint32_t pkk[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                __nv_bfloat162 h2 = __floats2bfloat162_rn(acc[2 * j], acc[2 * j + 1]);
                pkk[j] = *reinterpret_cast<uint32_t*>(&h2);
            }
            *reinterpret_cast<uint4*>(out_row + c0) = make_uint4(pkk[0], pkk[1], pkk[2], pkk[3]);
        }
    }
    if (lse_out != nullptr) *lse_out = (M + __log2f(Ltot)) * 0.6931471805599453f;
}

// Tail stream-K merge (DESIGN.md §5 "Schedule"): the last of a unit's pieces to
// finish combines its own unnormalised (O in TMEM, m, l) with the other pieces'
// fp32 partials for row r.  The n_pc <= 3 pieces are combined in the unit's
// piece order (own_pos = this piece's position, slot[k] = piece k's partial
// slot), whichever piece merges, so the result is deterministic:
// out_row[c] = sum_k 2^(m_k - M) O_k[c] / sum_k 2^(m_k - M) l_k, M = max_k m_k,
// the sum evaluated as a = w_0 O_0; a = fma(O_k, w_k, a) for k = 1, 2.
// One L2 round trip per remote piece: a round issues the loads of all its
// columns at once (the partial was written moments ago by another SM) and the
// running sum is kept in this piece's O columns of TMEM between rounds.
template <int D, int NC, int NR>
__device__ __forceinline__ void tail_round(uint32_t o_addr, int cb, const float* r0p, const float* r1p, float w0,
                                           float w1, bool own_after, bool fresh, float w_own, bool fin, float inv,
                                           int r, __nv_bfloat16* out_row) {
    float4 q[NR][NC / 4];
#pragma unroll
    for (int j = 0; j < NC / 4; ++j) {  // every load of the round in flight before the first use
        q[0][j] = __ldcg(reinterpret_cast<const float4*>(r0p) + (cb / 4 + j) * 128 + r);
        if (NR > 1) q[NR - 1][j] = __ldcg(reinterpret_cast<const float4*>(r1p) + (cb / 4 + j) * 128 + r);
    }
#pragma unroll
    for (int c = 0; c < NC; c += 32) {
        uint32_t oa[32];
        ptx::tmem_ld32(o_addr + cb + c, oa);
        ptx::tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 32; ++e) {
            const float t = __uint_as_float(oa[e]);
            const float4 v0 = q[0][(c + e) >> 2];
            const float x0 = (e & 3) == 0 ? v0.x : (e & 3) == 1 ? v0.y : (e & 3) == 2 ? v0.z : v0.w;
            float x1 = 0.f;
            if (NR > 1) {
                const float4 v1 = q[NR - 1][(c + e) >> 2];
                x1 = (e & 3) == 0 ? v1.x : (e & 3) == 1 ? v1.y : (e & 3) == 2 ? v1.z : v1.w;
            }
            float a;
            if (own_after) {  // remotes precede this piece in the unit's order
                a = fmaf(x0, w0, 0.f);
                if (NR > 1) a = fmaf(x1, w1, a);
                a = fmaf(t, w_own, a);
            } else {          // TMEM holds the running sum (or this piece's own O, fresh)
                a = fresh ? fmaf(t, w_own, 0.f) : t;
                a = fmaf(x0, w0, a);
                if (NR > 1) a = fmaf(x1, w1, a);
            }
            oa[e] = __float_as_uint(a);
        }
        if (fin) {
            if (out_row != nullptr) {
                uint32_t pk[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(oa[2 * j]) * inv,
                                                             __uint_as_float(oa[2 * j + 1]) * inv);
                    pk[j] = *reinterpret_cast<uint32_t*>(&h);
                }
                uint4* dst = reinterpret_cast<uint4*>(out_row + cb + c);
#pragma unroll
                for (int j = 0; j < 4; ++j) dst[j] = make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
            }
        } else {
            ptx::tmem_st32(o_addr + cb + c, oa);
        }
    }
    if (!fin) ptx::tmem_st_wait();
}

template <int D>
__device__ __noinline__ void tail_merge(uint32_t o_addr, float m_own, float l_own, const float* __restrict__ part0,
                                        size_t slot_floats, int n_pc, int own_pos, int s0, int s1, int s2, int r,
                                        __nv_bfloat16* out_row, float* lse_out) {
    const int sl[3] = {s0, s1, s2};
    const float* src[3];
    float mo[3], wo[3], lo[3];
    float M = -INFINITY;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        src[k] = part0 + (size_t)sl[k] * slot_floats;
        mo[k] = -INFINITY;
        lo[k] = 0.f;
        if (k == own_pos) {
            mo[k] = m_own;
            lo[k] = l_own;
        } else if (k < n_pc) {
            mo[k] = __ldcg(src[k] + 128 * D + r);
            lo[k] = __ldcg(src[k] + 128 * D + 128 + r);
        }
        M = fmaxf(M, mo[k]);
    }
    float Ltot = 0.f;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        wo[k] = mo[k] == -INFINITY ? 0.f : ptx::ex2(mo[k] - M);
        Ltot = fmaf(lo[k], wo[k], Ltot);
    }
    const float inv = 1.f / Ltot;
    const float wown = own_pos == 0 ? wo[0] : own_pos == 1 ? wo[1] : wo[2];
    if (n_pc <= 1) {  // (a merger has >= 2 pieces; kept defined)
#pragma unroll 1
        for (int c0 = 0; c0 < D; c0 += 32) {
            uint32_t oa[32];
            ptx::tmem_ld32(o_addr + c0, oa);
            ptx::tmem_ld_wait();
            if (out_row != nullptr) {
                uint32_t pk[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    __nv_bfloat162 h = __floats2bfloat162_rn(fmaf(__uint_as_float(oa[2 * j]), wown, 0.f) * inv,
                                                             fmaf(__uint_as_float(oa[2 * j + 1]), wown, 0.f) * inv);
                    pk[j] = *reinterpret_cast<uint32_t*>(&h);
                }
                uint4* dst = reinterpret_cast<uint4*>(out_row + c0);
#pragma unroll
                for (int j = 0; j < 4; ++j) dst[j] = make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
            }
        }
    } else if (own_pos == 0) {
        // a = own w0, then each later piece in order: one round per remote piece
        tail_round<D, D, 1>(o_addr, 0, src[1], nullptr, wo[1], 0.f, false, true, wown, n_pc == 2, inv, r, out_row);
        if (n_pc == 3)
            tail_round<D, D, 1>(o_addr, 0, src[2], nullptr, wo[2], 0.f, false, false, wown, true, inv, r, out_row);
    } else if (own_pos == 1) {
        tail_round<D, D, 1>(o_addr, 0, src[0], nullptr, wo[0], 0.f, true, false, wown, n_pc == 2, inv, r, out_row);
        if (n_pc == 3)
            tail_round<D, D, 1>(o_addr, 0, src[2], nullptr, wo[2], 0.f, false, false, wown, true, inv, r, out_row);
    } else {  // own last of three: both remotes first, half the columns per round
#pragma unroll 1
        for (int cb = 0; cb < D; cb += D / 2)
            tail_round<D, D / 2, 2>(o_addr, cb, src[0], src[1], wo[0], wo[1], true, false, wown, true, inv, r,
                                    out_row);
    }
    if (lse_out != nullptr) *lse_out = (M + __log2f(Ltot)) * 0.6931471805599453f;
}

// Partial-result slot of a tail piece: e = 0 for a CTA's first tail piece, 1 for its last.
template <int NQ>
__device__ __forceinline__ int tail_slot(int cta, int e, int grp) {
    return NQ == 1 ? 2 * cta + e : 4 * cta + 2 * e + grp;
}

// CS = thread-block cluster size (NQ = 1 only): the CS CTAs of a cluster take the
// CS q-tiles of one (request, kv head) unit and share its K/V stream -- each K or
// V tile is fetched by ONE of them (round robin over the tile's two operands) and
// multicast into all CS shared memories; every CTA releases a ring slot in all
// CS CTAs (DESIGN.md §5 "Clusters").
//
// PR = CTA pair (CS = 2, D = 128): the pair's q-tile j of CTA 0 and q-tile j of
// CTA 1 form ONE M = 256 tcgen05.mma.cta_group::2 issued by the leader (rank 0);
// each CTA loads only its half of every K tile (32 keys) and V tile (its d-chunk)
// -- half the TMA work and shared-memory traffic per CTA.  The peer's loads land
// on its own barriers; its warp 1 forwards each landing to the leader (after
// zeroing V rows past the valid keys of its half); the leader's MMA commits are
// multicast to both CTAs, and both CTAs' softmax warps arrive on the leader's
// p_full / o_empty barriers (DESIGN.md §5 "CTA pairs").
template <int D, int NQ, int CS, bool PR = false>
__global__ void __launch_bounds__(TcCfg<NQ>::THREADS, TcCfg<NQ>::CTAS)
    tree_attn_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_kc,
                        const __grid_constant__ CUtensorMap tm_vc, const __grid_constant__ CUtensorMap tm_kt,
                        const __grid_constant__ CUtensorMap tm_vt, const TcParams p) {
    static_assert(CS == 1 || CS == 2 || CS == 4, "cluster size");
    static_assert(!PR || (CS == 2 && D == 128), "CTA pairs: clusters of 2, head_dim 128");
    using S = TcSmem<D, NQ, PR>;
    constexpr int NCH = S::NCH;
    constexpr int kKStages = S::KST, kVStages = S::VST;
    constexpr uint16_t kMask = (uint16_t)((1u << CS) - 1);  // every CTA of the cluster
    // cluster coordinates (CS = 1: the CTA itself); the schedule is per cluster
    const int crank = CS > 1 ? (int)ptx::cluster_ctarank() : 0;
    const int cl = (int)blockIdx.x / CS;   // cluster index
    const int ncl = (int)gridDim.x / CS;   // clusters in the grid
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S::OFF_BAR);
    uint64_t* q_full = bars + 0;
    uint64_t* q_empty = bars + 1;
    uint64_t* k_full = bars + 2;
    uint64_t* k_empty = k_full + kKStages;
    uint64_t* v_full = k_empty + kKStages;
    uint64_t* v_empty = v_full + kVStages;
    uint64_t* qbars = v_empty + kVStages;  // per q-tile q: 8 barriers at qbars + 8q
    auto s_full = [&](int q, int b) { return qbars + 8 * q + 0 + b; };   // QK into S buffer b done
    auto p_full = [&](int q, int b) { return qbars + 8 * q + 2 + b; };   // softmax wrote P over S buffer b
    auto pv_done = [&](int q, int b) { return qbars + 8 * q + 4 + b; };  // PV reading buffer b done
    auto o_full = [&](int q) { return qbars + 8 * q + 6; };
    auto o_empty = [&](int q) { return qbars + 8 * q + 7; };
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + S::OFF_TMEM);

    const int warp = warp_id();
    const int lane = lane_id();
    unsigned long long t_entry = 0;  // debug mode 6: the per-CTA timeline starts at kernel entry
    if (kDebug && p.trace != nullptr && threadIdx.x == 0 && p.debug_mode == 6)
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_entry));
    pdl_launch_dependents();

    const bool leader = !PR || crank == 0;  // PR: the CTA that issues the pair's MMAs
    __shared__ int pcnt_s[NQ][2], ocnt_s[NQ];  // CTA pair, peer: softmax group arrival counters
    if (threadIdx.x < NQ) {
        pcnt_s[threadIdx.x][0] = pcnt_s[threadIdx.x][1] = 0;
        ocnt_s[threadIdx.x] = 0;
    }
    if (threadIdx.x == 0) {
        // PR: the leader's full barriers also wait for the peer's forwarded landing
        const int fw = (PR && leader) ? 2 : 1;
        ptx::mbar_init(q_full, fw);
        ptx::mbar_init(q_empty, NQ);  // one commit per MMA warp
        // a ring slot is free once every MMA warp of every CTA of the cluster released it
        // (PR: the leader's MMA warps release both CTAs' slots with multicast commits)
        for (int s = 0; s < kKStages; ++s) {
            ptx::mbar_init(k_full + s, fw);
            ptx::mbar_init(k_empty + s, PR ? NQ : NQ * CS);
        }
        for (int s = 0; s < kVStages; ++s) {
            ptx::mbar_init(v_full + s, fw);
            ptx::mbar_init(v_empty + s, PR ? NQ : NQ * CS);
        }
        for (int q = 0; q < NQ; ++q) {
            for (int b = 0; b < 2; ++b) {
                ptx::mbar_init(s_full(q, b), 1);
                // the q-tile's 4 softmax warps (PR leader: + one arrival forwarded for the peer's 4)
                ptx::mbar_init(p_full(q, b), (PR && leader) ? 5 : 4);
                ptx::mbar_init(pv_done(q, b), 1);
            }
            ptx::mbar_init(o_full(q), 1);
            ptx::mbar_init(o_empty(q), (PR && leader) ? 5 : 4);
        }
        ptx::fence_mbar_init();
        ptx::tma_prefetch(&tm_q);
        ptx::tma_prefetch(&tm_kc);
        ptx::tma_prefetch(&tm_vc);
        ptx::tma_prefetch(&tm_kt);
        ptx::tma_prefetch(&tm_vt);
    }
    if (warp == 1) {
        if (PR) ptx::tmem_alloc_pair(tmem_holder, TcCfg<NQ>::TMEM);
        else ptx::tmem_alloc(tmem_holder, TcCfg<NQ>::TMEM);
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (CS > 1) ptx::cluster_sync();  // peers' barriers initialised before any multicast or remote arrive
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_holder;
    pdl_wait();  // the trees come from the select kernel launched just before
    unsigned long long t_start = 0;
    if (kDebug && p.trace != nullptr && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));

    // ---------------- schedule plan (all threads; K/V rings used as scratch) ----------------
    __shared__ int sk_split;  // split-KV pieces per unit (0: whole units)
    __shared__ long long scan_tmp[33];
    __shared__ int red_tmp[3][16];  // per warp (<= 12 warps)
    RecCursor cur0;
    {
        const int n = p.n_req;
        // per-request prefixes and geometry (K/V rings as scratch)
        long long* pre = reinterpret_cast<long long*>(smem + S::OFF_K);
        long long* preu = pre + S::PLAN_N;
        int4* geo = reinterpret_cast<int4*>(preu + S::PLAN_N);
        const bool can_plan = n <= S::PLAN_N;
        const bool can_split = p.stream_k && can_plan;
        int my_units = 0, my_maxnt = 0, my_minnt = 0x7fffffff;
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            Req r;
            const int off = __ldg(p.tree_offsets + i);
            const int4 g = make_int4(off, __ldg(p.tree_offsets + i + 1) - off, __ldg(p.kv_len + i), 0);
            req_from(p, g.x, g.y, g.z, r);
            if (can_plan) geo[i] = g;
            // device errors carry the caller's request index (chunked launches add req_base)
            if (r.MT == 0 && r.K > AS_MAX_TREE) set_dev_error(p.ws, AS_DEV_TREE_TOO_BIG, p.req_base + i);
            else if (r.MT == 0 && r.K > 0) set_dev_error(p.ws, AS_DEV_ROWS_OVERFLOW, p.req_base + i);
            if (r.MT > 0 && g.z > p.max_pages * p.page_size)
                set_dev_error(p.ws, AS_DEV_PAGE_OVERFLOW, p.req_base + i);
            my_units += p.n_kv * r.MT;
            if (r.MT > 0) {
                my_maxnt = max(my_maxnt, r.nt);
                my_minnt = min(my_minnt, r.nt);
            }
            if (can_plan) {
                pre[i] = (long long)p.n_kv * r.MT * r.nt;
                preu[i] = (long long)p.n_kv * r.MT;
            }
        }
        // block reductions: total units, max unit tiles
        int wu = my_units, wm = my_maxnt, wn = my_minnt;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            wu += __shfl_xor_sync(0xffffffffu, wu, o);
            wm = max(wm, __shfl_xor_sync(0xffffffffu, wm, o));
            wn = min(wn, __shfl_xor_sync(0xffffffffu, wn, o));
        }
        if (lane == 0) {
            red_tmp[0][warp] = wu;
            red_tmp[1][warp] = wm;
            red_tmp[2][warp] = wn;
        }
        __syncthreads();
        if (kDebug && p.trace != nullptr && threadIdx.x == 0 && blockIdx.x < kTraceCtas && p.debug_mode == 6) {
            unsigned long long tn;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tn));
            p.trace[(size_t)(p.trace_cap + blockIdx.x) * 8 + 5] = tn;  // plan: loads + reductions done
        }
        int U = 0, maxnt = 0, minnt = 0x7fffffff;
        for (int k = 0; k < (int)(blockDim.x / 32); ++k) {
            U += red_tmp[0][k];
            maxnt = max(maxnt, red_tmp[1][k]);
            minnt = min(minnt, red_tmp[2][k]);
        }
        const int G = ncl;  // schedule slots = clusters
        long long T = 0;
        if (can_plan) {
            // exclusive scans of pre[] and preu[]: per-thread chunks, then warp and block totals
            for (int pass = 0; pass < 2; ++pass) {
                long long* a = pass == 0 ? pre : preu;
                const int chunk = (n + blockDim.x - 1) / blockDim.x;
                const int lo = threadIdx.x * chunk, hi = min(n, lo + chunk);
                long long loc = 0;
                for (int b = lo; b < hi; ++b) loc += a[b];
                long long inc = loc;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const long long y = __shfl_up_sync(0xffffffffu, inc, o);
                    if ((int)lane >= o) inc += y;
                }
                if (lane == 31) scan_tmp[warp] = inc;
                __syncthreads();
                if (threadIdx.x == 0) {
                    long long acc = 0;
                    for (int k = 0; k < (int)(blockDim.x / 32); ++k) {
                        const long long v = scan_tmp[k];
                        scan_tmp[k] = acc;
                        acc += v;
                    }
                    scan_tmp[32] = acc;
                }
                __syncthreads();
                long long run = scan_tmp[warp] + inc - loc;
                for (int b = lo; b < hi; ++b) {
                    const long long v = a[b];
                    a[b] = run;
                    run += v;
                }
                if (pass == 0) T = scan_tmp[32];
                __syncthreads();
            }
        }
        if (kDebug && p.trace != nullptr && threadIdx.x == 0 && blockIdx.x < kTraceCtas && p.debug_mode == 6) {
            unsigned long long tn;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tn));
            p.trace[(size_t)(p.trace_cap + blockIdx.x) * 8 + 4] = tn;  // plan: scans done
        }
        PieceRec* recs = reinterpret_cast<PieceRec*>(smem + S::OFF_REC);
        __shared__ int s_nrec;
        if (threadIdx.x == 0) {
            // Split-KV when units are at most half the CTAs: unit k's tiles are cut into
            // S = min(kMaxSplit, G / U) contiguous pieces, piece s on CTA k*S + s (one
            // piece per CTA); the CTA finishing a unit's last piece merges the fp32
            // partials (O, m, l).  Otherwise whole units, unit k on CTA k mod G.
            const int Sx = (can_split && U > 0) ? min(kMaxSplit, G / U) : 1;
            sk_split = Sx >= 2 ? Sx : 0;
            s_nrec = -1;
            if (sk_split) {
                s_nrec = 0;
                const int k = cl / Sx, sidx = cl - k * Sx;
                if (k < U) {
                    int lo_b = 0, hi_b = n - 1;  // last i with preu[i] <= k
                    while (lo_b < hi_b) {
                        const int mid = (lo_b + hi_b + 1) >> 1;
                        if (preu[mid] <= k) lo_b = mid; else hi_b = mid - 1;
                    }
                    Req r;
                    req_geo(p, geo, lo_b, r);
                    const int tb = r.nt * sidx / Sx, te = r.nt * (sidx + 1) / Sx;
                    if (te > tb) {
                        recs[0] = PieceRec{lo_b, (int)(k - preu[lo_b]), tb, te, r.off, r.K, r.L, sidx, 0, 0};
                        s_nrec = 1;
                    }
                }
            }
        }
        __syncthreads();
        __shared__ int s_ntail;
        __shared__ int s_geff;  // whole-unit schedule slots (balanced waves)
        if (!sk_split) {
            // Whole units, unit k on CTA k mod G.  Tail stream-K (units > CTAs and the
            // last partial wave more than half full): the W1 = U / G full waves stay
            // whole; the tiles of the R remainder units are cut evenly over all G CTAs
            // (each unit then spans at most 3 CTAs).  Every CTA runs its tail pieces
            // FIRST -- the pieces of a unit finish at about the same time, early, and
            // the last to finish merges them from its TMEM while the other CTAs
            // continue with their whole units (DESIGN.md §5 "Schedule").
            const int W1 = U / G, R = U - W1 * G;
            if (threadIdx.x == 0) {
                int nt_rec = 0;
                // Balanced whole-unit waves (below) for few waves, when they keep every SM busy:
                // W = ceil(U/G) <= 3 units per slot on Geff = ceil(U/W) slots; idle slots are
                // second CTAs of some SMs (c2: 512 units on 256 of 296 slots, 2 each -- no
                // pieces, no merges; measured 105 vs 111 us).  Otherwise tail stream-K: with
                // many waves its piece/merge overhead is amortised (c3, c4: 1-2 % faster), and
                // balanced waves would leave SMs empty (c5: 256 units, 148 one-CTA SMs).
                const int Wv0 = U > 0 ? (U + G - 1) / G : 1;
                const int Geff0 = U > 0 ? (U + Wv0 - 1) / Wv0 : G;
                const bool balanced_ok = Wv0 <= 3 && Geff0 * TcCfg<NQ>::CTAS >= G && p.tail_mode != 2;
                bool tail = p.stream_k && can_plan && W1 >= 1 && 2 * R > G && W1 + 2 <= kMaxRec && p.tail_mode &&
                            !balanced_ok;
                bool ok = can_plan;
                if (tail) {
                    const long long k0 = (long long)W1 * G;  // first remainder unit
                    int lo_b = 0, hi_b = n - 1;              // last i with preu[i] <= k0
                    while (lo_b < hi_b) {
                        const int mid = (lo_b + hi_b + 1) >> 1;
                        if (preu[mid] <= k0) lo_b = mid; else hi_b = mid - 1;
                    }
                    Req r0;
                    req_geo(p, geo, lo_b, r0);
                    const long long S0 = pre[lo_b] + (k0 - preu[lo_b]) * r0.nt;  // remainder stream start
                    const long long TR = T - S0;
                    // every unit must span at most 3 CTAs (the merger reads at most 2 partials)
                    if ((long long)maxnt * G > 2 * TR) tail = false;
                    const long long a = S0 + TR * cl / G, b = S0 + TR * (cl + 1) / G;
                    long long pos = tail ? a : b;
                    while (pos < b) {
                        if (nt_rec + W1 >= kMaxRec) { ok = false; break; }
                        int lb = 0, hb = n - 1;  // last i with pre[i] <= pos
                        while (lb < hb) {
                            const int mid = (lb + hb + 1) >> 1;
                            if (pre[mid] <= pos) lb = mid; else hb = mid - 1;
                        }
                        Req r;
                        req_geo(p, geo, lb, r);
                        const long long j = (pos - pre[lb]) / r.nt;
                        const long long ustart = pre[lb] + j * r.nt;
                        const int tb = (int)(pos - ustart);
                        const int te = (int)min((long long)r.nt, b - ustart);
                        const int x = (tb == 0 && te == r.nt) ? -1 : (pos == a ? -2 : -3);
                        recs[nt_rec++] = PieceRec{lb, (int)j, tb, te, r.off, r.K, r.L, x, (int)(ustart - S0), (int)TR};
                        pos = ustart + te;
                    }
                }
                // whole units in balanced waves (the first Geff slots; the rest idle)
                const int Geff = (tail || !balanced_ok) ? G : Geff0;
                s_geff = Geff;
                const int n_whole = tail ? W1 : ((U > cl && cl < Geff) ? (U - 1 - cl) / Geff + 1 : 0);
                ok = ok && n_whole <= kMaxRec;
                if (!ok) set_dev_error(p.ws, AS_DEV_TREE_TOO_BIG, -2);
                s_ntail = ok ? nt_rec : 0;
                s_nrec = ok ? nt_rec + n_whole : 0;
            }
            __syncthreads();
        }
        const int nrec_static = (!sk_split && s_nrec > 0) ? s_nrec - s_ntail : 0;
        const int rec_base = (!sk_split && s_nrec > 0) ? s_ntail : 0;
        for (int q = threadIdx.x; q < nrec_static; q += blockDim.x) {
            const long long k = (long long)cl + (long long)q * s_geff;
            int lo_b = 0, hi_b = n - 1;  // last i with preu[i] <= k
            while (lo_b < hi_b) {
                const int mid = (lo_b + hi_b + 1) >> 1;
                if (preu[mid] <= k) lo_b = mid; else hi_b = mid - 1;
            }
            Req r;
            req_geo(p, geo, lo_b, r);
            recs[rec_base + q] = PieceRec{lo_b, (int)(k - preu[lo_b]), 0, r.nt, r.off, r.K, r.L, -1, 0, 0};
        }
        cur0.nrec = s_nrec;
        cur0.q = 0;
        cur0.rec = recs;
        ptx::fence_proxy_async_smem();  // plan scratch (generic writes) is reused by TMA next
        __syncthreads();  // plan scratch (K/V rings) is free again; records are visible
    }
    if (kDebug && p.trace != nullptr && threadIdx.x == 0 && blockIdx.x < kTraceCtas) {
        unsigned long long tn;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tn));
        p.trace[(size_t)(p.trace_cap + blockIdx.x) * 8 + 2] = tn;  // plan done
    }

    constexpr int SM0 = NQ == 2 ? 4 : 1 + NQ;  // first softmax warp
    // setmaxnreg inside the role branches (warpgroup-uniform): in code common to all
    // roles ptxas compiled the whole kernel under the decreased budget
    if constexpr (NQ == 2) {
        if (warp < 4) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegLow));
    }
    if (warp == 0) {
        // ===================== TMA producer (whole warp) =====================
        // K_{t+lead} (lane 0) and V_t (lane 1) are issued by the same
        // instructions, in consumption order.  At each piece start (and every
        // kPtChunk pages) the 32 lanes stage the request's page-table row in
        // shared memory: no global load sits on the per-tile issue path.
        int* pt_s = reinterpret_cast<int*>(smem + S::OFF_PT);
        uint32_t itk = 0, itv = 0, unit_it = 0;
        const uint64_t pol = p.evict_first ? ptx::policy_evict_first() : ptx::policy_evict_normal();
        const int lead = p.k_lead;
        RecCursor sc = cur0;
        Piece pc;
        while (rec_next(p, sc, pc)) {
            const Unit& u = pc.u;
            const int n_pages_u = (u.L + p.page_size - 1) / p.page_size;
            int chunk0 = -1;  // first page index currently staged
            if (lane == 0) {
                // this CTA's q-tiles of the unit: crank*NQ + q (a CTA past the unit's
                // last q-tile only streams and releases K/V for its cluster)
                const int nq_loc = max(0, min(NQ, u.nq - crank * NQ));
                ptx::mbar_wait(q_empty, (unit_it & 1) ^ 1);
                ptx::mbar_arrive_expect_tx(q_full, (uint32_t)(nq_loc * S::Q_BYTES));
                for (int q = 0; q < nq_loc; ++q) {
                    const int node0 = u.off + (u.mt + crank * NQ + q) * (kBM / p.G);
                    ptx::tma_load_4d(smem + S::OFF_Q + q * S::Q_BYTES, &tm_q, q_full, 0, u.g * p.G, node0, 0);
                }
            }
            const int n = pc.te - pc.tb;
            for (int j = 0; j < n + lead; ++j) {
                const int tk = pc.tb + j;         // K tile issued at this step (lane 0)
                const int tv = pc.tb + j - lead;  // V tile issued at this step (lane 1)
                const int tlo = max(tv, pc.tb), thi = min(tk, pc.te - 1);
                if (tlo < u.n_prefix) {  // stage page-table entries covering both tiles (warp-uniform)
                    const int pg_first = tlo * kBN / p.page_size;
                    const int pg_last = (min(min(thi, u.n_prefix - 1) * kBN + kBN, u.L) - 1) / p.page_size;
                    if (chunk0 < 0 || pg_first < chunk0 || pg_last >= chunk0 + kPtChunk) {
                        chunk0 = pg_first;
                        __syncwarp();
                        for (int k = lane; k < kPtChunk && chunk0 + k < n_pages_u; k += 32)
                            pt_s[k] = __ldg(p.page_table + (size_t)u.i * p.max_pages + chunk0 + k);
                        __syncwarp();
                    }
                }
                const bool is_k = lane == 0;
                const int t = is_k ? tk : tv;
                if (lane < 2 && t >= pc.tb && t < pc.te) {
                    const uint32_t myit = is_k ? itk : itv;
                    const int n_st = is_k ? kKStages : kVStages;
                    const int st = myit % n_st;
                    const uint32_t ph = (myit / n_st) & 1;
                    uint64_t* full = (is_k ? k_full : v_full) + st;
                    uint64_t* empty = (is_k ? k_empty : v_empty) + st;
                    unsigned char* dst = smem + (is_k ? S::OFF_K : S::OFF_V) + st * S::KV_BYTES;
                    // cluster: operand 2t (K) / 2t+1 (V) is fetched by CTA (2t + !is_k) % CS and
                    // multicast; every CTA posts the bytes it will receive on its own barrier
                    const bool owner = CS == 1 || PR || (2 * t + (is_k ? 0 : 1)) % CS == crank;
                    if (PR && t < u.n_prefix) {
                        // this CTA's half: K keys [32 rank, 32 rank + 32) of the tile (box {64,
                        // 32, 2 chunks}); V d-chunk rank of all 64 keys (box {64, 64, 1 chunk})
                        const CUtensorMap* tm_c = is_k ? &tm_kc : &tm_vc;
                        const int key0 = t * kBN;
                        const int page = pt_s[key0 / p.page_size - chunk0];
                        const int slot = key0 % p.page_size;
                        if (page < 0 || page >= p.num_pages) set_dev_error(p.ws, AS_DEV_BAD_PAGE, p.req_base + u.i);
                        ptx::mbar_wait(empty, ph ^ 1);
                        AS_TRACE(is_k ? 0 : 1, myit);
                        ptx::mbar_arrive_expect_tx(full, (uint32_t)S::KV_BYTES);
                        if (is_k) ptx::tma_load_5d_hint(dst, tm_c, full, 0, slot + crank * (kBN / 2), 0, u.g, page, pol);
                        else ptx::tma_load_5d_hint(dst, tm_c, full, 0, slot, crank, u.g, page, pol);
                    } else if (PR) {
                        const CUtensorMap* tm_t = is_k ? &tm_kt : &tm_vt;
                        const int row0 = u.off + (t - u.n_prefix) * kBN;
                        ptx::mbar_wait(empty, ph ^ 1);
                        AS_TRACE(is_k ? 0 : 1, myit);
                        ptx::mbar_arrive_expect_tx(full, (uint32_t)S::KV_BYTES);
                        if (is_k) ptx::tma_load_4d(dst, tm_t, full, 0, row0 + crank * (kBN / 2), 0, u.g);
                        else ptx::tma_load_4d(dst, tm_t, full, 0, row0, crank, u.g);
                    } else if (t < u.n_prefix) {
                        const CUtensorMap* tm_c = is_k ? &tm_kc : &tm_vc;
                        const int key0 = t * kBN;
                        const int valid = min(kBN, u.L - key0);
                        const int nbox = (valid + p.box_rows - 1) / p.box_rows;
                        const uint32_t bytes = (uint32_t)(nbox * NCH * p.box_rows * 128);
                        ptx::mbar_wait(empty, ph ^ 1);
                        AS_TRACE(is_k ? 0 : 1, myit);
                        ptx::mbar_arrive_expect_tx(full, bytes);
                        for (int b = 0; owner && b < nbox; ++b) {
                            const int kp = key0 + b * p.box_rows;
                            const int page = pt_s[kp / p.page_size - chunk0];
                            const int slot = kp % p.page_size;
                            // out-of-range pages read as zeros (TMA bounds check); flag them
                            if (page < 0 || page >= p.num_pages) set_dev_error(p.ws, AS_DEV_BAD_PAGE, p.req_base + u.i);
                            if (p.kv_split_d) {
                                if (CS == 1) ptx::tma_load_5d_hint(dst, tm_c, full, 0, slot, 0, u.g, page, pol);
                                else ptx::tma_load_5d_mc(dst, tm_c, full, 0, slot, 0, u.g, page, kMask, pol);
                            } else {
#pragma unroll
                                for (int c = 0; c < NCH; ++c) {
                                    unsigned char* dc = dst + c * kBN * 128 + b * p.box_rows * 128;
                                    if (CS == 1) ptx::tma_load_4d_hint(dc, tm_c, full, c * 64, slot, u.g, page, pol);
                                    else ptx::tma_load_4d_mc(dc, tm_c, full, c * 64, slot, u.g, page, kMask, pol);
                                }
                            }
                        }
                    } else {
                        const CUtensorMap* tm_t = is_k ? &tm_kt : &tm_vt;
                        const int row0 = u.off + (t - u.n_prefix) * kBN;
                        ptx::mbar_wait(empty, ph ^ 1);
                        AS_TRACE(is_k ? 0 : 1, myit);
                        ptx::mbar_arrive_expect_tx(full, (uint32_t)(NCH * kBN * 128));
                        if (CS == 1) ptx::tma_load_4d(dst, tm_t, full, 0, row0, 0, u.g);
                        else if (owner) ptx::tma_load_4d_mc(dst, tm_t, full, 0, row0, 0, u.g, kMask, pol);
                    }
                }
                __syncwarp();
                if (tk < pc.te) ++itk;
                if (tv >= pc.tb && tv < pc.te) ++itv;
            }
            ++unit_it;
        }
        if (CS > 1 && lane < 2) {
            // drain: every CTA of the cluster released every slot's last use, so no
            // remote arrive or multicast write is still in flight to this CTA at exit
            const bool is_k = lane == 0;
            const uint32_t its = is_k ? itk : itv;
            const int n_st = is_k ? kKStages : kVStages;
            for (int st = 0; st < n_st; ++st)
                if (its > (uint32_t)st) {
                    const uint32_t last_use = (its - 1 - st) / n_st;
                    ptx::mbar_wait((is_k ? k_empty : v_empty) + st, last_use & 1);
                }
        }
    } else if (warp <= NQ) {
        // ===================== MMA issuers (warp 1 + q: q-tile q of each unit) =====================
        // Issue order per piece: QK_tb | QK_tb+1 PV_tb | QK_tb+2 PV_tb+1 | ... PV_te-1.
        // S/P buffers alternate with the q-tile's global tile count, so QK_{t+1}
        // overwrites the buffer PV_{t-1} read -- issued after it by this thread,
        // hence executed after it -- and never waits for the softmax; PV_t waits
        // for P_t.  Each q-tile has its own issuing warp, so the two q-tiles of a
        // unit never wait on each other; a K/V slot is free once every MMA warp
        // has released it (a warp whose q-tile the unit lacks releases it at once).
        const int q = warp - 1;
        // PR: M = 256 (this q-tile of both CTAs)
        constexpr uint32_t idesc_qk = ptx::idesc_bf16_f32(PR ? 2 * kBM : kBM, kBN, 0);
        constexpr uint32_t idesc_pv = ptx::idesc_bf16_f32(PR ? 2 * kBM : kBM, D, 1);
        const uint32_t q_base = ptx::smem_u32(smem + S::OFF_Q) + q * S::Q_BYTES;
        const uint32_t k_base = ptx::smem_u32(smem + S::OFF_K);
        const uint32_t v_base = ptx::smem_u32(smem + S::OFF_V);
        const uint32_t tq = tmem + q * S::TM_QT;  // S/P buffers at tq + 64 b, O at tq + 128
        const uint32_t o_col = tq + 128;
        uint32_t k_it = 0, v_it = 0, unit_it = 0, s_it = 0, p_it = 0, o_it = 0;
        RecCursor sc = cur0;
        Piece pc;
        // release of a K/V ring slot: in every CTA of the cluster (each counts all releases)
        auto release = [&](uint64_t* bar, bool after_mma) {
            if (CS == 1) {
                if (after_mma) ptx::mma_commit(bar);
                else ptx::mbar_arrive(bar);
            } else if (after_mma) {
                if (PR) ptx::mma_commit_pair(bar, kMask);
                else ptx::mma_commit_mc(bar, kMask);
            } else {
#pragma unroll
                for (int r2 = 0; r2 < CS; ++r2) ptx::mbar_arrive_remote(bar, (uint32_t)r2);
            }
        };
        // completion signal of the MMAs issued so far: the local barrier (PR: both CTAs')
        auto signal = [&](uint64_t* bar) {
            if (PR) ptx::mma_commit_pair(bar, kMask);
            else ptx::mma_commit(bar);
        };
        auto arrive_all = [&](uint64_t* bar) {  // non-MMA arrival (debug / idle paths)
            if (PR) {
                ptx::mbar_arrive_remote(bar, 0);
                ptx::mbar_arrive_remote(bar, 1);
            } else {
                ptx::mbar_arrive(bar);
            }
        };
        if (PR && !leader) {
            // ---- CTA-pair peer: warp 1 forwards each landing of this CTA's halves to
            // the leader's barrier, in the leader's consumption order (Q; K_tb; K_t+1,
            // V_t ...), zeroing V rows past the valid keys first (see do_pv); warp 2
            // (NQ = 2) forwards the softmax groups' P / O-drained signals: the softmax
            // warps arrive locally (a cluster-scope release costs their issuing thread
            // ~0.5 us per tile, measured) ----
            if (NQ == 2 && q == 1) {
                uint32_t gs[NQ], gu[NQ];
                for (int j = 0; j < NQ; ++j) gs[j] = gu[j] = 0;
                RecCursor sc2 = cur0;
                Piece pc2;
                while (rec_next(p, sc2, pc2)) {
                    const Unit& u = pc2.u;
                    for (int t = pc2.tb; t < pc2.te; ++t)
                        for (int j = 0; j < NQ; ++j) {
                            if (j >= u.nq) continue;  // the pair is inactive (the leader skips it too)
                            const uint32_t b = gs[j] & 1;
                            ptx::mbar_wait(p_full(j, b), (gs[j] >> 1) & 1);
                            if (lane == 0) ptx::mbar_arrive_remote(p_full(j, b), 0);
                            __syncwarp();
                            ++gs[j];
                        }
                    for (int j = 0; j < NQ; ++j) {
                        if (j >= u.nq) continue;
                        ptx::mbar_wait(o_empty(j), gu[j] & 1);
                        if (lane == 0) ptx::mbar_arrive_remote(o_empty(j), 0);
                        __syncwarp();
                        ++gu[j];
                    }
                }
            }
            if (q == 0) {
                uint32_t fk = 0, fv = 0, fu = 0;
                auto fwd_k = [&]() {
                    const int st = fk % kKStages;
                    ptx::mbar_wait(k_full + st, (fk / kKStages) & 1);
                    if (lane == 0) AS_TRACE(0, fk);
                    if (lane == 0) ptx::mbar_arrive_remote(k_full + st, 0);
                    __syncwarp();
                    ++fk;
                };
                auto fwd_v = [&](const Unit& u, int t) {
                    const int st = fv % kVStages;
                    ptx::mbar_wait(v_full + st, (fv / kVStages) & 1);
                    const int valid = t < u.n_prefix ? min(kBN, u.L - t * kBN) : min(kBN, u.K - (t - u.n_prefix) * kBN);
                    if (valid < kBN) {
                        unsigned char* vs = smem + S::OFF_V + st * S::KV_BYTES;
                        for (int x = lane; x < (kBN - valid) * 8; x += 32)
                            reinterpret_cast<uint4*>(vs + valid * 128)[x] = make_uint4(0, 0, 0, 0);
                        ptx::fence_proxy_async_smem();
                    }
                    __syncwarp();
                    if (lane == 0) AS_TRACE(1, fv);
                    if (lane == 0) ptx::mbar_arrive_remote(v_full + st, 0);
                    __syncwarp();
                    ++fv;
                };
                while (rec_next(p, sc, pc)) {
                    const Unit& u = pc.u;
                    ptx::mbar_wait(q_full, fu & 1);
                    if (lane == 0) ptx::mbar_arrive_remote(q_full, 0);
                    __syncwarp();
                    fwd_k();
                    for (int t = pc.tb; t < pc.te; ++t) {
                        if (t + 1 < pc.te) fwd_k();
                        fwd_v(u, t);
                    }
                    ++fu;
                }
            }
        } else while (rec_next(p, sc, pc)) {
            const Unit& u = pc.u;
            const bool mine = crank * NQ + q < u.nq;
            ptx::mbar_wait(q_full, unit_it & 1);
            auto do_qk = [&](int t) {
                const int st = k_it % kKStages;
                ptx::mbar_wait(k_full + st, (k_it / kKStages) & 1);
                if (lane == 0 && q == 0 && !(kDebug && p.debug_mode == 5)) AS_TRACE(2, k_it);
                ptx::tc_fence_after();
                if (lane == 0) {
                    if (!mine || (kDebug && p.debug_mode >= 2 && p.debug_mode < 5)) {
                        if (mine) arrive_all(s_full(q, s_it & 1));
                        release(k_empty + st, false);
                        if (t == pc.te - 1) {
                            if (PR) arrive_all(q_empty);
                            else ptx::mbar_arrive(q_empty);
                        }
                    } else {
                        const uint32_t s_col = tq + (s_it & 1) * 64;
                        if (q == 0 && !(kDebug && p.debug_mode == 5)) AS_TRACE(7, k_it);
#pragma unroll
                        for (int ks = 0; ks < D / 16; ++ks) {
                            const int c = ks >> 2, kk = ks & 3;
                            const uint64_t a = ptx::sw128_desc(q_base + c * kBM * 128 + kk * 32, 0, 1024);
                            const uint64_t b =
                                ptx::sw128_desc(k_base + st * S::KV_BYTES + c * S::KH_ROWS * 128 + kk * 32, 0, 1024);
                            if (PR) ptx::mma_bf16_ss_pair(s_col, a, b, idesc_qk, ks > 0 ? 1u : 0u);
                            else ptx::mma_bf16_ss(s_col, a, b, idesc_qk, ks > 0 ? 1u : 0u);
                        }
                        signal(s_full(q, s_it & 1));
                        release(k_empty + st, true);
                        if (t == pc.te - 1) signal(q_empty);
                    }
                }
                __syncwarp();
                ++k_it;
                if (mine) ++s_it;
            };
            auto do_pv = [&](int t) {
                const int st = v_it % kVStages;
                ptx::mbar_wait(v_full + st, (v_it / kVStages) & 1);
                if (lane == 0 && q == 0 && !(kDebug && p.debug_mode == 5)) AS_TRACE(3, v_it);
                if (!mine) {
                    if (lane == 0) release(v_empty + st, false);
                    __syncwarp();
                    ++v_it;
                    return;
                }
                // zero V rows past the prefix end, and in a tree tile the rows past
                // the request's last node (cache slots >= L, the next request's tree
                // rows or the caller's padding rows may hold NaN; P is 0 there but
                // 0 * NaN = NaN: verification must not depend on them);
                // with two MMA warps both write the same zeros (benign)
                {
                    const int valid = t < u.n_prefix ? min(kBN, u.L - t * kBN)
                                                     : min(kBN, u.K - (t - u.n_prefix) * kBN);
                    if (valid < kBN) {
                        unsigned char* vs = smem + S::OFF_V + st * S::KV_BYTES;
                        const int nvec = (kBN - valid) * 8;  // 16-byte vectors per chunk
                        for (int c = 0; c < (PR ? 1 : NCH); ++c)  // PR: this CTA's d-chunk only
                            for (int x = lane; x < nvec; x += 32)
                                reinterpret_cast<uint4*>(vs + c * kBN * 128 + valid * 128)[x] = make_uint4(0, 0, 0, 0);
                        ptx::fence_proxy_async_smem();
                    }
                }
                const uint32_t pbuf = p_it & 1;
                ptx::mbar_wait(p_full(q, pbuf), (p_it >> 1) & 1);
                if (lane == 0 && q == 0 && !(kDebug && p.debug_mode == 5)) AS_TRACE(4, v_it);
                if (t == pc.tb) ptx::mbar_wait(o_empty(q), (o_it & 1) ^ 1);  // O drained by the last epilogue
                ptx::tc_fence_after();
                __syncwarp();
                if (kDebug && p.debug_mode >= 2 && p.debug_mode < 5) {
                    if (lane == 0) {
                        release(v_empty + st, false);
                        arrive_all(pv_done(q, pbuf));
                    }
                } else if (lane == 0) {
#pragma unroll
                    for (int kk = 0; kk < kBN / 16; ++kk) {
                        // A = P_t: bf16 pairs over the first 32 columns of S buffer pbuf
                        const uint64_t b = ptx::sw128_desc(v_base + st * S::KV_BYTES + kk * 16 * 128, kBN * 128, 1024);
                        if (PR) ptx::mma_bf16_ts_pair(o_col, tq + pbuf * 64 + kk * 8, b, idesc_pv, (t > pc.tb || kk > 0) ? 1u : 0u);
                        else ptx::mma_bf16_ts(o_col, tq + pbuf * 64 + kk * 8, b, idesc_pv, (t > pc.tb || kk > 0) ? 1u : 0u);
                    }
                    release(v_empty + st, true);
                    signal(pv_done(q, pbuf));
                }
                __syncwarp();
                ++v_it;
                ++p_it;
            };
            for (int t = pc.tb; t < pc.te; ++t) {
                do_qk(t);
                if (t > pc.tb) do_pv(t - 1);
            }
            do_pv(pc.te - 1);
            if (mine) {
                if (lane == 0) {
                    if (kDebug && p.debug_mode >= 2 && p.debug_mode < 5) arrive_all(o_full(q));
                    else signal(o_full(q));
                }
                ++o_it;
            }
            __syncwarp();
            ++unit_it;
        }
    } else if (warp >= SM0) {
        // ============ softmax + epilogue (warps SM0 .. : 4 per q-tile) ============
        if constexpr (NQ == 2) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegHigh));
        const int grp = (warp - SM0) >> 2;  // q-tile of the unit this warp group handles
        const int quad = warp & 3;        // TMEM lane quadrant this warp may access
        const int r = quad * 32 + lane;   // Q row in the tile == TMEM lane
        const uint32_t lane_addr = (uint32_t)(quad * 32) << 16;
        const uint32_t sp_addr = tmem + lane_addr + grp * S::TM_QT;  // S/P buffer b at sp_addr + 64 b
        const uint32_t o_addr = sp_addr + 128;
        uint64_t* const of = o_full(grp);
        uint64_t* const oe = o_empty(grp);
        const int gtid = (int)threadIdx.x - 32 * SM0 - 128 * grp;  // 0..127 within the group
        const float sl2 = p.scale_log2;
        // this row's ancestor-or-self bit words, one per 64-node tree tile ([word][row]: conflict-free)
        uint64_t* const anc_s = reinterpret_cast<uint64_t*>(smem + S::OFF_ANC) + grp * kAncWords * kBM + r;
        uint32_t s_cnt = 0, unit_it = 0;
        int tbase = 0;  // CTA-local index of the piece's first tile (trace only)
        RecCursor sc = cur0;
        Piece pc;
        while (rec_next(p, sc, pc)) {
            const Unit& u = pc.u;
            const int qi = crank * NQ + grp;  // this group's q-tile within the unit
            if (PR ? grp >= u.nq : qi >= u.nq) continue;  // the unit has no q-tile (PR: pair) for this group
            if (PR && qi >= u.nq) {
                // CTA pair: the leader's half of this pair exists, ours does not -- keep the
                // barrier protocol (our TMEM rows are computed and ignored), no math, no output
                for (int t = pc.tb; t < pc.te; ++t, ++s_cnt) {
                    const uint32_t b = s_cnt & 1;
                    ptx::mbar_wait(s_full(grp, b), (s_cnt >> 1) & 1);
                    ptx::tc_fence_after();
                    ptx::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) {  // NQ = 2: forwarded by the peer's warp 2; NQ = 1: last warp forwards
                        if (NQ == 2) ptx::mbar_arrive(p_full(grp, b));
                        else peer_group_arrive(&pcnt_s[grp][b], p_full(grp, b));
                    }
                }
                ptx::mbar_wait(of, unit_it & 1);
                ptx::tc_fence_after();
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    if (NQ == 2) ptx::mbar_arrive(oe);
                    else peer_group_arrive(&ocnt_s[grp], oe);
                }
                ++unit_it;
                tbase += pc.te - pc.tb;
                continue;
            }
            const int G = p.G;
            const int rr = (u.mt + qi) * kBM + r;
            const bool row_ok = rr < u.K * G;
            const int node = rr / G;
            const int hh = rr - node * G;
            // ancestor-or-self bit words of this row's node (R15); parents staged in smem
            int* tp_s = reinterpret_cast<int*>(smem + S::OFF_TP) + (grp * 2 + (unit_it & 1)) * AS_MAX_TREE;
            for (int j = gtid; j < u.K; j += 128) tp_s[j] = __ldg(p.tree_parent + u.off + j);
            group_bar(grp);
            {
                static_assert(kAncWords == 4, "ancestor words: four named registers below");
                uint64_t a0 = 0, a1 = 0, a2 = 0, a3 = 0;  // named, not an array: stays in registers
                if (row_ok) {
                    int v = node, steps = 0;
                    for (;;) {
                        const uint64_t bit = 1ull << (v & 63);
                        const int wv = v >> 6;
                        a0 |= wv == 0 ? bit : 0ull;
                        a1 |= wv == 1 ? bit : 0ull;
                        a2 |= wv == 2 ? bit : 0ull;
                        a3 |= wv == 3 ? bit : 0ull;
                        if (v == 0) break;
                        const int pv = tp_s[v];
                        if (pv < 0 || pv >= v || ++steps > u.K) {
                            set_dev_error(p.ws, AS_DEV_BAD_PARENT, p.req_base + u.i);
                            break;
                        }
                        v = pv;
                    }
                }
                anc_s[0 * kBM] = a0;
                anc_s[1 * kBM] = a1;
                anc_s[2 * kBM] = a2;
                anc_s[3 * kBM] = a3;
            }
            float m_ref = -INFINITY, l_sum = 0.f;
            for (int t = pc.tb; t < pc.te; ++t, ++s_cnt) {
                const uint32_t b = s_cnt & 1;
                const uint32_t s_addr = sp_addr + b * 64;
                ptx::mbar_wait(s_full(grp, b), (s_cnt >> 1) & 1);
                if (lane == 0 && quad == 0 && grp == 0) AS_TRACE(5, tbase + t - pc.tb);
                if (kDebug && t == pc.tb && p.trace != nullptr && gtid == 0 && grp == 0 && blockIdx.x < kTraceCtas) {
                    unsigned long long tn;
                    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tn));
                    p.trace[(size_t)(p.trace_cap + blockIdx.x) * 8 + 6] = tn;  // first S tile seen
                }
                ptx::tc_fence_after();
                uint32_t sr[kBN];
                ptx::tmem_ld32(s_addr, *reinterpret_cast<uint32_t(*)[32]>(&sr[0]));
                ptx::tmem_ld32(s_addr + 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[32]));
                ptx::tmem_ld_wait();
                if (kDebug && p.debug_mode == 5 && lane == 0 && quad == 0 && grp == 0) AS_TRACE(2, tbase + t - pc.tb);
                if (kDebug && p.debug_mode >= 1 && p.debug_mode < 5) {  // timing experiment: no softmax math
                    ptx::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) {
                        if (leader) ptx::mbar_arrive(p_full(grp, b));
                        else if (NQ == 2) ptx::mbar_arrive(p_full(grp, b));
                        else peer_group_arrive(&pcnt_s[grp][b], p_full(grp, b));
                    }
                    continue;
                }
                float* x = reinterpret_cast<float*>(sr);
                if (t < u.n_prefix) {
                    const int valid = u.L - t * kBN;
                    if (valid < kBN) {
#pragma unroll
                        for (int c = 0; c < kBN; ++c) x[c] = (c < valid) ? x[c] : -INFINITY;
                    }
                } else {
                    const uint64_t bits = anc_s[(t - u.n_prefix) * kBM];
#pragma unroll
                    for (int c = 0; c < kBN; ++c) x[c] = ((bits >> c) & 1ull) ? x[c] : -INFINITY;
                }
                // tree max of the raw scores (sm_scale > 0 commutes with max)
                // 3-input max (FMNMX3): 32 instructions for the 64 scores instead of 63
                float mx[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) mx[j] = ptx::max3(x[j], x[j + 8], x[j + 16]);
#pragma unroll
                for (int j = 0; j < 8; ++j) mx[j] = ptx::max3(mx[j], x[j + 24], x[j + 32]);
#pragma unroll
                for (int j = 0; j < 8; ++j) mx[j] = ptx::max3(mx[j], x[j + 40], x[j + 48]);
#pragma unroll
                for (int j = 0; j < 8; ++j) mx[j] = fmaxf(mx[j], x[j + 56]);
                const float tmax = ptx::max3(ptx::max3(mx[0], mx[1], mx[2]), ptx::max3(mx[3], mx[4], mx[5]),
                                             fmaxf(mx[6], mx[7])) * sl2;
                const float m_new = fmaxf(m_ref, tmax);
                if (kDebug && p.debug_mode == 5 && lane == 0 && quad == 0 && grp == 0) AS_TRACE(3, tbase + t - pc.tb);
                if (t > pc.tb) {
                    const bool need = m_new > m_ref + kRescaleThresh;
                    if (__any_sync(0xffffffffu, need)) {
                        // O must be stable: PV_{t-1} (read the other buffer) completed
                        ptx::mbar_wait(pv_done(grp, b ^ 1), ((s_cnt - 1) >> 1) & 1);
                        ptx::tc_fence_after();
                        const float sc2 = need ? ptx::ex2(m_ref - m_new) : 1.f;
#pragma unroll
                        for (int c0 = 0; c0 < D; c0 += 32) {
                            uint32_t o[32];
                            ptx::tmem_ld32(o_addr + c0, o);
                            ptx::tmem_ld_wait();
#pragma unroll
                            for (int j = 0; j < 32; ++j) o[j] = __float_as_uint(__uint_as_float(o[j]) * sc2);
                            ptx::tmem_st32(o_addr + c0, o);
                        }
                        ptx::tmem_st_wait();
                        if (need) {
                            l_sum *= sc2;
                            m_ref = m_new;
                        }
                    }
                } else {
                    m_ref = m_new;
                }
                const float neg_m = (m_ref == -INFINITY) ? 0.f : -m_ref;
                // the softmax warps are issue-bound (two groups per SM): scale/shift and the
                // row sum run as packed f32x2 FFMA2 / FADD2, two columns per instruction
                // (moving a quarter of the ex2 off MUFU onto a polynomial measured 15 % slower)
                const uint64_t s2 = ptx::f2pack(sl2, sl2), nm2 = ptx::f2pack(neg_m, neg_m);
                uint64_t rsa = 0ull, rsb = 0ull;  // packed (even, odd) column partial sums
                uint32_t pk[kBN / 2];
#pragma unroll
                for (int c = 0; c < kBN; c += 2) {
                    const uint64_t y = ptx::ffma2(ptx::f2pack(x[c], x[c + 1]), s2, nm2);
                    const float p0 = ptx::ex2(ptx::f2lo(y));
                    const float p1 = ptx::ex2(ptx::f2hi(y));
                    if ((c >> 1) & 1) rsb = ptx::fadd2(rsb, ptx::f2pack(p0, p1));
                    else rsa = ptx::fadd2(rsa, ptx::f2pack(p0, p1));
                    __nv_bfloat162 h2 = __floats2bfloat162_rn(p0, p1);
                    pk[c >> 1] = *reinterpret_cast<uint32_t*>(&h2);
                }
                rsa = ptx::fadd2(rsa, rsb);
                l_sum += ptx::f2lo(rsa) + ptx::f2hi(rsa);
                if (kDebug && p.debug_mode == 5 && lane == 0 && quad == 0 && grp == 0) AS_TRACE(4, tbase + t - pc.tb);
                // P_t over the first 32 columns of S_t's buffer (S_t already in registers)
                ptx::tmem_st32(s_addr, *reinterpret_cast<uint32_t(*)[32]>(&pk[0]));
                ptx::tmem_st_wait();
                if (kDebug && p.debug_mode == 5 && lane == 0 && quad == 0 && grp == 0) AS_TRACE(7, tbase + t - pc.tb);
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) {  // PR: the leader's barrier counts both CTAs' warps
                    if (leader) ptx::mbar_arrive(p_full(grp, b));
                    else if (NQ == 2) ptx::mbar_arrive(p_full(grp, b));
                    else peer_group_arrive(&pcnt_s[grp][b], p_full(grp, b));
                }
                if (lane == 0 && quad == 0 && grp == 0) AS_TRACE(6, tbase + t - pc.tb);
            }
            // ---- epilogue ----
            AS_EPI_TRACE(0, unit_it);  // last P written
            ptx::mbar_wait(of, unit_it & 1);
            ptx::tc_fence_after();
            AS_EPI_TRACE(1, unit_it);  // O complete
            if (kDebug && p.trace != nullptr && gtid == 0 && grp == 0 && blockIdx.x < kTraceCtas) {
                unsigned long long tn;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tn));
                p.trace[(size_t)(p.trace_cap + blockIdx.x) * 8 + 7] = tn;  // O of the (last) piece ready
            }
            const bool full = (pc.tb == 0 && pc.te == u.nt);
            const bool tailp = !full && pc.x <= -2;  // tail stream-K piece (else co-resident split-KV)
            const int lead_warp = SM0 + 4 * grp;  // first softmax warp of this group
            const int wq = pc.w + qi;                // counters of this q-tile
            const size_t orow = (size_t)(u.off + node) * p.n_q + (size_t)u.g * G + hh;
            __shared__ int s_merge[NQ];
            bool merge_now = false;
            if (tailp) {
                // every other piece already published (their counts are in): merge straight
                // from this piece's TMEM and publish nothing
                if (warp == lead_warp && lane == 0)
                    s_merge[grp] = *reinterpret_cast<volatile int*>(p.cnt + wq) + (pc.te - pc.tb) == u.nt;
                group_bar(grp);
                merge_now = s_merge[grp] != 0;
                group_bar(grp);
            }
            if (!merge_now) {
                const float inv = full ? 1.f / l_sum : 1.f;  // partial piece: keep (O, m, l) unnormalised
                // co-resident split-KV: one piece per CTA, one slot per q-tile; tail: tail_slot()
                const int slot = tailp ? tail_slot<NQ>((int)blockIdx.x, -2 - pc.x, grp) : 2 * (int)blockIdx.x + grp;
                float* part = p.partial + (size_t)slot * p.slot_floats;  // O as [D/4][128] float4, then m[128], l[128]
                if (full) {
                    // output row: 64 columns per TMEM round trip (two loads, one wait), bf16,
                    // 32-byte stores (full L2 sectors; the row is contiguous, 2*D bytes)
#pragma unroll
                    for (int c0 = 0; c0 < D; c0 += 64) {
                        uint32_t oa[64];
                        ptx::tmem_ld32(o_addr + c0, *reinterpret_cast<uint32_t(*)[32]>(&oa[0]));
                        ptx::tmem_ld32(o_addr + c0 + 32, *reinterpret_cast<uint32_t(*)[32]>(&oa[32]));
                        ptx::tmem_ld_wait();
                        if (row_ok) {
                            uint32_t pkk[32];
#pragma unroll
                            for (int j = 0; j < 32; ++j) {
                                __nv_bfloat162 h2 = __floats2bfloat162_rn(__uint_as_float(oa[2 * j]) * inv,
                                                                          __uint_as_float(oa[2 * j + 1]) * inv);
                                pkk[j] = *reinterpret_cast<uint32_t*>(&h2);
                            }
                            unsigned char* dst = reinterpret_cast<unsigned char*>(p.out + orow * D + c0);
#pragma unroll
                            for (int j = 0; j < 4; ++j) ptx::st_global_v8(dst + 32 * j, &pkk[8 * j]);
                        }
                    }
                } else {
#pragma unroll
                    for (int c0 = 0; c0 < D; c0 += 32) {
                        uint32_t oa[32];
                        ptx::tmem_ld32(o_addr + c0, oa);
                        ptx::tmem_ld_wait();
                        // column-quad-major [D/4][128] float4: a warp's store is 512 contiguous bytes
                        float4* dst = reinterpret_cast<float4*>(part) + (c0 / 4) * 128 + r;
#pragma unroll
                        for (int j = 0; j < 8; ++j)
                            dst[j * 128] = make_float4(__uint_as_float(oa[4 * j]), __uint_as_float(oa[4 * j + 1]),
                                                       __uint_as_float(oa[4 * j + 2]), __uint_as_float(oa[4 * j + 3]));
                    }
                }
                if (full && row_ok && p.lse) p.lse[orow] = (m_ref + __log2f(l_sum)) * 0.6931471805599453f;
                if (!full) {
                    part[128 * D + r] = m_ref;
                    part[128 * D + 128 + r] = l_sum;
                }
                AS_EPI_TRACE(2, unit_it);  // O stored (partial or output)
                if (tailp) {
                    // publish, then count this piece's tiles in; the piece completing the count merges
                    __threadfence();
                    AS_EPI_TRACE(3, unit_it);  // partial visible
                    group_bar(grp);
                    if (warp == lead_warp && lane == 0)
                        s_merge[grp] = atomicAdd(p.cnt + wq, pc.te - pc.tb) + (pc.te - pc.tb) == u.nt;
                    group_bar(grp);
                    merge_now = s_merge[grp] != 0;
                    group_bar(grp);
                }
            }
            AS_EPI_TRACE(4, unit_it);  // published / merge decided
            if (merge_now) {
                __threadfence();  // the other pieces' partials, published before their counts
                // the unit's pieces: the CTAs whose remainder-stream ranges [tr*c/G, tr*(c+1)/G)
                // meet [x0, x0 + nt); a CTA's piece is its first (e = 0) unless the unit starts
                // strictly inside that CTA's range (then it is its last, e = 1)
                const long long Gd = ncl, tr = pc.tr;  // the partition is over clusters
                auto start = [&](long long c) { return tr * c / Gd; };
                auto cta_of = [&](long long x) {
                    long long c = x * Gd / (tr > 0 ? tr : 1);
                    while (c + 1 < Gd && start(c + 1) <= x) ++c;
                    while (c > 0 && start(c) > x) --c;
                    return c;
                };
                const long long cA = cta_of(pc.x0), cB = cta_of((long long)pc.x0 + u.nt - 1);
                int slots[3] = {0, 0, 0}, n_pc = 0, own_pos = 0;  // the unit's pieces in stream order
                for (long long c = cA; c <= cB && n_pc < 3; ++c) {
                    const int e = (c > cA || start(cA) == pc.x0) ? 0 : 1;
                    if (c == (long long)cl) own_pos = n_pc;
                    slots[n_pc++] = tail_slot<NQ>((int)c * CS + crank, e, grp);  // same rank in cluster c
                }
                tail_merge<D>(o_addr, m_ref, l_sum, p.partial, p.slot_floats, n_pc, own_pos, slots[0], slots[1],
                              slots[2], r, row_ok ? p.out + orow * D : nullptr,
                              (row_ok && p.lse != nullptr) ? p.lse + orow : nullptr);
                if (warp == lead_warp && lane == 0) p.cnt[wq] = 0;  // last user of the counter this launch
                if (kDebug && p.trace != nullptr && gtid == 0 && grp == 0 && blockIdx.x < kTraceCtas) {
                    unsigned long long tn;
                    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tn));
                    p.trace[(size_t)(p.trace_cap + blockIdx.x) * 8 + 4] = tn;  // tail merge done
                }
            }
            AS_EPI_TRACE(5, unit_it);  // merge done (or nothing)
            AS_EPI_TRACE(6, unit_it + (merge_now ? 1000 : 0) * 0);
            if (kDebug && p.trace != nullptr && blockIdx.x == 0 && gtid == 0 && grp == 0 && unit_it < 64)
                p.trace[(size_t)(3000 + unit_it) * 8 + 7] = (unsigned long long)((merge_now ? 2 : 0) + (tailp ? 1 : 0) + (full ? 4 : 0));
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (leader) ptx::mbar_arrive(oe);
                else if (NQ == 2) ptx::mbar_arrive(oe);
                else peer_group_arrive(&ocnt_s[grp], oe);
            }
            if (kDebug && !full && p.trace != nullptr && gtid == 0 && grp == 0 && blockIdx.x < kTraceCtas) {
                unsigned long long tn;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tn));
                p.trace[(size_t)(p.trace_cap + blockIdx.x) * 8 + 5] = tn;  // partial written
            }
            if (!full && !tailp) {
                // split-KV merge, shared by the unit's pieces: once every piece has
                // published its fp32 (O, m, l), piece CTA s merges its share of the
                // columns for all rows (all pieces of a unit are co-resident: one piece
                // per CTA of a persistent grid), so no CTA merges a whole unit alone.
                const int Sx = sk_split;
                const int sidx = cl % Sx;
                const int b0 = cl - sidx;  // cluster of the unit's piece 0; piece s2 on cluster b0 + s2
                auto live = [&](int s2) { return u.nt * (s2 + 1) / Sx > u.nt * s2 / Sx; };
                int n_live = 0, my_rank = 0;
                for (int s2 = 0; s2 < Sx; ++s2)
                    if (live(s2)) {
                        if (s2 < sidx) ++my_rank;
                        ++n_live;
                    }
                __threadfence();
                group_bar(grp);
                if (warp == lead_warp && lane == 0) {
                    atomicAdd(p.cnt + wq, pc.te - pc.tb);
                    // the unit's pieces are co-resident by construction (one per CTA of a grid
                    // sized to the device); if another tenant (MPS, a concurrent kernel) holds
                    // SMs they may not be -- give up after 0.5 s with a device error instead
                    // of hanging (a cooperative launch is not capturable with PDL edges)
                    unsigned long long t0w, tw;
                    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0w));
                    while (*reinterpret_cast<volatile int*>(p.cnt + wq) < u.nt) {
                        __nanosleep(64);
                        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tw));
                        if (tw - t0w > 500000000ull) {
                            set_dev_error(p.ws, AS_DEV_NOT_RESIDENT, p.req_base + u.i);
                            break;
                        }
                    }
                }
                group_bar(grp);
                __threadfence();
                if (kDebug && p.trace != nullptr && gtid == 0 && grp == 0 && blockIdx.x < kTraceCtas) {
                    unsigned long long tn;
                    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tn));
                    p.trace[(size_t)(p.trace_cap + blockIdx.x) * 8 + 3] = tn;  // all pieces published
                }
                split_merge<D>(p.partial + (size_t)(2 * (b0 * CS + crank) + grp) * p.slot_floats,
                               (size_t)2 * CS * p.slot_floats, Sx, u.nt, r,
                               my_rank, n_live, row_ok ? p.out + orow * D : nullptr,
                               (my_rank == 0 && row_ok && p.lse != nullptr) ? p.lse + orow : nullptr);
                if (kDebug && p.trace != nullptr && gtid == 0 && grp == 0 && blockIdx.x < kTraceCtas) {
                    unsigned long long tn;
                    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tn));
                    p.trace[(size_t)(p.trace_cap + blockIdx.x) * 8 + 4] = tn;  // merge done
                }
                // the last piece done reading the partials resets the counters (reusable workspace)
                group_bar(grp);
                if (warp == lead_warp && lane == 0) {
                    if (atomicAdd(p.cnt2 + wq, 1) == n_live - 1) {
                        p.cnt[wq] = 0;
                        p.cnt2[wq] = 0;
                        __threadfence();
                    }
                }
            }
            ++unit_it;
            tbase += pc.te - pc.tb;
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (CS > 1) ptx::cluster_sync();  // no peer still multicasts into, or arrives on, this CTA
    if (warp == 1) {
        ptx::tc_fence_after();
        if (PR) ptx::tmem_dealloc_pair(tmem, TcCfg<NQ>::TMEM);
        else ptx::tmem_dealloc(tmem, TcCfg<NQ>::TMEM);
    }
    if (kDebug && p.trace != nullptr && threadIdx.x == 0 && blockIdx.x < kTraceCtas) {
        // per-CTA timeline (debug): start/end globaltimer, after the CTA-0 tile trace
        unsigned long long t_end;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
        unsigned long long* rec = p.trace + (size_t)(p.trace_cap + blockIdx.x) * 8;
        rec[0] = p.debug_mode == 6 ? t_entry : t_start;
        rec[1] = t_end;
        if (!sk_split) {  // (split-KV uses slot 3 for "all pieces published")
            unsigned smid;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            rec[3] = (1ull << 40) | ((unsigned long long)cur0.nrec << 16) | smid;
        }
    }
}

// ---------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------
template <int D, int NQ, int CS, bool PR = false>
static int launch_shape(const CUtensorMap* maps, const TcParams& p, int grid, cudaStream_t stream) {
    const int smem = TcSmem<D, NQ, PR>::ALLOC;
    if (cudaFuncSetAttribute(tree_attn_tc_kernel<D, NQ, CS, PR>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) !=
        cudaSuccess)
        return -1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(TcCfg<NQ>::THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    cfg.attrs = attr;
    int na = 0;
    if (CS > 1) {
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = CS;
        attr[na].val.clusterDim.y = 1;
        attr[na].val.clusterDim.z = 1;
        ++na;
    }
    na += fill_launch_attrs(attr + na);
    cfg.numAttrs = na;
    if (cudaLaunchKernelEx(&cfg, tree_attn_tc_kernel<D, NQ, CS, PR>, maps[0], maps[1], maps[2], maps[3], maps[4], p) !=
        cudaSuccess)
        return -1;
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

// CTAs of a cluster shape that can be resident at once (the persistent grid and the
// co-resident split-KV pieces need every CTA resident): per device, cached.
template <int D, int NQ, int CS, bool PR = false>
static int resident_ctas(int n_sms) {
    const int want = n_sms * TcCfg<NQ>::CTAS;
    if (CS == 1) return want;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 0;
    static std::mutex mu;
    static int cache[64] = {0};
    std::lock_guard<std::mutex> lk(mu);
    if (cache[dev] == 0) {
        const int smem = TcSmem<D, NQ, PR>::ALLOC;
        if (cudaFuncSetAttribute(tree_attn_tc_kernel<D, NQ, CS, PR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 smem) != cudaSuccess)
            return 0;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(want);
        cfg.blockDim = dim3(TcCfg<NQ>::THREADS);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = CS;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int nc = 0;
        if (cudaOccupancyMaxActiveClusters(&nc, tree_attn_tc_kernel<D, NQ, CS, PR>, &cfg) != cudaSuccess) {
            cudaGetLastError();
            return 0;
        }
        cache[dev] = min(want, nc * CS);
    }
    return cache[dev];
}

int tc_ctas_per_sm() { return kCtasPerSm; }

// p0.nq selects the CTA shape: 1 (one q-tile per CTA, 2 CTAs/SM), 2 (paired q-tiles
// sharing K/V in one CTA, 1 CTA/SM); p0.cs > 1 (with nq 1): clusters of cs one-q-tile
// CTAs sharing each K/V tile fetch by multicast.  Every CTA replays a list of at most
// kMaxRec pieces built in its prologue: batches with more units than kMaxRec * grid
// are verified in request chunks.
int launch_attn_tc(const CUtensorMap* maps, const TcParams& p0, int head_dim, int n_sms, cudaStream_t stream) {
    const int nq = p0.nq == 2 ? 2 : 1;
    const bool pair = p0.pair != 0 && head_dim == 128;  // CTA pairs (cta_group::2); the host checked the shape
    int cs = pair ? 2 : ((nq == 1 && (p0.cs == 2 || p0.cs == 4)) || (nq == 2 && p0.cs == 2)) ? p0.cs : 1;
    int grid_full = n_sms * (nq == 2 ? TcCfg<2>::CTAS : TcCfg<1>::CTAS);
    if (pair) {
        const int res = nq == 2 ? resident_ctas<128, 2, 2, true>(n_sms) : resident_ctas<128, 1, 2, true>(n_sms);
        if (res < 2) return -1;  // (the maps were built for half tiles: no fallback here)
        grid_full = res / 2 * 2;
#ifdef AS_DEBUG
        if (getenv("AS_ATTN_PAIR_GRID")) grid_full = atoi(getenv("AS_ATTN_PAIR_GRID"));  // A/B: force the grid
        if (getenv("AS_ATTN_VERBOSE")) fprintf(stderr, "pair nq=%d resident=%d grid=%d\n", nq, res, grid_full);
#endif
    } else if (cs > 1) {
        const int res = nq == 2 ? (head_dim == 128 ? resident_ctas<128, 2, 2>(n_sms) : resident_ctas<64, 2, 2>(n_sms))
                      : head_dim == 128 ? (cs == 2 ? resident_ctas<128, 1, 2>(n_sms) : resident_ctas<128, 1, 4>(n_sms))
                                        : (cs == 2 ? resident_ctas<64, 1, 2>(n_sms) : resident_ctas<64, 1, 4>(n_sms));
        if (res >= cs) grid_full = res / cs * cs;
        else cs = 1;  // the device cannot co-schedule the cluster shape: same result without it
    }
    const int qpu = nq * cs;  // q-tiles per unit
    const int units_per_req = p0.n_kv * ((p0.mt_max + qpu - 1) / qpu);
    int chunk = units_per_req > 0 ? max(1, kMaxRec * (grid_full / cs) / units_per_req) : p0.n_req;
    // the prologue's schedule plan holds at most PLAN_N requests (prefix sums, geometry)
    const int plan_half = pair ? (nq == 2 ? TcSmem<128, 2, true>::PLAN_N : TcSmem<128, 1, true>::PLAN_N)
                          : head_dim == 128 ? (nq == 2 ? TcSmem<128, 2>::PLAN_N : TcSmem<128, 1>::PLAN_N)
                                            : (nq == 2 ? TcSmem<64, 2>::PLAN_N : TcSmem<64, 1>::PLAN_N);
    chunk = min(chunk, plan_half);
    for (int r0 = 0; r0 < p0.n_req; r0 += chunk) {
        TcParams p = p0;
        p.nq = qpu;
        p.cs = cs;
        p.n_req = min(chunk, p0.n_req - r0);
        p.page_table = p0.page_table + (size_t)r0 * p0.max_pages;
        p.kv_len = p0.kv_len + r0;
        p.tree_offsets = p0.tree_offsets + r0;
        p.req_base = p0.req_base + r0;
        p.n_units = units_per_req * p.n_req;
        int grid = grid_full;
        if (!p.stream_k && p.n_units * cs < grid) grid = p.n_units * cs;
        if (grid <= 0) continue;
        int rc;
        if (pair) {
            rc = nq == 2 ? launch_shape<128, 2, 2, true>(maps, p, grid, stream)
                         : launch_shape<128, 1, 2, true>(maps, p, grid, stream);
        } else if (head_dim == 128) {
            rc = nq == 2 ? (cs == 2 ? launch_shape<128, 2, 2>(maps, p, grid, stream)
                                    : launch_shape<128, 2, 1>(maps, p, grid, stream))
                 : cs == 2 ? launch_shape<128, 1, 2>(maps, p, grid, stream)
                 : cs == 4 ? launch_shape<128, 1, 4>(maps, p, grid, stream)
                           : launch_shape<128, 1, 1>(maps, p, grid, stream);
        } else {
            rc = nq == 2 ? (cs == 2 ? launch_shape<64, 2, 2>(maps, p, grid, stream)
                                    : launch_shape<64, 2, 1>(maps, p, grid, stream))
                 : cs == 2 ? launch_shape<64, 1, 2>(maps, p, grid, stream)
                 : cs == 4 ? launch_shape<64, 1, 4>(maps, p, grid, stream)
                           : launch_shape<64, 1, 1>(maps, p, grid, stream);
        }
        if (rc != 0) return -1;
    }
    return 0;
}

}  // namespace as
