// sample.cu -- NEXT-3(a): as_sample_tokens, one target sample per tree node by
// Gumbel-max (reading R23), the input of the lossless stochastic walk (R13:
// E[accept_len] = sum_v f(v), Thm. 1).
//
// The arithmetic is fixed by R23 so the result is bit-identical to the CPU
// oracle: Philox4x32-10 (key = seed, counter = (t/4, row, offset)), u =
// fl32((x >> 9)*2 + 1) * 2^-24, g = -ln(-ln u) with R23's fp32 logarithm, every
// float operation an explicit round-to-nearest intrinsic (no FMA contraction),
// score = fl(fl(logit * inv_T) + g), argmax with the lowest index on ties.
//
// sample_rows_kernel: one CTA per row; each thread owns 4-token groups (one
// Philox call each), reads the group's logits with one 16-byte (fp32) or 8-byte
// (bf16) load, and keeps its best (score, index); warp then CTA reduction.
// ALU-bound: 10 Philox rounds per 4 tokens, and two logarithms with a division
// each for every token that can still win -- the rest are pruned exactly
// against the row's best score so far (below), which the threads share.
#include "params.cuh"

namespace as {

// The ten round keys (k0 + r*W0, k1 + r*W1) are computed on the host and passed
// as kernel parameters: the XORs read them from the constant bank, no key
// schedule arithmetic in the per-token loop.
struct PhiloxKeys {
    uint32_t k[20];
};

__device__ __forceinline__ void philox4x32_10(uint32_t c[4], const PhiloxKeys& ks) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t lo0 = 0xD2511F53u * c[0], hi0 = __umulhi(0xD2511F53u, c[0]);
        const uint32_t lo1 = 0xCD9E8D57u * c[2], hi1 = __umulhi(0xCD9E8D57u, c[2]);
        const uint32_t n0 = hi1 ^ c[1] ^ ks.k[2 * r], n2 = hi0 ^ c[3] ^ ks.k[2 * r + 1];
        c[0] = n0;
        c[1] = lo1;
        c[2] = n2;
        c[3] = lo0;
    }
}

// R23's logarithm of a positive normal fp32 value.
__device__ __forceinline__ float ln_r23(float x) {
    const uint32_t b = __float_as_uint(x);
    int e = (int)(b >> 23) - 127;
    float m = __uint_as_float((b & 0x7FFFFFu) | 0x3F800000u);
    if (m > __uint_as_float(0x3FB504F3u)) {  // fl32(sqrt 2)
        m = __fmul_rn(m, 0.5f);
        e += 1;
    }
    const float f = __fsub_rn(m, 1.0f);
    const float s = __fdiv_rn(f, __fadd_rn(2.0f, f));
    const float z = __fmul_rn(s, s);
    float p = __fmul_rn(2.0f / 9.0f, z);
    p = __fadd_rn(p, 2.0f / 7.0f);
    p = __fmul_rn(p, z);
    p = __fadd_rn(p, 2.0f / 5.0f);
    p = __fmul_rn(p, z);
    p = __fadd_rn(p, 2.0f / 3.0f);
    p = __fmul_rn(p, z);
    const float t = __fmul_rn(s, p);
    const float ln1p = __fadd_rn(__fmul_rn(2.0f, s), t);
    return __fadd_rn(__fmul_rn((float)e, 0.6931471805599453f), ln1p);
}

__device__ __forceinline__ float gumbel_r23(uint32_t x) {
    const float u = __fmul_rn(__fadd_rn(__fmul_rn((float)(x >> 9), 2.0f), 1.0f), 5.9604644775390625e-08f);  // 2^-24
    return -ln_r23(-ln_r23(u));
}

__device__ __forceinline__ void better_s(float& bv, int& bi, float v, int i) {
    if (v > bv || (v == bv && i < bi)) {
        bv = v;
        bi = i;
    }
}

template <typename T>
__device__ __forceinline__ void load4(const T* r, int t0, int vocab, bool vec, float x[4]);
template <>
__device__ __forceinline__ void load4<float>(const float* r, int t0, int vocab, bool vec, float x[4]) {
    if (vec && t0 + 3 < vocab) {
        const float4 v = __ldcs(reinterpret_cast<const float4*>(r + t0));
        x[0] = v.x;
        x[1] = v.y;
        x[2] = v.z;
        x[3] = v.w;
    } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) x[j] = t0 + j < vocab ? r[t0 + j] : 0.f;
    }
}
template <>
__device__ __forceinline__ void load4<__nv_bfloat16>(const __nv_bfloat16* r, int t0, int vocab, bool vec, float x[4]) {
    if (vec && t0 + 3 < vocab) {
        const uint2 v = __ldcs(reinterpret_cast<const uint2*>(r + t0));
        x[0] = __uint_as_float(v.x << 16);
        x[1] = __uint_as_float(v.x & 0xFFFF0000u);
        x[2] = __uint_as_float(v.y << 16);
        x[3] = __uint_as_float(v.y & 0xFFFF0000u);
    } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) x[j] = t0 + j < vocab ? __bfloat162float(r[t0 + j]) : 0.f;
    }
}

// Exact pruning: a token whose score cannot reach the row's best score so far
// need not have its logarithms evaluated.  For draws in the tier v = x >> 9 <
// kTierV (u <= 1 - 2^-10), g <= g_tier = g(top of the tier) + 1e-3 (the margin
// covers R23's last-ulp non-monotonicity); fl32 addition is monotone, so
// score = fl(s + g) <= fl(s + g_tier), and fl(s + g_tier) < B (a score some
// token of this row already achieved) proves the token is not the argmax.
constexpr uint32_t kTierV = (1u << 23) - (1u << 13);

__device__ __forceinline__ int ord_of(float f) {  // order-preserving float -> int
    const int i = __float_as_int(f);
    return i >= 0 ? i : i ^ 0x7FFFFFFF;
}
__device__ __forceinline__ float float_of_ord(int i) { return __int_as_float(i >= 0 ? i : i ^ 0x7FFFFFFF); }

template <typename T>
__global__ void __launch_bounds__(512, 3) sample_rows_kernel(const T* __restrict__ logits, int n_rows, int vocab,
                                                          float inv_t, const PhiloxKeys ks, uint32_t o0,
                                                          uint32_t o1, int32_t* __restrict__ out, void* ws) {
    __shared__ float sv[16];
    __shared__ int si[16];
    __shared__ int s_best;  // ord_of(best score seen by any thread of this row)
    if (threadIdx.x == 0) s_best = ord_of(-INFINITY);
    __syncthreads();
    pdl_launch_dependents();
    pdl_wait();
    const int row = blockIdx.x;
    if (row >= n_rows) return;
    const T* r = logits + (size_t)row * vocab;
    const bool vec = (reinterpret_cast<uintptr_t>(r) % (4 * sizeof(T))) == 0;
    float bv = -INFINITY;
    int bi = 0x7fffffff;
    bool nan = false;
    const float g_tier = __fadd_rn(gumbel_r23((kTierV - 1u) << 9 | 0x1FFu), 1e-3f);
    const int nblk = (vocab + 3) / 4;
    int published = ord_of(-INFINITY);
    for (int b = threadIdx.x; b < nblk; b += blockDim.x) {
        const int t0 = 4 * b;
        float x[4];
        load4<T>(r, t0, vocab, vec, x);
        uint32_t c[4] = {(uint32_t)b, (uint32_t)row, o0, o1};
        philox4x32_10(c, ks);
        const float B = fmaxf(bv, float_of_ord(*reinterpret_cast<volatile int*>(&s_best)));
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (t0 + j >= vocab) break;
            nan |= (x[j] != x[j]);
            const float sj = __fmul_rn(x[j], inv_t);
            if ((c[j] >> 9) < kTierV && __fadd_rn(sj, g_tier) < B) continue;  // provably below the best
            const float sc = __fadd_rn(sj, gumbel_r23(c[j]));
            better_s(bv, bi, sc, t0 + j);
        }
        if (ord_of(bv) > published) {  // share the bound with the row's other threads
            published = ord_of(bv);
            atomicMax(&s_best, published);
        }
    }
    if (nan) set_dev_error(ws, AS_DEV_NAN_LOGIT, row);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        better_s(bv, bi, ov, oi);
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
        sv[warp] = bv;
        si[warp] = bi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) better_s(bv, bi, sv[w], si[w]);
        out[row] = bi < vocab ? bi : 0;  // a row of -inf logits (inv_t * -inf) draws token 0
    }
}

int launch_sample(const void* logits, int logits_bf16, int n_rows, int vocab, float inv_t, unsigned long long seed,
                  unsigned long long offset, int32_t* out, void* ws, cudaStream_t stream) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(n_rows);
    cfg.blockDim = dim3(512);
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    cfg.attrs = attr;
    cfg.numAttrs = fill_launch_attrs(attr);
    PhiloxKeys ks;
    for (int r = 0; r < 10; ++r) {
        ks.k[2 * r] = (uint32_t)seed + (uint32_t)r * 0x9E3779B9u;
        ks.k[2 * r + 1] = (uint32_t)(seed >> 32) + (uint32_t)r * 0xBB67AE85u;
    }
    const uint32_t o0 = (uint32_t)offset, o1 = (uint32_t)(offset >> 32);
    cudaError_t e;
    if (logits_bf16)
        e = cudaLaunchKernelEx(&cfg, sample_rows_kernel<__nv_bfloat16>, reinterpret_cast<const __nv_bfloat16*>(logits),
                               n_rows, vocab, inv_t, ks, o0, o1, out, ws);
    else
        e = cudaLaunchKernelEx(&cfg, sample_rows_kernel<float>, reinterpret_cast<const float*>(logits), n_rows, vocab,
                               inv_t, ks, o0, o1, out, ws);
    if (e != cudaSuccess) return -1;
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace as
