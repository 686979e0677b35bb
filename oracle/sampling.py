"""NEXT-3(a) oracle: per-node target samples by Gumbel-max (reading R23).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Plain numpy, one step per
line of the specification below, no blocking; shares nothing with the CUDA
path (csrc/sample.cu implements the same specification independently).

The stochastic walk (R13, "tree-based verification ... prior work")
needs one sample t ~ softmax(logits / T) of the target distribution per tree
node; E[accept_len] = sum_v f(v) (Thm. 1) then holds exactly.  So
that the GPU sample can be compared BIT-EXACTLY with this oracle, R23 fixes
the arithmetic:

* Philox4x32-10 (Salmon et al., SC'11): key (seed_lo, seed_hi), counter
  (t // 4, row, offset_lo, offset_hi); word t % 4 is token t's 32-bit draw x.
* u = fl32((x >> 9) * 2 + 1) * 2^-24, exactly representable, in (0, 1).
* ln_f32: x = m 2^e (m in [sqrt(1/2), sqrt 2)), f = m - 1 (exact),
  s = f / (2 + f), z = s^2, ln = e ln2 + 2s + s z (2/3 + z (2/5 + z (2/7 + z 2/9))),
  every operation one IEEE fp32 round-to-nearest (no fused multiply-add).
* g = -ln_f32(-ln_f32(u)) (a standard Gumbel draw);
  score_t = fl32(fl32(logit_t * inv_T) + g_t);
  sample = argmax_t score_t, the lowest t on ties.

Pins (tests/test_oracle_sampling.py): the Random123 known-answer vectors for
Philox4x32-10; ln_f32 against the fp64 logarithm within 3e-7 relative; and a
chi-squared test that the sampler's frequencies follow softmax(logits * inv_T)
(the Gumbel-max theorem) on small vocabularies.
"""
from __future__ import annotations

import numpy as np

_M0 = np.uint64(0xD2511F53)
_M1 = np.uint64(0xCD9E8D57)
_W0 = np.uint64(0x9E3779B9)
_W1 = np.uint64(0xBB67AE85)
_MASK = np.uint64(0xFFFFFFFF)
_F32 = np.float32


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Philox4x32 with 10 rounds; arguments are uint32 arrays (broadcast)."""
    c = [np.asarray(x, np.uint64) & _MASK for x in (c0, c1, c2, c3)]
    k0 = np.asarray(k0, np.uint64) & _MASK
    k1 = np.asarray(k1, np.uint64) & _MASK
    for _ in range(10):
        p0 = _M0 * c[0]
        p1 = _M1 * c[2]
        hi0, lo0 = p0 >> np.uint64(32), p0 & _MASK
        hi1, lo1 = p1 >> np.uint64(32), p1 & _MASK
        c = [hi1 ^ c[1] ^ k0, lo1, hi0 ^ c[3] ^ k1, lo0]
        k0 = (k0 + _W0) & _MASK
        k1 = (k1 + _W1) & _MASK
    return [x.astype(np.uint32) for x in c]


def uniform_from_bits(x):
    """u = fl32((x >> 9) * 2 + 1) * 2^-24 in (0, 1), exact."""
    x = np.asarray(x, np.uint32)
    return ((x >> np.uint32(9)).astype(np.float32) * _F32(2.0) + _F32(1.0)) * _F32(2.0 ** -24)


_SQRT2 = np.array([0x3FB504F3], np.uint32).view(np.float32)[0]  # fl32(sqrt 2)
_LN2 = _F32(0.6931471805599453)
_C3, _C5, _C7, _C9 = _F32(2.0 / 3.0), _F32(2.0 / 5.0), _F32(2.0 / 7.0), _F32(2.0 / 9.0)


def ln_f32(x):
    """R23's fp32 natural logarithm of positive normal fp32 x (array)."""
    x = np.asarray(x, np.float32)
    b = x.view(np.uint32)
    e = (b >> np.uint32(23)).astype(np.int32) - 127
    m = ((b & np.uint32(0x7FFFFF)) | np.uint32(0x3F800000)).view(np.float32)
    big = m > _SQRT2
    m = np.where(big, m * _F32(0.5), m).astype(np.float32)
    e = np.where(big, e + 1, e)
    f = (m - _F32(1.0)).astype(np.float32)
    s = (f / (_F32(2.0) + f)).astype(np.float32)
    z = (s * s).astype(np.float32)
    p = (_C9 * z).astype(np.float32)
    p = (p + _C7).astype(np.float32)
    p = (p * z).astype(np.float32)
    p = (p + _C5).astype(np.float32)
    p = (p * z).astype(np.float32)
    p = (p + _C3).astype(np.float32)
    p = (p * z).astype(np.float32)        # z (2/3 + z (...))
    t = (s * p).astype(np.float32)        # s z (...)
    ln1p = ((_F32(2.0) * s).astype(np.float32) + t).astype(np.float32)
    return ((e.astype(np.float32) * _LN2).astype(np.float32) + ln1p).astype(np.float32)


def gumbel(rows, vocab, seed, offset=0):
    """g[r, t] for rows `rows` (array of row ids) and tokens [0, vocab)."""
    rows = np.asarray(rows, np.int64)
    t = np.arange(vocab, dtype=np.int64)
    blk = (t // 4).astype(np.uint32)[None, :]
    word = (t % 4)[None, :]
    k0, k1 = np.uint32(seed & 0xFFFFFFFF), np.uint32((seed >> 32) & 0xFFFFFFFF)
    o0, o1 = np.uint32(offset & 0xFFFFFFFF), np.uint32((offset >> 32) & 0xFFFFFFFF)
    out = np.empty((len(rows), vocab), np.float32)
    step = max(1, (1 << 22) // max(1, vocab))  # rows per chunk (memory bound only)
    for a in range(0, len(rows), step):
        r = rows[a:a + step].astype(np.uint32)[:, None]
        w = philox4x32_10(blk, r, o0, o1, k0, k1)
        x = np.where(word == 0, w[0], np.where(word == 1, w[1], np.where(word == 2, w[2], w[3])))
        u = uniform_from_bits(x)
        out[a:a + step] = -ln_f32(-ln_f32(u))
    return out


def sample_rows(logits, inv_temperature, seed, offset=0, row_ids=None):
    """One Gumbel-max sample per row of `logits` [rows, vocab] (fp32 values;
    bf16 inputs are converted exactly first).  Returns int32 [rows]."""
    lg = np.asarray(logits, np.float32)
    n, V = lg.shape
    rows = np.arange(n) if row_ids is None else np.asarray(row_ids)
    g = gumbel(rows, V, seed, offset)
    score = ((lg * _F32(inv_temperature)).astype(np.float32) + g).astype(np.float32)
    return np.argmax(score, axis=1).astype(np.int32)  # first maximum = lowest index on ties
