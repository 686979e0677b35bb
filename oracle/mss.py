"""NEXT-3(b) oracle: SpecInfer multi-step speculative sampling (reading R25).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Plain Python/numpy, one
step per line of the specification below, no blocking; shares nothing with
the CUDA path (csrc/mss.cu implements the same specification independently).

PAPER.md leaves the acceptance rule to "tree-based verification ... prior
work" (Step 4) -- for a stochastic (sampling) target that prior work is
SpecInfer's multi-step speculative sampling (MSS).  Reading R25 fixes it:

At every tree node u (in any order -- each node's outcome depends only on its
own inputs), with children c_1 < ... < c_k (local index order) whose draft
tokens x_j were drawn i.i.d. from the draft distribution q_u = draft_probs[u]
(SpecInfer's stochastic speculation), target distribution p_u =
target_probs[u] (both over the vocabulary, fp32 inputs, computed in fp64):

  p~ = p_u;  N = sum_v p~(v)                       (the residual and its mass)
  for j = 1..k:
      accept c_j  iff  p~(x_j) > 0  and  r_{c_j} * N * q_u(x_j) <= p~(x_j)
                       (r ~ U(0,1] is child c_j's own uniform: "r <= p(x)/q(x)")
      if accepted: u emits x_j (the walk moves to c_j) and stops trying
      else:        p~(v) <- max(0, p~(v) - N q_u(v)) for every v, p~(x_j) <- 0
                   (the residual norm(max(0, p - q)); for the rejected token the
                   bound is exact: p~(x_j) < r N q(x_j) <= N q(x_j)),
                   N <- sum_v p~(v); if N == 0 the residual is empty: stop
                   trying and sample from the previous p~
  if no child was accepted (or u is a leaf): u emits the bonus token
      b = min { v : sum_{w <= v} p~(w) >= r_b(u) * N }   (inverse CDF,
      r_b(u) ~ U(0,1] = bonus_uniforms[u]).

A rejected token has p~ = 0 afterwards, so it can neither be accepted again
nor be the bonus: the emitted token identifies the accepted child uniquely,
and the greedy-token walk of as_accept_tokens (move to the lowest-index child
whose draft token equals the node's emitted token, R13) IS the MSS walk; the
path and the bonus token follow.

Precision: element updates are done in fp64 in the order above; every mass N
is the exactly rounded sum (math.fsum) -- the plain definition of a sum.  The
GPU's fp64 block reductions differ from it only in the last bits, so a
decision can differ only when it sits within ~1e-13 (relative) of its
threshold; `mss_node` reports each decision's relative margin so a parity
test can tell such a tie from an error.

Pins (tests/test_oracle_mss.py): losslessness -- the first emitted token is
distributed as p_root, and the second (given the first was accepted) as
p(.|first), by chi-squared tests over i.i.d.-drafted trees; the single-child
case accepts with probability sum_x min(p(x), q(x)) (Leviathan et al.);
a mutant without the residual update fails the same chi-squared test.
"""
from __future__ import annotations

import math

import numpy as np


def _residual_value(p_v, q_v, v, hist):
    """p~(v) after the rejections in `hist` = [(N_k, x_k), ...], in order."""
    t = float(p_v)
    for n_k, x_k in hist:
        t = 0.0 if v == x_k else max(0.0, t - n_k * float(q_v))
    return t


def _residual_row(p, q, hist):
    return [_residual_value(p[v], q[v], v, hist) for v in range(len(p))]


def mss_node(p, q, child_tokens, child_uniforms, bonus_uniform):
    """MSS at one node (R25).  p, q: fp32 rows [V]; child_tokens / child_uniforms:
    the children's draft tokens and uniforms in local index order.  Returns
    (emitted token, accepted child position or -1, min relative decision margin)."""
    p = np.asarray(p, np.float64)
    q = np.asarray(q, np.float64)
    hist = []
    res = [float(x) for x in p]
    N = math.fsum(res)
    margin = math.inf
    for j, (x, r) in enumerate(zip(child_tokens, child_uniforms)):
        x = int(x)
        lhs = float(np.float32(r)) * N * float(q[x])
        rhs = res[x]
        if rhs > 0.0:
            margin = min(margin, abs(lhs - rhs) / max(abs(lhs), abs(rhs), 1e-300))
        if rhs > 0.0 and lhs <= rhs:
            return x, j, margin
        new_hist = hist + [(N, x)]
        new_res = _residual_row(p, q, new_hist)
        new_N = math.fsum(new_res)
        if new_N == 0.0:
            break
        hist, res, N = new_hist, new_res, new_N
    # bonus: inverse CDF of the residual, in index order
    thr = float(np.float32(bonus_uniform)) * N
    cum = 0.0
    last_pos = 0
    for v, val in enumerate(res):
        if val > 0.0:
            last_pos = v
        cum += val
        if cum >= thr and val > 0.0:
            margin = min(margin, abs(cum - thr) / max(thr, 1e-300), abs(cum - val - thr) / max(thr, 1e-300))
            return v, -1, margin
    return last_pos, -1, margin  # rounding left the threshold unreached: the last token with mass


def mss_tokens(tree_offsets, tree_parent, tree_tokens, target_probs, draft_probs, uniforms, bonus_uniforms):
    """Emitted token per tree node (R25) for every request; also the per-node
    decision margins.  Children of node u: the nodes j > u of its request whose
    parent is u, in index order."""
    to = [int(x) for x in tree_offsets]
    out = np.zeros(to[-1], np.int32)
    margins = np.full(to[-1], math.inf)
    for i in range(len(to) - 1):
        o, K = to[i], to[i + 1] - to[i]
        for u in range(K):
            kids = [c for c in range(u + 1, K) if int(tree_parent[o + c]) == u]
            tok, _, m = mss_node(target_probs[o + u], draft_probs[o + u], [tree_tokens[o + c] for c in kids],
                                 [uniforms[o + c] for c in kids], bonus_uniforms[o + u])
            out[o + u] = tok
            margins[o + u] = m
    return out, margins


def mss_walk(tree_offsets, tree_parent, tree_tokens, target_probs, draft_probs, uniforms, bonus_uniforms, max_path):
    """The MSS acceptance walk (R25 + R14) per request: from the root, run
    mss_node at the current node; an accepted child becomes the next node, else
    the node's emitted token is the bonus and the walk stops.  Returns
    accept_len [n], bonus_token [n], accept_path [n, max_path] (-1 padded; the
    root counts, as in accept_walk), and the minimum decision margin per request."""
    to = [int(x) for x in tree_offsets]
    n = len(to) - 1
    acc_len = np.zeros(n, np.int32)
    bonus = np.zeros(n, np.int32)
    paths = np.full((n, max_path), -1, np.int32)
    margins = np.full(n, math.inf)
    for i in range(n):
        o, K = to[i], to[i + 1] - to[i]
        u, path = 0, [0]
        while True:
            kids = [c for c in range(u + 1, K) if int(tree_parent[o + c]) == u]
            tok, j, m = mss_node(target_probs[o + u], draft_probs[o + u], [tree_tokens[o + c] for c in kids],
                                 [uniforms[o + c] for c in kids], bonus_uniforms[o + u])
            margins[i] = min(margins[i], m)
            if j < 0:
                bonus[i] = tok
                break
            u = kids[j]
            path.append(u)
        acc_len[i] = min(len(path), max_path)
        paths[i, :acc_len[i]] = path[:max_path]
    return {"accept_len": acc_len, "bonus_token": bonus, "accept_path": paths, "margin": margins}
