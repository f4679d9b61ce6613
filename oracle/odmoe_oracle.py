"""Plain, slow, obviously-correct CPU oracle of the OD-MoE decode hot path.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): never imported by the product.

Every function follows a passage of the paper (P:L = /root/reference/PAPER.md line L)
or, where the paper is silent, a reading listed in DESIGN.md §4 (Qn = SURVEY.md §8(c)
reading n). Arithmetic is numpy float64; dot products are numpy matmul (a library
primitive, allowed as a step). No blocking, fusion or reordering.

Parity pins (tests/test_oracle_pins.py, -m "not gpu"):
  rms_norm            pinned: closed form on [3,4]; scale invariance; unit RMS.
  router_logits       pinned: one-hot rows select coordinates; brute force on tiny ints.
  top_k               pinned: SPEC S:80-81 worked examples; brute force over all C(E,k)
                      subsets; constructed ties; expert-permutation equivariance.
  mixture_weights     pinned: k=1 -> 1; k=E -> scipy.special.softmax; sum = 1; hand values.
  expert_ffn          pinned: zero in -> zero out; selector-matrix closed forms that
                      distinguish W1 from W3 and W2 from W2^T; silu(1) constant.
  moe_layer           pinned: identical experts -> y = FFN(u) for any routing; hand example.
  decode_token        pinned: determinism; override neutrality; constructed
                      LM-head argmax ties.
  quantize_int8_rows  pinned: SPEC S:70 example ([1,-0.5] -> codes [127,-64]); half-step
                      bound; zero fixed point.
  round_bf16          pinned: hand values (exact, ties to even, overflow-free carry into the
                      exponent); torch's bf16 cast on random data (a library routine).
  NF4_CODEBOOK        pinned: QLoRA's construction from normal quantiles (nf4_codebook_from_
                      quantiles, scipy.stats.norm) within 2 fp32 ulp; symmetry ends, exact 0.
  quantize_nf4_blocks pinned: brute-force nearest-code search with Python floats; codes of the
                      codebook values themselves map to themselves; midpoint ties; zero blocks;
                      dequantised error <= half the local codebook gap x absmax.
  round_e4m3 / quantize_fp8_rows
                      pinned: torch.float8_e4m3fn casts (library) on random data incl. ties and
                      subnormals; value table endpoints (448, 2^-9); row max -> +-448 exactly.
  rope                pinned: position 0 = identity; norm preserved; relative-position identity
                      <rope(q,m), rope(k,n)> = <rope(q,m+j), rope(k,n+j)>; hd = 2 rotation by pos rad.
  attention_decode    pinned: one position -> v; equal keys -> mean of values; torch's
                      scaled_dot_product_attention (library, GQA by repeat) on random data.
  attn_block          pinned: W_o = 0 -> h unchanged; one position with selector W_v, W_o -> closed form.
  shadow_predict      pinned: same-precision shadow => recall exactly 1.0.
  plan_* / misprediction_reloads / max_load_budget
                      pinned: SPEC examples S:271-273.
  recall_eq2/eq3      pinned: SPEC S:201-202 examples; brute-force triple loop.
  random predictor    pinned: closed form E[recall] = k/E ("recall in Case 5 is only ~25%").
  recall VALUE on random weights: parity unpinned (paper's 99.94/97.34/95.67% are Mixtral +
                      LongWriter values); only the accounting is pinned.
"""
from __future__ import annotations

import math
from fractions import Fraction
from itertools import combinations

import numpy as np

__all__ = [
    "rms_norm", "router_logits", "top_k", "top_k_bruteforce", "mixture_weights", "silu",
    "expert_ffn", "moe_layer", "final_logits", "greedy_argmax", "decode_token", "decode_sequence",
    "quantize_int8_rows", "dequantize_int8_rows", "quantize_model_int8", "shadow_predict",
    "round_bf16", "shadow_model_bf16", "ROPE_THETA", "rope", "attention_decode", "attn_block", "new_cache",
    "decode_token_attn", "NF4_CODEBOOK", "NF4_BLOCK", "nf4_codebook_from_quantiles",
    "quantize_nf4_blocks", "dequantize_nf4_blocks", "quantize_model_nf4", "e4m3_values", "round_e4m3",
    "quantize_fp8_rows", "dequantize_fp8_rows", "quantize_model_fp8",
    "sliced_expert_partials", "near_tie", "tied_run", "ids_excusable", "expected_loads", "shadow_greedy_token", "shadow_decode",
    "plan_group_size", "plan_groups", "assign_layer", "assign_experts",
    "misprediction_reloads", "max_load_budget", "residency_bound", "recall_eq2", "recall_eq3",
    "recall_bruteforce", "prefill_permutation", "prefill_reference", "expert_counts",
]


# ---------------------------------------------------------------- O1 RMSNorm (Q7)
def rms_norm(h, gamma=None, eps: float = 1e-5):
    """u = h * gamma / sqrt(mean(h^2) + eps).

    The paper places "normalization networks" on the main node and in M_l
    but does not print the formula; Mixtral's RMSNorm with eps=1e-5 and gamma=1 is the
    reading Q7. Works on [d] or [m, d].
    """
    h = np.asarray(h, dtype=np.float64)
    ms = np.mean(h * h, axis=-1, keepdims=True)
    u = h / np.sqrt(ms + eps)
    if gamma is not None:
        u = u * np.asarray(gamma, dtype=np.float64)
    return u


# ---------------------------------------------------------------- O2 router logits
def router_logits(w_gate, u):
    """r_e = sum_j W_g[e, j] * u_j  ("the gating network is activated as in a standard MoE
    system to determine expert routing"). w_gate [E, d], u [d] or [m, d]."""
    W = np.asarray(w_gate, dtype=np.float64)
    return np.asarray(u, dtype=np.float64) @ W.T


# ---------------------------------------------------------------- O3 top-k (Q3)
def top_k(r, k: int):
    """Indices of the k largest logits, ordered by (logit descending, index ascending).

    Top-k activation (k=2 for Mixtral); ties go to the lower expert index
    (reading Q3). r is a 1-D array of E logits.
    """
    r = [float(x) for x in np.asarray(r, dtype=np.float64).ravel()]
    order = sorted(range(len(r)), key=lambda e: (-r[e], e))
    return order[:k]


def top_k_bruteforce(r, k: int):
    """Brute force: among all C(E, k) subsets, the one whose sorted logit vector is
    lexicographically largest, ties resolved toward lower indices."""
    r = [float(x) for x in np.asarray(r, dtype=np.float64).ravel()]
    best = None
    for sub in combinations(range(len(r)), k):
        key = sorted(((-r[e], e) for e in sub))
        if best is None or key < best[0]:
            best = (key, sub)
    return [e for _, e in best[0]]


# ---------------------------------------------------------------- O4 mixture weights (Q2)
def mixture_weights(r, S):
    """w_i = exp(r_i - m) / sum_{j in S} exp(r_j - m), m = max_{j in S} r_j.

    The paper does not restate Mixtral's mixture rule; softmax over the k selected logits
    (reading Q2) equals Mixtral's softmax-then-renormalise. Returned in the
    order of S."""
    r = np.asarray(r, dtype=np.float64).ravel()
    sel = np.array([r[i] for i in S], dtype=np.float64)
    m = sel.max()
    e = np.exp(sel - m)
    return e / e.sum()


# ---------------------------------------------------------------- O5 expert FFN (Q1)
def silu(x):
    x = np.asarray(x, dtype=np.float64)
    return x / (1.0 + np.exp(-x))


def expert_ffn(W1, W3, W2, u):
    """Expert computation EC_l: the Mixtral SwiGLU expert (reading Q1):
    g = W1 u, v = W3 u, a = silu(g) * v, y = W2 a.
    W1, W3 [F, d]; W2 [d, F]; u [d]."""
    u = np.asarray(u, dtype=np.float64)
    g = np.asarray(W1, dtype=np.float64) @ u
    v = np.asarray(W3, dtype=np.float64) @ u
    a = silu(g) * v
    return np.asarray(W2, dtype=np.float64) @ a


def sliced_expert_partials(W1, W3, W2, u, n: int):
    """Sliced loading (the B200 generalisation of P:126's "(N_W - k)-fold" I/O
    multiplication): the expert's F intermediate units are split into n contiguous blocks
    B_r = [r F/n, (r+1) F/n); GPU r holds rows B_r of W1 and W3 and columns B_r of W2 and computes
    partial_r = W2[:, B_r] (silu(W1[B_r] u) * (W3[B_r] u)). The F-sum of O5 regrouped: sum_r
    partial_r = expert_ffn(W1, W3, W2, u). Returns the list of n partials [d]."""
    W1 = np.asarray(W1, dtype=np.float64)
    W3 = np.asarray(W3, dtype=np.float64)
    W2 = np.asarray(W2, dtype=np.float64)
    u = np.asarray(u, dtype=np.float64)
    F = W1.shape[0]
    if F % n:
        raise ValueError("F must be divisible by the number of slices")
    out = []
    for r in range(n):
        B = slice(r * F // n, (r + 1) * F // n)
        a = silu(W1[B] @ u) * (W3[B] @ u)
        out.append(W2[:, B] @ a)
    return out


# ---------------------------------------------------------------- O6 one MoE layer
def moe_layer(h, w_gate, experts, k: int, eps: float = 1e-5, u=None, S=None):
    """One decode layer of the MoE block: norm -> gate -> top-k -> weighted expert sum ->
    residual (combine rule S:125; residual in fp32/fp64, reading Q6).

    `experts` maps expert id -> (W1, W3, W2). `u` (teacher forcing of the normalised input)
    and `S` (routing override) are optional. Returns a dict of every intermediate.
    """
    h = np.asarray(h, dtype=np.float64)
    if u is None:
        u = rms_norm(h, eps=eps)
    u = np.asarray(u, dtype=np.float64)
    r = router_logits(w_gate, u)
    sel = top_k(r, k)
    if S is None:
        S = sel
    w = mixture_weights(r, S)
    wmap = {int(e): float(wi) for e, wi in zip(S, w)}
    ys = {}
    y = np.zeros_like(h)
    for e in sorted(int(x) for x in S):  # O6: ascending expert order
        W1, W3, W2 = experts[e]
        ys[e] = wmap[e] * expert_ffn(W1, W3, W2, u)
        y = y + ys[e]
    return dict(u=u, logits=r, S=list(S), topk=sel, w=wmap, y_parts=ys, y=y, h_next=h + y)


# ---------------------------------------------------------------- O7 LM head + greedy
def final_logits(lm_head, h, eps: float = 1e-5):
    """z = W_o RMSNorm(h_L)."""
    return np.asarray(lm_head, dtype=np.float64) @ rms_norm(h, eps=eps)


def greedy_argmax(z):
    """Greedy decoding selects the maximum-likelihood token; ties to the lowest id
    (S:95). np.argmax returns the first maximal index."""
    return int(np.argmax(np.asarray(z, dtype=np.float64)))


def decode_token(weights, token: int, k: int, eps: float = 1e-5, override=None, layers=None):
    """One decode iteration on the hot path (reading Q22: no attention):
    h0 = Emb[t]; for l: h = moe_layer(h); t' = argmax(W_o RMSNorm(h_L)).
    `weights` as produced by inputs.gen_model_weights (stored values). Returns
    (next_token, [per-layer dict])."""
    L = sorted(weights["router"].keys()) if layers is None else layers
    h = np.asarray(weights["emb"][token], dtype=np.float64)
    recs = []
    for li, l in enumerate(L):
        S = None if override is None else override[li]
        out = moe_layer(h, weights["router"][l], weights["experts"][l], k, eps, S=S)
        out["h_in"] = h
        recs.append(out)
        h = out["h_next"]
    z = final_logits(weights["lm_head"], h, eps)
    return greedy_argmax(z), recs, z


def decode_sequence(weights, first_token: int, n_tokens: int, k: int, eps: float = 1e-5):
    """Greedy decode n_tokens starting from first_token; returns (tokens, routing[n][l])."""
    toks, routes, t = [], [], int(first_token)
    for _ in range(n_tokens):
        t_next, recs, _ = decode_token(weights, t, k, eps)
        routes.append([sorted(r["S"]) for r in recs])
        toks.append(t_next)
        t = t_next
    return toks, routes


# ---------------------------------------------------------------- attention block (Q29)
# The paper's main node runs "attention layers ... and normalization networks" of
# Mixtral-8x7B; it prints no formula. Reading Q29: Mixtral's block -- pre-RMSNorm (gamma = 1), GQA
# with H query and Hkv key/value heads of head_dim = d/H, rotary embedding (rotate-half form,
# theta = 1e6), causal softmax(q k^T / sqrt(head_dim)) v, output projection, residual add.
ROPE_THETA = 1.0e6


def rope(x, pos: int, theta: float = ROPE_THETA):
    """Rotary embedding of x [..., hd] at position pos: with half = hd/2, f_i = theta^(-2i/hd),
    a_i = pos * f_i: (x1, x2) -> (x1 cos a - x2 sin a, x2 cos a + x1 sin a) on the two halves."""
    x = np.asarray(x, dtype=np.float64)
    hd = x.shape[-1]
    half = hd // 2
    ang = pos * theta ** (-np.arange(half, dtype=np.float64) * 2.0 / hd)
    c, s = np.cos(ang), np.sin(ang)
    x1, x2 = x[..., :half], x[..., half:]
    return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1)


def attention_decode(q, K, V):
    """One query position against T cached positions (GQA): q [H, hd], K, V [T, Hkv, hd].
    Query head i reads key/value head i // (H / Hkv). o_i = softmax(K_g q_i / sqrt(hd)) V_g."""
    q = np.asarray(q, dtype=np.float64)
    K = np.asarray(K, dtype=np.float64)
    V = np.asarray(V, dtype=np.float64)
    H, hd = q.shape
    rep = H // K.shape[1]
    o = np.zeros((H, hd))
    for i in range(H):
        g = i // rep
        s = K[:, g, :] @ q[i] / math.sqrt(hd)
        p = np.exp(s - np.max(s))
        p /= np.sum(p)
        o[i] = p @ V[:, g, :]
    return o


def attn_block(h, attn_w, heads, cache_l, pos: int, eps: float = 1e-5):
    """h + W_o attention(RMSNorm(h)) at position pos; appends this position's k, v (after RoPE for
    k) to cache_l = {"K": [...], "V": [...]} (positions 0..pos-1 already there). Returns
    (h_out, dict with x, q, k, v, o)."""
    Wq, Wk, Wv, Wo = attn_w
    H, Hkv = heads
    d = Wq.shape[1]
    hd = d // H
    h = np.asarray(h, dtype=np.float64)
    x = rms_norm(h, eps=eps)
    q = rope((np.asarray(Wq, dtype=np.float64) @ x).reshape(H, hd), pos)
    k = rope((np.asarray(Wk, dtype=np.float64) @ x).reshape(Hkv, hd), pos)
    v = (np.asarray(Wv, dtype=np.float64) @ x).reshape(Hkv, hd)
    assert len(cache_l["K"]) == pos
    cache_l["K"].append(k)
    cache_l["V"].append(v)
    o = attention_decode(q, np.stack(cache_l["K"]), np.stack(cache_l["V"]))
    return h + np.asarray(Wo, dtype=np.float64) @ o.reshape(-1), {"x": x, "q": q, "k": k, "v": v, "o": o}


def new_cache(L):
    return {l: {"K": [], "V": []} for l in L}


def decode_token_attn(weights, token: int, pos: int, cache, k: int, eps: float = 1e-5):
    """One decode iteration with the attention block (Q29): h0 = Emb[t]; for l: h = attn_block(h),
    h = moe_layer(h); t' = argmax(LM head). `cache` (new_cache) gains position pos."""
    L = sorted(weights["router"].keys())
    h = np.asarray(weights["emb"][token], dtype=np.float64)
    recs = []
    for l in L:
        h_att, arec = attn_block(h, weights["attn"][l], weights["heads"], cache[l], pos, eps)
        out = moe_layer(h_att, weights["router"][l], weights["experts"][l], k, eps)
        out["h_in"] = h
        out["h_att"] = h_att
        out["attn"] = arec
        recs.append(out)
        h = out["h_next"]
    z = final_logits(weights["lm_head"], h, eps)
    return greedy_argmax(z), recs, z


# ---------------------------------------------------------------- O8 shadow / SEP
def quantize_int8_rows(W):
    """INT8 shadow quantiser (P:86, P:164 name INT8 without a format; reading Q9):
    per output row r, m_r = max_j |W_rj|; q_rj = clamp(RNE((W_rj * 127) / m_r), -127, 127)
    with the product and quotient in fp64; s_r = fl32(m_r / 127) (fp64 quotient rounded to
    fp32). A row with m_r = 0 gives q = 0, s = 1. Generalises SPEC's per-matrix grid
    (S:65): for one row they coincide.
    Returns (q int8 [R, C], s float32 [R])."""
    W = np.asarray(W, dtype=np.float64)
    if W.ndim == 1:
        W = W[None, :]
    m = np.max(np.abs(W), axis=1)
    q = np.zeros(W.shape, dtype=np.int8)
    s = np.ones(W.shape[0], dtype=np.float32)
    nz = m > 0
    quot = (W[nz] * 127.0) / m[nz][:, None]
    q[nz] = np.clip(np.rint(quot), -127, 127).astype(np.int8)  # np.rint = round half to even
    s[nz] = (m[nz] / 127.0).astype(np.float32)
    return q, s


def dequantize_int8_rows(q, s):
    """Q(W)_rj = s_r * q_rj (exact in fp64)."""
    return np.asarray(s, dtype=np.float64)[:, None] * np.asarray(q, dtype=np.float64)


def quantize_model_int8(weights):
    """Q(W) for every matrix of the model: embedding, routers, experts and (when present) the
    LM head, which the shadow needs only to take its own greedy token (cross-token speculation,
    P:188-203). Returns a weights dict of the same structure holding the dequantised fp64 values."""
    dq = lambda W: dequantize_int8_rows(*quantize_int8_rows(W))  # noqa: E731
    out = {"emb": dq(weights["emb"]), "router": {}, "experts": {}}
    if "lm_head" in weights:
        out["lm_head"] = dq(weights["lm_head"])
    for l, Wg in weights["router"].items():
        out["router"][l] = dq(Wg)
        out["experts"][l] = {e: tuple(dq(M) for M in mats) for e, mats in weights["experts"][l].items()}
    return out


def round_bf16(W):
    """Round to the nearest bfloat16, ties to even (IEEE-754 binary32 with the low 16 bits of
    the significand rounded away): the format of the half-precision shadow of an FP32 main
    model (P:86, P:164 use an FP16 shadow; BF16 is the B200 reading Q26).
    The value is first rounded to fp32 (the main model's own precision). Returns fp64."""
    x = np.ascontiguousarray(np.asarray(W, dtype=np.float32))
    u = x.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    u = ((u + 0x7FFF + lsb) & 0xFFFF0000).astype(np.uint32)
    return u.view(np.float32).astype(np.float64)


def shadow_model_bf16(weights):
    """The BF16 shadow (every matrix of the model rounded by round_bf16), same structure."""
    out = {"emb": round_bf16(weights["emb"]), "router": {}, "experts": {}}
    for l, Wg in weights["router"].items():
        out["router"][l] = round_bf16(Wg)
        out["experts"][l] = {e: tuple(round_bf16(M) for M in mats) for e, mats in weights["experts"][l].items()}
    return out


# NF4 codebook, as published with QLoRA (Dettmers et al. 2023, "NormalFloat4"; the table of its
# reference implementation). The paper's third shadow precision (95.67 % recall)
# names NF4 without further detail: reading Q27 takes QLoRA's NF4 with blocks of 64 weights
# along a row and one fp32 absmax per block (no double quantisation).
NF4_CODEBOOK = (
    -1.0, -0.6961928009986877, -0.5250730514526367, -0.39491748809814453,
    -0.28444138169288635, -0.18477343022823334, -0.09105003625154495, 0.0,
    0.07958029955625534, 0.16093020141124725, 0.24611230194568634, 0.33791524171829224,
    0.44070982933044434, 0.5626170039176941, 0.7229568362236023, 1.0,
)
NF4_BLOCK = 64


def nf4_codebook_from_quantiles(offset: float = 0.9677083):
    """NF4's construction (QLoRA §3): 8 positive and 7 negative quantiles of N(0, 1) at evenly
    spaced probabilities from `offset` to 1/2, plus an exact zero, normalised to [-1, 1]."""
    from scipy.stats import norm
    pos = norm.ppf(np.linspace(offset, 0.5, 9)[:-1])
    neg = -norm.ppf(np.linspace(offset, 0.5, 8)[:-1])
    v = np.sort(np.concatenate([pos, [0.0], neg]))
    return v / np.max(np.abs(v))


def quantize_nf4_blocks(W, block: int = NF4_BLOCK):
    """NF4 blockwise quantiser (reading Q27): per block of `block` consecutive weights of a row,
    a = max |w| (exact, stored fp32); x = w / a in fp64; code = index of the codebook entry
    nearest to x (|x - c_i| in fp64, the lower index on an exact tie). a = 0 -> all codes 7
    (the codebook's 0.0). Returns (codes uint8 [R, C] in 0..15, absmax float32 [R, C/block])."""
    W = np.asarray(W, dtype=np.float64)
    if W.ndim == 1:
        W = W[None, :]
    R, C = W.shape
    assert C % block == 0
    cb = np.asarray(NF4_CODEBOOK, dtype=np.float32).astype(np.float64)
    Wb = W.reshape(R, C // block, block)
    a = np.max(np.abs(Wb), axis=2)
    x = np.zeros_like(Wb)
    nz = a > 0
    x[nz] = Wb[nz] / a[nz][:, None]
    dist = np.abs(x[..., None] - cb)                        # [R, nb, block, 16]
    codes = np.argmin(dist, axis=-1).astype(np.uint8)      # argmin returns the first minimum
    codes[~nz] = 7
    return codes.reshape(R, C), a.astype(np.float32)


def dequantize_nf4_blocks(codes, absmax, block: int = NF4_BLOCK):
    """Q(W)_rj = c[code_rj] * a_r,j/block (fp64)."""
    cb = np.asarray(NF4_CODEBOOK, dtype=np.float32).astype(np.float64)
    codes = np.asarray(codes)
    a = np.repeat(np.asarray(absmax, dtype=np.float64), block, axis=1)
    return cb[codes] * a


# ---------------------------------------------------------------- FP8 (E4M3) row shadow (reading Q28)
def e4m3_values():
    """The 127 non-negative finite E4M3 ("fn": no infinities, S.1111.111 = NaN) values in code
    order 0x00..0x7E, from the format: exponent bias 7, 3 mantissa bits, subnormals at e = 0."""
    vals = []
    for e in range(16):
        for m in range(8):
            if e == 15 and m == 7:
                continue
            vals.append(m / 8.0 * 2.0 ** -6 if e == 0 else (1.0 + m / 8.0) * 2.0 ** (e - 7))
    return np.asarray(vals)


def round_e4m3(x):
    """Round to the nearest E4M3 value, ties to the even code, saturating at +-448 (satfinite).
    Returns (values fp64, codes uint8 with the sign in bit 7)."""
    x = np.asarray(x, dtype=np.float64)
    V = e4m3_values()
    a = np.abs(x)
    i = np.clip(np.searchsorted(V, a, side="left"), 1, len(V) - 1)
    lo, hi = V[i - 1], V[i]
    dlo, dhi = a - lo, hi - a
    pick_hi = (dhi < dlo) | ((dhi == dlo) & (i % 2 == 0))
    idx = np.where(pick_hi, i, i - 1)
    idx = np.where(a >= V[-1], len(V) - 1, idx)
    idx = np.where(a == 0, 0, idx)
    neg = np.signbit(x)
    vals = np.where(neg, -V[idx], V[idx])
    codes = (idx | (neg.astype(np.int64) << 7)).astype(np.uint8)
    return vals, codes


def quantize_fp8_rows(W):
    """FP8 row shadow (reading Q28): per row r, m_r = max|w|, s_r = fl32(m_r / 448) (fp64 quotient
    rounded to fp32); x = fl32(w / s_r) (fp64 quotient rounded to fp32); q = E4M3(x) (RNE,
    satfinite). A zero row gives q = 0, s = 1. Returns (codes uint8 [R, C], s float32 [R])."""
    W = np.asarray(W, dtype=np.float64)
    if W.ndim == 1:
        W = W[None, :]
    m = np.max(np.abs(W), axis=1)
    s = np.ones(W.shape[0], dtype=np.float32)
    nz = m > 0
    s[nz] = (m[nz] / 448.0).astype(np.float32)
    x = (W / s.astype(np.float64)[:, None]).astype(np.float32)
    _, codes = round_e4m3(x)
    codes[~nz] = 0
    return codes, s


def dequantize_fp8_rows(codes, s):
    V = e4m3_values()
    codes = np.asarray(codes)
    mag = V[np.minimum(codes & 0x7F, len(V) - 1)]
    val = np.where(codes & 0x80, -mag, mag)
    return np.asarray(s, dtype=np.float64)[:, None] * val


def quantize_model_nf4(weights):
    """The NF4 shadow (reading Q27): every expert matrix NF4-blockwise; the embedding and the
    routers int8-row as in the INT8 shadow (0.3 % of the bytes). Dequantised fp64, same structure."""
    dq8 = lambda W: dequantize_int8_rows(*quantize_int8_rows(W))  # noqa: E731
    dq4 = lambda W: dequantize_nf4_blocks(*quantize_nf4_blocks(W))  # noqa: E731
    out = {"emb": dq8(weights["emb"]), "router": {}, "experts": {}}
    for l, Wg in weights["router"].items():
        out["router"][l] = dq8(Wg)
        out["experts"][l] = {e: tuple(dq4(M) for M in mats) for e, mats in weights["experts"][l].items()}
    return out


def quantize_model_fp8(weights):
    """The FP8 shadow (reading Q28): expert matrices E4M3 row-scaled; embedding and routers
    int8-row as in the INT8 shadow. Dequantised fp64, same structure."""
    dq8 = lambda W: dequantize_int8_rows(*quantize_int8_rows(W))  # noqa: E731
    dqf = lambda W: dequantize_fp8_rows(*quantize_fp8_rows(W))  # noqa: E731
    out = {"emb": dq8(weights["emb"]), "router": {}, "experts": {}}
    for l, Wg in weights["router"].items():
        out["router"][l] = dq8(Wg)
        out["experts"][l] = {e: tuple(dqf(M) for M in mats) for e, mats in weights["experts"][l].items()}
    return out


def shadow_predict(shadow_weights, main_token: int, k: int, eps: float = 1e-5):
    """SEP, Mode A (reading Q10): token alignment every iteration -- the
    shadow starts from ITS OWN embedding row of the MAIN model's token and runs all L layers
    with its own (quantised) weights and its own routing; P[l] = its top-k at layer l
    ("uses the future expert activations that are already unfolded by the scaled-down
    shadow model"). No attention => no KV state, i.e. the paper's T1_KV1 regime.
    Returns (P [L][k] in rank order, per-layer dicts)."""
    L = sorted(shadow_weights["router"].keys())
    h = np.asarray(shadow_weights["emb"][main_token], dtype=np.float64)
    P, recs = [], []
    for l in L:
        out = moe_layer(h, shadow_weights["router"][l], shadow_weights["experts"][l], k, eps)
        out["h_in"] = h
        P.append(out["S"])
        recs.append(out)
        h = out["h_next"]
    return P, recs


def shadow_greedy_token(shadow_weights, h_L, eps: float = 1e-5) -> int:
    """The shadow's own next token: greedy argmax of its quantised LM head on RMSNorm(h_L) (the
    paper's "the quantized model may generate a different token"; lowest id on ties)."""
    return greedy_argmax(final_logits(shadow_weights["lm_head"], h_L, eps))


def shadow_decode(shadow_weights, main_tokens, k: int, period: int, eps: float = 1e-5):
    """SEP with token alignment period T_p ("align the tokens ... once every few
    autoregression iterations"; Fig. 6 T_i; S:165-173 shadow_decode_step). Iteration n (0-based)
    predicts the main model's iteration n, whose input is main_tokens[n]. If n mod T_p == 0 the
    shadow's input is the main token (token alignment); otherwise it is the shadow's OWN greedy
    token from iteration n-1. Each iteration runs all L layers (no attention: no KV state, so only
    the token axis of alignment exists, reading Q22). Returns (P [N][L] lists of k ids in rank
    order, shadow input tokens [N], shadow output tokens [N])."""
    if period < 1:
        raise ValueError("alignment period must be >= 1")
    P, t_in, t_out = [], [], []
    own = None
    for n, tm in enumerate(main_tokens):
        t = int(tm) if (n % period == 0 or own is None) else own
        preds, recs = shadow_predict(shadow_weights, t, k, eps)
        own = shadow_greedy_token(shadow_weights, recs[-1]["h_next"], eps)
        P.append(preds)
        t_in.append(t)
        t_out.append(own)
    return P, t_in, t_out


def near_tie(r, k: int, rel: float = 1e-3) -> bool:
    """North-star excuse window (reading Q4): the oracle's k-th and (k+1)-th largest logits
    differ by less than rel * max(|r_(k)|, |r_(k+1)|); both zero counts as a tie."""
    srt = sorted((float(x) for x in np.asarray(r).ravel()), reverse=True)
    if k >= len(srt):
        return False
    a, b = srt[k - 1], srt[k]
    if a == 0.0 and b == 0.0:
        return True
    return abs(a - b) < rel * max(abs(a), abs(b))


def _close(a: float, b: float, rel: float) -> bool:
    return (a == 0.0 and b == 0.0) or abs(a - b) < rel * max(abs(a), abs(b))


def tied_run(r, k: int, rel: float = 1e-3):
    """The tied run at the selection boundary (reading Q4; SURVEY §8(c) Parity 2): every index whose
    logit lies inside the near-tie window of the k-th largest logit r_(k), i.e.
    |r_e - r_(k)| < rel * max(|r_e|, |r_(k)|) (both zero counts). Contains the k-th itself."""
    r = [float(x) for x in np.asarray(r).ravel()]
    kth = sorted(r, reverse=True)[k - 1]
    return {e for e, x in enumerate(r) if _close(x, kth, rel)}


def ids_excusable(ids, r, k: int, rel: float = 1e-3):
    """Parity protocol 2 (north_star: "Selected expert IDs must match the oracle exactly, except
    where the oracle's k-th and (k+1)-th logits differ by less than 1e-3 relative").
    `ids` (k ids in rank order) is accepted iff
      (a) they are k distinct indices;
      (b) as a set they equal top_k(r, k), or near_tie(r, k) holds and the symmetric difference with
          top_k lies inside tied_run(r, k) (only members of the tied run were swapped);
      (c) the rank order is by descending oracle logit, except between two near-equal logits.
    Returns (ok, excused) with excused = (ids != top_k(r, k))."""
    ids = [int(x) for x in ids]
    ref = top_k(r, k)
    if ids == ref:
        return True, False
    rr = [float(x) for x in np.asarray(r).ravel()]
    if len(set(ids)) != k or any(e < 0 or e >= len(rr) for e in ids):
        return False, True
    diff = set(ids) ^ set(ref)
    if diff and not (near_tie(r, k, rel) and diff <= tied_run(r, k, rel)):
        return False, True
    for a, b in zip(ids, ids[1:]):
        if rr[b] > rr[a] and not _close(rr[a], rr[b], rel):
            return False, True
    return True, True


# ---------------------------------------------------------------- O9 placement
def plan_group_size(k: int, n_gpus: int) -> int:
    """G = k in the paper ("G=2 since a top-2 activation policy"); with fewer GPUs
    than k one GPU takes several experts: G = min(k, N) (reading Q14)."""
    return min(k, n_gpus)


def plan_groups(n_workers: int, G: int):
    """N_W/G groups of G contiguous workers. N_W must be divisible by G."""
    if G <= 0 or n_workers % G != 0:
        raise ValueError("n_workers must be divisible by the group size")
    return [list(range(g * G, (g + 1) * G)) for g in range(n_workers // G)]


def assign_layer(layer: int, n_groups: int) -> int:
    """Round-robin layer -> group (Fig. 2): l mod N_G."""
    return layer % n_groups


def assign_experts(experts, workers):
    """One-to-one expert -> worker: sorted experts paired with sorted workers.
    With fewer workers than experts (G < k), sorted expert i goes to sorted worker
    i * G // k (each worker takes k/G consecutive experts; reading Q14)."""
    ex = sorted(int(e) for e in experts)
    wk = sorted(int(w) for w in workers)
    k, G = len(ex), len(wk)
    if G == 0 or k % G != 0:
        raise ValueError("cardinality mismatch in placement")
    return {e: wk[i * G // k] for i, e in enumerate(ex)}


def misprediction_reloads(true_S, resident):
    """Misprediction fallback ("the expert computation task waits for the completion
    of expert reloading"). `resident` maps expert -> worker for the layer's loaded
    (predicted) experts. Reload set = true \\ resident, placed on the workers holding the
    wrong experts, sorted-paired (reading Q15). Returns sorted [(expert, worker)]."""
    true_S = sorted(int(e) for e in true_S)
    missing = [e for e in true_S if e not in resident]
    stale_workers = sorted(w for e, w in resident.items() if e not in true_S)
    if len(stale_workers) < len(missing):
        raise ValueError("not enough stale workers for the reload set")
    return list(zip(missing, stale_workers[: len(missing)]))


def expected_loads(true_S, issued) -> int:
    r"""Expert loads of one decode token ("minimal I/O bandwidth waste"; "waits for the
    completion of expert reloading"; SURVEY §8(c) "Loader accounting (a6 <-> a12)"). Per layer l the
    loader performs the loads issued from the prediction before the router ran, I_l, and after the
    router the reloads S_l \ I_l (handle_misprediction): |I_l| + |S_l \ I_l| =
    k + |I_l \ S_l|. Summed over layers: L*k + (number of issued loads that were wrong). `true_S`,
    `issued`: per-layer id collections. Bytes = loads x blob bytes."""
    total = 0
    for S, I in zip(true_S, issued):
        S, I = set(int(x) for x in S), set(int(x) for x in I)
        total += len(I) + len(S - I)
    return total


def max_load_budget(t_M: float, t_W: float, n_groups: int) -> float:
    """Eq. 1 with the worked example's reading (4t^M+3t^W at four groups;
    reading Q12): t_maxload = N_G * t_M + (N_G - 1) * t_W."""
    if t_M < 0 or t_W < 0:
        raise ValueError("negative time")
    return n_groups * t_M + (n_groups - 1) * t_W


def residency_bound(lookahead: int, n_groups: int) -> int:
    """Per-worker residency bound ceil(D / N_G) + 1 experts."""
    return -(-lookahead // n_groups) + 1


# ---------------------------------------------------------------- O10 recall (Eqs. 2-3)
def _c_count(true_S, pred_S, avail=True):
    """c(q,n,l) = |true ∩ predicted| in [0, k]; 0 if the prediction was unavailable."""
    if not avail or pred_S is None:
        return 0
    return len(set(int(x) for x in true_S) & set(int(x) for x in pred_S))


def recall_eq2(c, A, k: int):
    """Eq. 2: recall(n) = sum_q sum_l c(q,n,l) A(q,n) / (k L sum_q A(q,n)).
    c: int array [Q, N, L]; A: {0,1} array [Q, N]. Returns list of Fraction (None where
    the denominator is 0)."""
    c = np.asarray(c, dtype=np.int64)
    A = np.asarray(A, dtype=np.int64)
    Q, N, L = c.shape
    out = []
    for n in range(N):
        num = int(sum(int(c[q, n, l]) * int(A[q, n]) for q in range(Q) for l in range(L)))
        den = k * L * int(sum(int(A[q, n]) for q in range(Q)))
        out.append(Fraction(num, den) if den else None)
    return out


def recall_eq3(c, A, k: int):
    """Eq. 3: sum_n sum_q sum_l c A / (k L sum_n sum_q A), one exact division."""
    c = np.asarray(c, dtype=np.int64)
    A = np.asarray(A, dtype=np.int64)
    Q, N, L = c.shape
    num = 0
    den = 0
    for n in range(N):
        for q in range(Q):
            den += int(A[q, n])
            for l in range(L):
                num += int(c[q, n, l]) * int(A[q, n])
    return Fraction(num, k * L * den) if den else None


def recall_bruteforce(records, k: int, L: int):
    """Triple loop straight from the definition "the number of correctly predicted experts
    out of all activated experts" over explicit records
    {(q, n): [(true_S, pred_S, avail) per layer]}."""
    correct = 0
    activated = 0
    for (_q, _n), layers in records.items():
        for (true_S, pred_S, avail) in layers:
            activated += len(true_S)
            correct += _c_count(true_S, pred_S, avail)
    return Fraction(correct, activated) if activated else None


# ---------------------------------------------------------------- prefill
def prefill_permutation(ids):
    """Group (token, expert) pairs by expert, stable by token ("embeddings are grouped
    by their desired experts"). ids int [T, k]. Returns (perm_token [T*k], perm_slot [T*k],
    offsets [E+1]) for E = max id + 1 ... computed by a plain stable sort."""
    ids = np.asarray(ids)
    T, k = ids.shape
    pairs = [(int(ids[t, j]), t, j) for t in range(T) for j in range(k)]
    pairs.sort(key=lambda p: (p[0], p[1], p[2]))
    return pairs


def expert_counts(ids, E: int):
    """Tokens routed to each expert (P:214 footnote counts activated experts)."""
    ids = np.asarray(ids)
    return np.array([int(np.sum(ids == e)) for e in range(E)], dtype=np.int64)


def prefill_reference(h, w_gate, experts, k: int, eps: float = 1e-5, u=None):
    """Prefill MoE layer over T tokens: without attention tokens are independent, so
    each row is the decode layer's computation; grouping only changes the order of work.
    Returns per-token dicts from moe_layer."""
    h = np.asarray(h, dtype=np.float64)
    return [moe_layer(h[t], w_gate, experts, k, eps, u=None if u is None else u[t]) for t in range(h.shape[0])]


def softmax_all(r):
    """Plain softmax over all logits (used only to pin mixture_weights at k=E)."""
    r = np.asarray(r, dtype=np.float64)
    e = np.exp(r - r.max())
    return e / e.sum()


def _isclose(a, b, tol=1e-12):
    return math.isclose(a, b, rel_tol=tol, abs_tol=tol)
