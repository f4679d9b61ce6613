"""Pins of the CPU oracle against what the paper and mathematics fix (-m "not gpu").

Each test names the passage / closed form it relies on. None of them re-types the
oracle's own formula: they use worked examples (tests/golden/*.json), closed forms,
brute force, invariants and special cases that reduce to library routines.
"""
import json
import math
import os
from fractions import Fraction
from itertools import permutations

import numpy as np
import pytest
import scipy.special

import oracle as O
from inputs import TINY, gen_model_weights

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ------------------------------------------------------------------ O1 RMSNorm
def test_rmsnorm_closed_form():
    g = gold("rmsnorm_closed_form.json")
    u = O.rms_norm(np.array(g["h"]), eps=g["eps"])
    assert np.allclose(u, g["u"], rtol=1e-15, atol=0)


def test_rmsnorm_scale_invariance_and_unit_rms():
    rng = np.random.default_rng(0)
    h = rng.standard_normal(257)
    u1 = O.rms_norm(h, eps=0.0)
    u2 = O.rms_norm(h * 1234.5, eps=0.0)
    assert np.allclose(u1, u2, rtol=1e-13)
    assert math.isclose(float(np.sqrt(np.mean(u1 ** 2))), 1.0, rel_tol=1e-13)
    # eps is added to the mean square, not to the root: a zero vector stays zero
    assert np.all(O.rms_norm(np.zeros(8)) == 0.0)
    # gamma scales elementwise
    gam = rng.standard_normal(257)
    assert np.allclose(O.rms_norm(h, gam, 0.0), u1 * gam, rtol=1e-13)


# ------------------------------------------------------------------ O2 router logits
def test_router_logits_selector_rows():
    # one-hot gate rows select coordinates of u (catches transposed W_g)
    E, d = 3, 5
    W = np.zeros((E, d))
    W[0, 4] = 1.0
    W[1, 0] = 2.0
    W[2, 2] = -1.0
    u = np.array([1.0, 2.0, 3.0, 4.0, 5.0])
    assert list(O.router_logits(W, u)) == [5.0, 2.0, -3.0]


def test_router_logits_bruteforce_integers():
    rng = np.random.default_rng(1)
    W = rng.integers(-5, 6, size=(8, 16)).astype(float)
    u = rng.integers(-5, 6, size=16).astype(float)
    r = O.router_logits(W, u)
    for e in range(8):
        assert r[e] == sum(W[e, j] * u[j] for j in range(16))


# ------------------------------------------------------------------ O3 top-k
def test_topk_spec_examples():
    for case in gold("topk_S80.json")["cases"]:
        assert O.top_k(case["r"], case["k"]) == case["S"], case


@pytest.mark.parametrize("seed", range(20))
def test_topk_matches_bruteforce(seed):
    rng = np.random.default_rng(seed)
    E = int(rng.integers(2, 9))
    k = int(rng.integers(1, E + 1))
    # small integer logits => many exact ties
    r = rng.integers(-3, 4, size=E).astype(float)
    assert O.top_k(r, k) == O.top_k_bruteforce(r, k)


def test_topk_permutation_equivariance():
    rng = np.random.default_rng(2)
    r = rng.standard_normal(8)
    S = set(O.top_k(r, 2))
    for _ in range(20):
        pi = rng.permutation(8)  # new index i holds old expert pi[i]
        Sp = {int(pi[i]) for i in O.top_k(r[pi], 2)}
        assert Sp == S


# ------------------------------------------------------------------ O4 mixture weights
def test_mixture_weights_hand_value():
    w = O.mixture_weights([math.log(3.0), 0.0, -7.0], [0, 1])
    assert np.allclose(w, [0.75, 0.25], rtol=1e-15)


def test_mixture_weights_k1_and_kE():
    rng = np.random.default_rng(3)
    r = rng.standard_normal(8)
    assert O.mixture_weights(r, [5]).tolist() == [1.0]
    S = list(range(8))
    assert np.allclose(O.mixture_weights(r, S), scipy.special.softmax(r), rtol=1e-14)
    S2 = O.top_k(r, 2)
    w2 = O.mixture_weights(r, S2)
    assert abs(w2.sum() - 1.0) < 1e-15
    # softmax-then-renormalise over S (Mixtral) equals softmax over the selected logits
    p = scipy.special.softmax(r)
    assert np.allclose(w2, p[S2] / p[S2].sum(), rtol=1e-13)


# ------------------------------------------------------------------ O5 expert FFN
def test_expert_closed_form():
    g = gold("expert_closed_form.json")
    W1, W3, W2, u = (np.array(g[k], dtype=float) for k in ("W1", "W3", "W2", "u"))
    y = O.expert_ffn(W1, W3, W2, u)
    assert np.allclose(y, g["y"], rtol=1e-15, atol=1e-16)
    # W1/W3 are not interchangeable, W2 is not symmetric in use
    assert not np.allclose(O.expert_ffn(W3, W1, W2, u), g["y"])
    assert not np.allclose(O.expert_ffn(W1, W3, W2.T, u), g["y"])
    assert math.isclose(float(O.silu(1.0)), 0.7310585786300049, rel_tol=1e-15)


def test_expert_zero_in_zero_out_and_purity():
    W1, W3, W2 = gen_model_weights(TINY, 5, layers=[0])["experts"][0][3]
    assert np.all(O.expert_ffn(W1, W3, W2, np.zeros(TINY.d)) == 0.0)
    u = np.linspace(-1, 1, TINY.d)
    assert np.array_equal(O.expert_ffn(W1, W3, W2, u), O.expert_ffn(W1, W3, W2, u))


def test_expert_dense_swiglu_library_special_case():
    """E=1, k=1: the MoE layer is a dense SwiGLU FFN; compare with torch's float64 silu."""
    import torch
    rng = np.random.default_rng(4)
    d, F = 16, 24
    W1, W3, W2 = rng.standard_normal((F, d)), rng.standard_normal((F, d)), rng.standard_normal((d, F))
    h = rng.standard_normal(d)
    out = O.moe_layer(h, np.ones((1, d)), {0: (W1, W3, W2)}, k=1, eps=1e-5)
    u = torch.tensor(O.rms_norm(h))
    ref = torch.nn.functional.linear(
        torch.nn.functional.silu(torch.nn.functional.linear(u, torch.tensor(W1))) * torch.nn.functional.linear(u, torch.tensor(W3)),
        torch.tensor(W2))
    assert np.allclose(out["y"], ref.numpy(), rtol=1e-12, atol=1e-12)
    assert np.allclose(out["h_next"], h + ref.numpy(), rtol=1e-12, atol=1e-12)


# ------------------------------------------------------------------ O6 combine
def test_identical_experts_any_routing():
    rng = np.random.default_rng(6)
    d, F, E = 8, 12, 8
    mats = (rng.standard_normal((F, d)), rng.standard_normal((F, d)), rng.standard_normal((d, F)))
    experts = {e: mats for e in range(E)}
    h = rng.standard_normal(d)
    Wg = rng.standard_normal((E, d))
    dense = O.expert_ffn(*mats, O.rms_norm(h))
    for S in ([0, 1], [7, 2], [3, 4]):
        out = O.moe_layer(h, Wg, experts, 2, S=S)
        assert np.allclose(out["y"], dense, rtol=1e-13)


def test_moe_layer_expert_permutation_invariance():
    rng = np.random.default_rng(7)
    d, F, E = 8, 12, 8
    experts = {e: (rng.standard_normal((F, d)), rng.standard_normal((F, d)), rng.standard_normal((d, F))) for e in range(E)}
    Wg = rng.standard_normal((E, d))
    h = rng.standard_normal(d)
    base = O.moe_layer(h, Wg, experts, 2)
    pi = rng.permutation(E)
    Wg_p = Wg[pi]
    experts_p = {i: experts[int(pi[i])] for i in range(E)}
    out = O.moe_layer(h, Wg_p, experts_p, 2)
    assert {int(pi[i]) for i in out["S"]} == set(base["S"])
    assert np.allclose(out["y"], base["y"], rtol=1e-13)


# ------------------------------------------------------------------ O7 decode iteration
@pytest.fixture(scope="module")
def tiny_fp32():
    return gen_model_weights(TINY, 2512, dtype="fp32")


def test_decode_determinism_and_override_neutrality(tiny_fp32):
    t1, recs1, z1 = O.decode_token(tiny_fp32, 17, TINY.k)
    t2, recs2, z2 = O.decode_token(tiny_fp32, 17, TINY.k)
    assert t1 == t2 and np.array_equal(z1, z2)
    natural = [r["S"] for r in recs1]
    t3, recs3, z3 = O.decode_token(tiny_fp32, 17, TINY.k, override=natural)
    assert t3 == t1 and np.array_equal(z3, z1)
    # a different override changes values (the override is honoured)
    other = [[(s[0] + 1) % 8, (s[1] + 1) % 8] if (s[0] + 1) % 8 != (s[1] + 1) % 8 else s for s in natural]
    _, _, z4 = O.decode_token(tiny_fp32, 17, TINY.k, override=other)
    assert not np.array_equal(z4, z1)


def test_greedy_argmax_ties_lowest_id():
    z = np.array([0.0, 2.0, 5.0, 5.0, 1.0, 5.0])
    assert O.greedy_argmax(z) == 2


def test_lm_head_constructed_tie(tiny_fp32):
    w = dict(tiny_fp32)
    t, recs, z = O.decode_token(w, 5, TINY.k)
    lm = np.array(w["lm_head"], copy=True)
    lm[900] = lm[t]  # an identical row at a higher id
    lm[3] = lm[t]    # and at a lower id: the lower one must win
    w2 = dict(w)
    w2["lm_head"] = lm
    t2, _, _ = O.decode_token(w2, 5, TINY.k)
    assert t2 == min(3, t)


# ------------------------------------------------------------------ O8 quantiser + shadow
def test_quantizer_spec_example():
    g = gold("quantizer_S70.json")
    q, s = O.quantize_int8_rows(np.array(g["W"]))
    assert q.tolist() == g["codes"]
    assert np.allclose(O.dequantize_int8_rows(q, s), g["values"], rtol=g["values_rel_tol"], atol=0)


def test_quantizer_half_step_bound_and_zero():
    rng = np.random.default_rng(8)
    W = rng.uniform(-0.02, 0.02, size=(64, 300)).astype(np.float32).astype(np.float64)
    q, s = O.quantize_int8_rows(W)
    m = np.max(np.abs(W), axis=1)
    # codes are the nearest grid points: |q - W*127/m| <= 1/2
    assert np.all(np.abs(q - W * 127.0 / m[:, None]) <= 0.5 + 1e-12)
    assert np.all(np.abs(q) <= 127) and np.all(np.max(np.abs(q), axis=1) == 127)
    # dequantised error <= half a step (+ fp32 rounding of the scale)
    err = np.abs(O.dequantize_int8_rows(q, s) - W)
    assert np.all(err <= (m / 127.0)[:, None] * (0.5 + 1e-6))
    qz, sz = O.quantize_int8_rows(np.zeros((3, 7)))
    assert np.all(qz == 0) and np.all(sz == 1.0)
    assert np.all(O.dequantize_int8_rows(qz, sz) == 0.0)  # S:72 zero fixed point
    # exact half ties round to even (the S:70 mechanism): with m = 127 the quotient is W
    qh, _ = O.quantize_int8_rows(np.array([[127.0, 2.5, 3.5, -0.5, -1.5, 0.5]]))
    assert qh[0].tolist() == [127, 2, 4, 0, -2, 0]


def test_round_bf16_hand_values_and_library():
    """BF16 = fp32 with 7 stored significand bits, round to nearest, ties to even."""
    e = 2.0 ** -8                                     # half an ulp of 1.0 in bf16
    x = np.array([1.0, 1.0 + e, 1.0 + 3 * e, 1.0 + e + 2.0 ** -20, -(1.0 + 3 * e), 0.0,
                  2.0 - e / 2, 3.0e38, 1.5, -0.0])
    want = [1.0, 1.0, 1.0 + 4 * e, 1.0 + 2 * e, -(1.0 + 4 * e), 0.0, 2.0, 3.0e38, 1.5, 0.0]
    got = O.round_bf16(x)
    assert np.allclose(got, want, rtol=2.0 ** -8, atol=0)
    assert got[:7].tolist() == want[:7]               # exact: ties to even (1+e -> 1, 1+3e -> 1+4e)
    assert np.signbit(got[9])                          # -0 keeps its sign
    import torch
    rng = np.random.default_rng(26)
    r = (rng.standard_normal(4096) * rng.choice([1e-3, 1.0, 1e3], 4096)).astype(np.float32)
    lib = torch.from_numpy(r).to(torch.bfloat16).to(torch.float64).numpy()
    assert np.array_equal(O.round_bf16(r), lib)
    # relative error <= u = 2^-8 (unit roundoff of an 8-bit significand)
    assert np.all(np.abs(O.round_bf16(r) - r) <= 2.0 ** -8 * np.abs(r.astype(np.float64)))


def test_nf4_codebook_matches_quantile_construction():
    pub = np.asarray(O.NF4_CODEBOOK, dtype=np.float32)
    der = O.nf4_codebook_from_quantiles()
    assert len(pub) == 16 and np.all(np.diff(pub) > 0)
    assert pub[0] == -1.0 and pub[15] == 1.0 and pub[7] == 0.0
    # the published table was computed in fp32 (values normalised to 1): agree to 2 ulp of 1.0
    assert np.all(np.abs(pub.astype(np.float64) - der) <= 2 * 2.0 ** -23), np.abs(pub - der)


def test_nf4_quantizer_brute_force_and_properties():
    rng = np.random.default_rng(27)
    W = (rng.standard_normal((6, 128)) * 0.02).astype(np.float32).astype(np.float64)
    W[2, 64:] = 0.0                                       # one all-zero block
    W[3, :64] = np.asarray(O.NF4_CODEBOOK * 4, dtype=np.float32) * 0.5   # codebook values x a
    codes, a = O.quantize_nf4_blocks(W)
    assert codes.shape == (6, 128) and a.shape == (6, 2) and codes.dtype == np.uint8
    cb = [float(np.float32(c)) for c in O.NF4_CODEBOOK]
    for r in range(6):
        for j in range(128):
            amax = max(abs(float(v)) for v in W[r, (j // 64) * 64:(j // 64) * 64 + 64])
            if amax == 0.0:
                assert codes[r, j] == 7
                continue
            assert a[r, j // 64] == np.float32(amax)
            x = float(W[r, j]) / amax
            best = min(range(16), key=lambda i: (abs(x - cb[i]), i))     # brute force, Python floats
            assert codes[r, j] == best, (r, j)
    assert codes[3, :64].tolist() == list(range(16)) * 4  # codebook points are fixed points
    deq = O.dequantize_nf4_blocks(codes, a)
    assert np.all(deq[2, 64:] == 0.0)
    gaps = np.diff(np.asarray(cb))
    half_gap = np.max(gaps) / 2
    assert np.all(np.abs(deq - W) <= half_gap * np.repeat(a.astype(np.float64), 64, axis=1) + 1e-12)
    # an exact midpoint between codes 7 (0.0) and 8 goes to the lower index
    m = cb[8] / 2
    c2, _ = O.quantize_nf4_blocks(np.array([[1.0, m] + [0.0] * 62]))
    assert c2[0, 1] == 7 and c2[0, 0] == 15


def test_e4m3_rounding_matches_library_cast():
    import torch
    V = O.e4m3_values()
    assert len(V) == 127 and V[-1] == 448.0 and V[1] == 2.0 ** -9 and np.all(np.diff(V) > 0)
    lib_tbl = torch.arange(127, dtype=torch.uint8).view(torch.float8_e4m3fn).to(torch.float64).numpy()
    assert np.array_equal(V, lib_tbl)
    rng = np.random.default_rng(28)
    x = np.concatenate([rng.standard_normal(20000) * 50, rng.standard_normal(2000) * 1e-3,
                        (V[:-1] + V[1:]) / 2, -(V[:-1] + V[1:]) / 2,            # exact midpoints (ties)
                        [0.0, 448.0, 447.9, 449.0, 500.0, -600.0]]).astype(np.float32)
    vals, codes = O.round_e4m3(x)
    lib = torch.from_numpy(x).to(torch.float8_e4m3fn)
    inr = np.abs(x) < 464.0            # torch's cast gives NaN past the last rounding boundary
    assert np.array_equal(codes[inr], lib.view(torch.uint8).numpy()[inr])
    assert np.array_equal(vals[inr], lib.to(torch.float64).numpy()[inr])
    assert np.all(np.abs(vals[~inr]) == 448.0)   # satfinite (the quantiser never gets there)


def test_fp8_row_quantizer_properties():
    rng = np.random.default_rng(29)
    W = (rng.standard_normal((16, 256)) * 0.02).astype(np.float32).astype(np.float64)
    W[4] = 0.0
    codes, s = O.quantize_fp8_rows(W)
    deq = O.dequantize_fp8_rows(codes, s)
    assert np.all(codes[4] == 0) and s[4] == 1.0
    rows = [r for r in range(16) if r != 4]
    # the row maximum maps to +-448 (code 0x7E / 0xFE) and the error is within half an E4M3 step
    for r in rows:
        j = int(np.argmax(np.abs(W[r])))
        assert codes[r, j] & 0x7F == 0x7E
        assert np.all(np.abs(deq[r] - W[r]) <= np.abs(W[r]) * 2.0 ** -4 + s[r] * 2.0 ** -10)


# ------------------------------------------------------------------ attention block (Q29)
def test_rope_closed_forms():
    rng = np.random.default_rng(30)
    x = rng.standard_normal((3, 64))
    assert np.allclose(O.rope(x, 0), x, rtol=0, atol=0)
    assert np.allclose(np.linalg.norm(O.rope(x, 17), axis=-1), np.linalg.norm(x, axis=-1), rtol=1e-12)
    q, k = rng.standard_normal(64), rng.standard_normal(64)
    a = O.rope(q, 9) @ O.rope(k, 4)
    b = O.rope(q, 9 + 123) @ O.rope(k, 4 + 123)
    assert abs(a - b) < 1e-9 * max(1.0, abs(a))
    # hd = 2: a plane rotation by pos radians (frequency theta^0 = 1)
    r = O.rope(np.array([1.0, 0.0]), 3)
    assert np.allclose(r, [math.cos(3), math.sin(3)], rtol=0, atol=1e-15)


def test_attention_decode_special_cases_and_library():
    import torch
    rng = np.random.default_rng(31)
    H, Hkv, hd, T = 8, 2, 16, 11
    q = rng.standard_normal((H, hd))
    K, V = rng.standard_normal((T, Hkv, hd)), rng.standard_normal((T, Hkv, hd))
    o1 = O.attention_decode(q, K[:1], V[:1])                     # one position -> its value
    assert np.allclose(o1, np.repeat(V[0], H // Hkv, axis=0), rtol=0, atol=1e-15)
    Ke = np.repeat(K[:1], T, axis=0)                               # equal keys -> mean of values
    assert np.allclose(O.attention_decode(q, Ke, V), np.repeat(V.mean(axis=0), H // Hkv, axis=0), atol=1e-12)
    o = O.attention_decode(q, K, V)
    tq = torch.from_numpy(q)[None, :, None, :]                    # [1, H, 1, hd]
    tk = torch.from_numpy(K).permute(1, 0, 2).repeat_interleave(H // Hkv, dim=0)[None]
    tv = torch.from_numpy(V).permute(1, 0, 2).repeat_interleave(H // Hkv, dim=0)[None]
    ref = torch.nn.functional.scaled_dot_product_attention(tq, tk, tv)[0, :, 0, :].numpy()
    assert np.allclose(o, ref, rtol=1e-10, atol=1e-12)


def test_attn_block_closed_forms():
    rng = np.random.default_rng(32)
    d, H, Hkv = 16, 4, 2
    hd = d // H
    Wq, Wk = rng.standard_normal((d, d)), rng.standard_normal((Hkv * hd, d))
    Wv = rng.standard_normal((Hkv * hd, d))
    h = rng.standard_normal(d)
    cache = O.new_cache([0])
    out, _ = O.attn_block(h, (Wq, Wk, Wv, np.zeros((d, d))), (H, Hkv), cache[0], 0)
    assert np.array_equal(out, h)                                  # W_o = 0: residual only
    # one position: attention returns v of the query head's group; W_v selects coordinates
    sel = np.zeros((Hkv * hd, d))
    for i in range(Hkv * hd):
        sel[i, i] = 1.0
    Wo = np.zeros((d, d))
    Wo[0, 0] = 2.0                                                 # out_0 = 2 * o[head 0][0]
    cache = O.new_cache([0])
    out, rec = O.attn_block(h, (Wq, Wk, sel, Wo), (H, Hkv), cache[0], 0)
    x = O.rms_norm(h)
    assert np.allclose(out[0], h[0] + 2.0 * x[0], rtol=1e-12) and np.allclose(out[1:], h[1:])
    assert len(cache[0]["K"]) == 1


def test_same_precision_shadow_recall_is_one(tiny_fp32):
    """a full-precision shadow with token alignment predicts exactly."""
    toks, routes = O.decode_sequence(tiny_fp32, 11, 6, TINY.k)
    prev = [11] + toks[:-1]
    c = np.zeros((1, len(toks), TINY.L), dtype=int)
    for n, t in enumerate(prev):
        P, _ = O.shadow_predict(tiny_fp32, t, TINY.k)
        for l in range(TINY.L):
            c[0, n, l] = len(set(P[l]) & set(routes[n][l]))
    assert O.recall_eq3(c, np.ones((1, len(toks)), dtype=int), TINY.k) == 1


def test_int8_shadow_predicts_most_experts(tiny_fp32):
    """Not a value pin (parity unpinned on random weights): the INT8 shadow of a random
    model agrees on a large majority of activations (sanity)."""
    sw = O.quantize_model_int8(tiny_fp32)
    toks, routes = O.decode_sequence(tiny_fp32, 11, 8, TINY.k)
    prev = [11] + toks[:-1]
    hit = tot = 0
    for n, t in enumerate(prev):
        P, _ = O.shadow_predict(sw, t, TINY.k)
        for l in range(TINY.L):
            hit += len(set(P[l]) & set(routes[n][l]))
            tot += TINY.k
    assert hit / tot > 0.8


# ------------------------------------------------------------------ O9 placement
def test_plan_examples():
    g = gold("plan_examples.json")
    for c in g["groups"]:
        assert O.plan_groups(c["N"], c["G"]) == c["groups"]
    for c in g["groups_error"]:
        with pytest.raises(ValueError):
            O.plan_groups(c["N"], c["G"])
    for c in g["assign_layer"]:
        assert O.assign_layer(c["l"], c["NG"]) == c["g"]
    for c in g["assign_experts"]:
        assert O.assign_experts(c["experts"], c["workers"]) == {int(k): v for k, v in c["map"].items()}
    for c in g["budget"]:
        assert math.isclose(O.max_load_budget(c["tM"], c["tW"], c["NG"]), c["t"], rel_tol=1e-12)
    for c in g["reloads"]:
        res = {int(k): v for k, v in c["resident"].items()}
        assert [list(x) for x in O.misprediction_reloads(c["true"], res)] == c["reload"]
    for c in g["residency_bound"]:
        assert O.residency_bound(c["D"], c["NG"]) == c["bound"]


def test_plan_group_size_and_single_gpu_pairing():
    assert O.plan_group_size(2, 1) == 1 and O.plan_group_size(2, 8) == 2
    assert O.assign_experts([6, 1], [0]) == {1: 0, 6: 0}
    with pytest.raises(ValueError):
        O.assign_experts([1, 2, 3], [0, 1])


def test_pairing_is_one_to_one_and_layer_groups_cycle():
    for experts in permutations(range(8), 2):
        m = O.assign_experts(list(experts), [4, 5])
        assert sorted(m.values()) == [4, 5]
    NG = 4
    assert [O.assign_layer(l, NG) for l in range(9)] == [0, 1, 2, 3, 0, 1, 2, 3, 0]


# ------------------------------------------------------------------ O10 recall
def test_recall_spec_examples():
    for case in gold("recall_S201.json")["cases"]:
        c, A, k = np.array(case["c"]), np.array(case["A"]), case["k"]
        eq2 = O.recall_eq2(c, A, k)
        assert [float(x) for x in eq2] == case["eq2"]
        eq3 = O.recall_eq3(c, A, k)
        want = case["eq3"]
        assert eq3 == (Fraction(*want) if isinstance(want, list) else Fraction(want))


def test_recall_matches_bruteforce_on_random_records():
    """1,000 random record sets (Q<=5, N<=20, L<=8, k<=3, early stops)."""
    rng = np.random.default_rng(9)
    for _ in range(1000):
        Q, N, L, k = (int(rng.integers(1, 6)), int(rng.integers(1, 21)), int(rng.integers(1, 9)), int(rng.integers(1, 4)))
        E = k + int(rng.integers(0, 4))
        lengths = rng.integers(0, N + 1, size=Q)
        c = np.zeros((Q, N, L), dtype=int)
        A = np.zeros((Q, N), dtype=int)
        records = {}
        for q in range(Q):
            for n in range(N):
                A[q, n] = int(n < lengths[q])
                if not A[q, n]:
                    continue
                layers = []
                for l in range(L):
                    t = list(rng.choice(E, size=k, replace=False))
                    p = list(rng.choice(E, size=k, replace=False))
                    avail = bool(rng.random() < 0.9)
                    layers.append((t, p, avail))
                    c[q, n, l] = len(set(t) & set(p)) if avail else 0
                records[(q, n)] = layers
        assert O.recall_eq3(c, A, k) == O.recall_bruteforce(records, k, L)
        eq2 = O.recall_eq2(c, A, k)
        for n in range(N):
            sub = {key: v for key, v in records.items() if key[1] == n}
            assert eq2[n] == O.recall_bruteforce(sub, k, L)


def test_random_prediction_closed_form():
    """"an easy calculation shows that the recall in Case 5 is only ~25%": a uniform
    random k-subset of E experts has E[c] = k^2/E, so E[recall] = k/E = 0.25 for k=2, E=8."""
    rng = np.random.default_rng(10)
    Q, N, L, k, E = 4, 128, 32, 2, 8
    c = np.zeros((Q, N, L), dtype=int)
    for q in range(Q):
        for n in range(N):
            for l in range(L):
                t = set(rng.choice(E, size=k, replace=False).tolist())
                p = set(rng.choice(E, size=k, replace=False).tolist())
                c[q, n, l] = len(t & p)
    r = float(O.recall_eq3(c, np.ones((Q, N), dtype=int), k))
    p = k / E
    sigma = math.sqrt(p * (1 - p) / (k * L * N * Q))
    assert abs(r - 0.25) < 4 * sigma * 1.5


# ------------------------------------------------------------------ prefill grouping
def test_prefill_permutation_coverage_and_stability():
    rng = np.random.default_rng(11)
    T, k, E = 37, 2, 8
    ids = np.array([rng.choice(E, size=k, replace=False) for _ in range(T)])
    pairs = O.prefill_permutation(ids)
    assert sorted((t, j) for _, t, j in pairs) == [(t, j) for t in range(T) for j in range(k)]
    es = [e for e, _, _ in pairs]
    assert es == sorted(es)
    for e in range(E):
        toks = [t for ee, t, _ in pairs if ee == e]
        assert toks == sorted(toks)
    assert O.expert_counts(ids, E).sum() == T * k


def test_paper_constants_shapes():
    """P:260, P:51, P:379, P:403 numbers reproduced from the Mixtral shape in fp32."""
    g = gold("paper_constants.json")
    d, F, E, L = 4096, 14336, 8, 32
    assert d * 4 == g["embedding_bytes_fp32"]
    assert 2 * 8 * 128 * 4 == g["kv_bytes_per_token_layer_fp32"]
    assert 2 * 8 * 128 * 4 * L == g["kv_payload_per_token"]
    expert_fp32 = 3 * d * F * 4
    assert expert_fp32 < g["worker_GB_max"] * 1e9
    assert abs(E * L * expert_fp32 / 1e9 - g["fully_cached_GB"]) < 1.0
    assert abs(E * L * 3 * d * F / 1e9 - g["shadow_GB"]) < 0.5


# ------------------------------------------------------------------ parity protocol (north_star; Q4)
def test_near_tie_and_tied_run_golden_cases():
    """The excuse window of the parity protocol, pinned case by case: k-th vs (k+1)-th (not
    k-1 / k), relative not absolute, both zero, negatives, just inside / just outside."""
    for c in gold("near_tie_cases.json")["near_tie"]:
        assert O.near_tie(c["r"], c["k"]) == c["tie"], c
        assert O.tied_run(c["r"], c["k"]) == set(c["run"]), c


def test_ids_excusable_golden_cases():
    """A GPU set may differ from the oracle's only by swapping members of the tied run; rank order
    must follow the oracle logits except between near-equal ones."""
    for c in gold("near_tie_cases.json")["ids"]:
        assert O.ids_excusable(c["ids"], c["r"], c["k"]) == (c["ok"], c["excused"]), c


def test_ids_excusable_bruteforce_small():
    """Brute force over every ordered k-tuple on small integer logits with ties: accepted tuples
    are exactly those whose sorted logit vector equals the top-k's (exact ties only, so the
    window reduces to equality) and that are ordered by non-increasing logit."""
    rng = np.random.default_rng(21)
    for _ in range(200):
        E, k = int(rng.integers(2, 6)), int(rng.integers(1, 4))
        k = min(k, E)
        r = rng.integers(-2, 3, size=E).astype(float) * 4.0  # ties or gaps >= 4 (far outside 1e-3)
        want = sorted(r, reverse=True)[:k]
        for ids in permutations(range(E), k):
            vals = [r[i] for i in ids]
            expect = sorted(vals, reverse=True) == want and vals == sorted(vals, reverse=True)
            ok, _ = O.ids_excusable(list(ids), r, k)
            assert ok == expect, (r, k, ids)


def test_final_logits_apply_the_rmsnorm():
    """z = W_o RMSNorm(h): with W_o = I and h = [3, 4], z = h / sqrt(12.5 + 1e-5) (closed form); a
    missing or doubled norm is off by >= 4e-6 relative."""
    z = O.final_logits(np.eye(2), np.array([3.0, 4.0]))
    want = np.array([3.0, 4.0]) / math.sqrt(12.5 + 1e-5)
    assert np.allclose(z, want, rtol=1e-14, atol=0)
    assert not np.allclose(z, np.array([3.0, 4.0]), rtol=1e-6)
    assert not np.allclose(z, O.rms_norm(want), rtol=1e-6, atol=0)


# ------------------------------------------------------------------ loader accounting (a6 <-> a12)
def test_expected_loads_spec_examples():
    for c in gold("loads_S311.json")["cases"]:
        assert O.expected_loads(c["S"], c["I"]) == c["loads"], c


def test_expected_loads_recall_identity_on_random_records():
    """when every layer's k predicted experts were issued before its router,
    loads = L*k*(2 - recall(n)) exactly (recall from Eq. 2 over one token); PERFECT => L*k."""
    rng = np.random.default_rng(22)
    for _ in range(300):
        L, k = int(rng.integers(1, 9)), int(rng.integers(1, 4))
        E = k + int(rng.integers(0, 5))
        S = [list(rng.choice(E, size=k, replace=False)) for _ in range(L)]
        P = [list(rng.choice(E, size=k, replace=False)) for _ in range(L)]
        c = np.array([[[len(set(s) & set(p)) for s, p in zip(S, P)]]])
        rec = O.recall_eq2(c, np.ones((1, 1), dtype=int), k)[0]
        assert Fraction(O.expected_loads(S, P)) == L * k * (2 - rec)
        assert O.expected_loads(S, S) == L * k
        assert O.expected_loads(S, [[] for _ in S]) == L * k


def test_misprediction_reload_set_is_true_minus_issued():
    """the reload set is exactly true \\ resident, one reload per stale worker."""
    rng = np.random.default_rng(23)
    for _ in range(300):
        E, k = 8, 2
        S = list(rng.choice(E, size=k, replace=False))
        I = list(rng.choice(E, size=k, replace=False))
        rel = O.misprediction_reloads(S, {int(e): 0 for e in I})
        assert sorted(e for e, _ in rel) == sorted(set(int(x) for x in S) - set(int(x) for x in I))
        assert len(rel) + len(set(I)) == O.expected_loads([S], [I])


# ------------------------------------------------------------------ cross-token speculation
@pytest.fixture(scope="module")
def tiny_shadow(tiny_fp32):
    return O.quantize_model_int8(tiny_fp32)


def test_shadow_decode_period_one_is_mode_a(tiny_fp32, tiny_shadow):
    """T_p = 1 aligns every iteration: identical to the token-aligned shadow (Mode A) per token."""
    toks, _ = O.decode_sequence(tiny_fp32, 11, 6, TINY.k)
    main_in = [11] + toks[:-1]
    P, t_in, _ = O.shadow_decode(tiny_shadow, main_in, TINY.k, period=1)
    assert t_in == main_in
    for n, t in enumerate(main_in):
        assert P[n] == O.shadow_predict(tiny_shadow, t, TINY.k)[0]


def test_shadow_decode_same_precision_recall_one_for_every_period(tiny_fp32):
    """S:171/S:217 generalised: a shadow identical to the main model generates the main model's
    own tokens, so its predictions are exact for every alignment period."""
    toks, routes = O.decode_sequence(tiny_fp32, 11, 8, TINY.k)
    main_in = [11] + toks[:-1]
    for period in (1, 2, 4, 8):
        P, t_in, t_out = O.shadow_decode(tiny_fp32, main_in, TINY.k, period)
        assert t_in == main_in and t_out == toks
        assert all(sorted(P[n][l]) == routes[n][l] for n in range(8) for l in range(TINY.L))


def test_shadow_decode_unaligned_iterations_ignore_the_main_token(tiny_fp32, tiny_shadow):
    """At n mod T_p != 0 the shadow consumes its own previous token: the main token there has no
    influence, and t_in[n] = t_out[n-1]."""
    toks, _ = O.decode_sequence(tiny_fp32, 5, 6, TINY.k)
    main_in = [5] + toks[:-1]
    P, t_in, t_out = O.shadow_decode(tiny_shadow, main_in, TINY.k, period=3)
    scrambled = [t if n % 3 == 0 else (t + 101) % TINY.V for n, t in enumerate(main_in)]
    P2, t_in2, _ = O.shadow_decode(tiny_shadow, scrambled, TINY.k, period=3)
    assert P2 == P and t_in2 == t_in
    for n in range(1, 6):
        if n % 3:
            assert t_in[n] == t_out[n - 1]
        else:
            assert t_in[n] == main_in[n]


# ------------------------------------------------------------------ sliced loading
def test_sliced_partials_closed_form_and_sum():
    """W1 = W3 = W2 = I (F = d = 4, n = 2): expert_ffn(u) = silu(u) * u; slice 0 owns units 0-1 and
    writes only outputs 0-1 through W2's COLUMNS 0-1, slice 1 the rest (closed form). On random
    weights the partials sum to expert_ffn and n = 1 is expert_ffn itself."""
    u = np.array([0.5, -1.0, 2.0, 0.25])
    I = np.eye(4)
    p = O.sliced_expert_partials(I, I, I, u, 2)
    s = u / (1.0 + np.exp(-u)) * u
    assert np.allclose(p[0], [s[0], s[1], 0, 0], rtol=0, atol=1e-15)
    assert np.allclose(p[1], [0, 0, s[2], s[3]], rtol=0, atol=1e-15)
    W2 = np.arange(16.0).reshape(4, 4)   # distinguishes columns from rows
    p = O.sliced_expert_partials(I, I, W2, u, 2)
    assert np.allclose(p[0], W2[:, :2] @ s[:2], rtol=1e-15) and np.allclose(p[1], W2[:, 2:] @ s[2:], rtol=1e-15)
    rng = np.random.default_rng(24)
    W1, W3 = rng.normal(size=(64, 16)), rng.normal(size=(64, 16))
    W2r = rng.normal(size=(16, 64))
    x = rng.normal(size=16)
    full = O.expert_ffn(W1, W3, W2r, x)
    for n in (1, 2, 4, 8):
        parts = O.sliced_expert_partials(W1, W3, W2r, x, n)
        assert len(parts) == n and np.allclose(np.sum(parts, axis=0), full, rtol=1e-12, atol=1e-12)
    assert np.array_equal(O.sliced_expert_partials(W1, W3, W2r, x, 1)[0], full)
    with pytest.raises(ValueError):
        O.sliced_expert_partials(W1, W3, W2r, x, 3)
