"""Cross-token speculation: the shadow's token alignment period T_p ("align
the tokens ... once every few autoregression iterations", Fig. 6 T_i; S:165-173 shadow_decode_step)
through the C ABI vs the CPU oracle (-m gpu).

At iterations n with n mod T_p != 0 the shadow decodes with its OWN greedy token (its INT8-row LM
head), so its pass for n + 1 runs while the main model still decodes n and the loads of the next
token's first layers may start inside the lookahead window. Values never change; only the
predictions (and so the loads) do."""
import time

import numpy as np
import pytest

import oracle as O
from inputs import TINY, gen_model_weights, gen_prompt
from tests.gpu_util import assert_close, ids_match, token_match, torch

pytestmark = pytest.mark.gpu
SEED = 2512
K = TINY.k
BLOB = 3 * TINY.d * TINY.F * 2


@pytest.fixture(scope="module")
def od():
    t = torch()
    assert t.cuda.is_available(), "gpu tests need a B200"
    from paper_2512_03927_b200 import odmoe
    return odmoe


def engine(od, **kw):
    args = dict(dtype=od.BF16, weight_seed=SEED)
    args.update(kw)
    return od.Engine(TINY.L, TINY.E, TINY.k, TINY.d, TINY.F, TINY.V, **args)


def f32(eng, what, layer, n):
    return np.frombuffer(eng.debug_read(what, layer, 4 * n), dtype=np.float32).astype(np.float64)


def bf16(eng, what, layer, n):
    b = np.frombuffer(eng.debug_read(what, layer, 2 * n), dtype=np.uint16)
    return (b.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def i32(eng, what, layer, n):
    return np.frombuffer(eng.debug_read(what, layer, 4 * n), dtype=np.int32)


def _sets(a, k=8):
    return sorted(int(x) for x in a[:k] if x >= 0)


def run(eng, first, n):
    toks, recs_all, t = [], [], first
    for _ in range(n):
        t, recs = eng.decode_step(t)
        toks.append(t)
        recs_all.append(recs)
    return toks, recs_all


@pytest.mark.parametrize("period", [2, 4])
def test_same_precision_shadow_exact_for_every_period(od, period):
    """A shadow identical to the main model generates the main model's tokens, so speculative
    passes predict exactly (recall 1, S:171 generalised): every load is a predicted one, L*k loads
    and L*k blobs per token, and next-token loads were issued early."""
    first = int(gen_prompt(TINY, 2, 1)[0])
    base = engine(od, predictor=od.PRED_NONE, slots_per_gpu=2)
    ref_toks, _ = run(base, first, 12)
    base.close()
    eng = engine(od, predictor=od.PRED_SHADOW_SAME, slots_per_gpu=4, lookahead=2)
    eng.set_align_period(period)
    t, toks, early_prev = first, [], 0
    for n in range(12):
        st0 = eng.stats()
        t, recs = eng.decode_step(t)
        st1 = eng.stats()
        toks.append(t)
        assert all(r.correct == K for r in recs)
        S = [_sets(r.true_ids, K) for r in recs]
        I = [_sets(r.issued_ids) for r in recs]
        # the loader's loads of this step serve this token, except the next token's early loads;
        # this token's own early loads were issued (and counted) during the previous step
        early = st1["early_loads"] - st0["early_loads"]
        assert st1["loads_issued"] - st0["loads_issued"] - early + early_prev == O.expected_loads(S, I), n
        early_prev = early
        if all(r.pred_in_time for r in recs):
            assert I == S
    st = eng.stats()
    eng.close()
    assert toks == ref_toks
    assert st["correct"] == st["predicted_total"] == 12 * TINY.L * K
    assert st["spec_steps"] == sum(1 for n in range(12) if n % period)
    assert st["early_loads"] > 0


def test_int8_shadow_own_token_teacher_forced(od):
    """T_p = 2, INT8 shadow: per step, the pass that produced the predictions started from the main
    token (aligned steps) or from the previous pass's own token (unaligned), its own token is the
    oracle's argmax of Q(W_o) RMSNorm(h_L^shadow) (teacher-forced on the GPU's final shadow state,
    near-tie rule), its final state is h_{L-1} + y_{L-1} of its last layer, and its routing is the
    oracle's on its own states. Outputs equal the no-predictor run; recall accounting is exact."""
    W = gen_model_weights(TINY, SEED, dtype="bf16")
    SW = O.quantize_model_int8(W)
    d, L, E = TINY.d, TINY.L, TINY.E
    first = int(gen_prompt(TINY, 3, 1)[0])
    eng = engine(od, predictor=od.PRED_SHADOW_INT8, slots_per_gpu=4, lookahead=2, debug_capture=1)
    eng.set_align_period(2)
    t, prev_own, toks, excused = first, None, [], 0
    for n in range(10):
        nxt, recs = eng.decode_step(t)
        t_in = t if n % 2 == 0 else prev_own
        assert np.allclose(f32(eng, "SH_H_IN", 0, d), SW["emb"][t_in], rtol=1e-6, atol=1e-9), n
        for l in range(L):
            sh = f32(eng, "SH_H_IN", l, d)
            su = bf16(eng, "SH_U", l, d)
            assert np.all(np.abs(su - O.rms_norm(sh)) <= 2.0 ** -8 * np.abs(O.rms_norm(sh)) + 1e-6)
            r_ref = O.router_logits(SW["router"][l], su)
            sids = i32(eng, "SH_IDS", l, K)
            ok, exc = ids_match(sids, r_ref, K)
            assert ok, (n, l, sids)
            excused += exc
            assert _sets(recs[l].pred_ids, K) == sorted(int(x) for x in sids)
        # last layer's expert outputs -> the shadow's final state
        sh = f32(eng, "SH_H_IN", L - 1, d)
        su = bf16(eng, "SH_U", L - 1, d)
        sids = [int(x) for x in i32(eng, "SH_IDS", L - 1, K)]
        w = O.mixture_weights(O.router_logits(SW["router"][L - 1], su), sids)
        y = sum(w[j] * O.expert_ffn(*SW["experts"][L - 1][sids[j]], su) for j in range(K))
        hf = f32(eng, "SH_H_FINAL", 0, d)
        assert_close(hf, sh + y, 1e-4, what=("shadow h_L", n))
        own = int(i32(eng, "SH_TOK", 0, 1)[0])
        z_ref = O.final_logits(SW["lm_head"], hf)
        ok, exc = token_match(own, z_ref)
        assert ok, (n, own, O.greedy_argmax(z_ref))
        excused += exc
        z = f32(eng, "SH_LM_LOGITS", 0, TINY.V)
        z_same = SW["lm_head"] @ O.round_bf16(O.rms_norm(hf))
        assert_close(z, z_same, 1e-4, 1e-3, what=("shadow lm logits", n))
        for l in range(L):
            assert recs[l].correct == len(set(_sets(recs[l].true_ids, K)) & set(_sets(recs[l].pred_ids, K)))
        prev_own = own
        toks.append(nxt)
        t = nxt
    assert excused <= 3
    st = eng.stats()
    eng.close()
    assert st["spec_steps"] == 5
    base = engine(od, predictor=od.PRED_NONE, slots_per_gpu=2)
    ref_toks, _ = run(base, first, 10)
    base.close()
    assert toks == ref_toks


def test_predictions_match_oracle_shadow_decode(od):
    """Free-running against O.shadow_decode (period 3) over the GPU's own main tokens: wherever the
    GPU shadow consumed the same token as the oracle's, its predictions are the oracle's (barring
    near-ties, counted); the oracle's T_p = 1 run is Mode A."""
    W = gen_model_weights(TINY, SEED, dtype="bf16")
    SW = O.quantize_model_int8(W)
    first = int(gen_prompt(TINY, 4, 1)[0])
    eng = engine(od, predictor=od.PRED_SHADOW_INT8, slots_per_gpu=4, lookahead=2, debug_capture=1)
    eng.set_align_period(3)
    t, main_in, P_gpu, tin_gpu, own_prev = first, [], [], [], None
    for n in range(9):
        main_in.append(t)
        t_next, recs = eng.decode_step(t)
        P_gpu.append([_sets(r.pred_ids, K) for r in recs])
        own = int(i32(eng, "SH_TOK", 0, 1)[0])
        tin_gpu.append(t if n % 3 == 0 else own_prev)
        own_prev = own
        t = t_next
    eng.close()
    P_ref, tin_ref, _ = O.shadow_decode(SW, main_in, K, period=3)
    same, diff = 0, 0
    for n in range(9):
        if tin_ref[n] != tin_gpu[n]:
            continue
        for l in range(TINY.L):
            if sorted(P_ref[n][l]) == P_gpu[n][l]:
                same += 1
            else:
                diff += 1
    assert same > 0 and diff <= 2, (same, diff)


def test_early_loads_window_and_trace(od):
    """Loads for the next token are issued only inside the window (position L + m <= l_cur + D),
    they land before the next step uses them, and per-token load accounting stays exact."""
    eng = engine(od, predictor=od.PRED_SHADOW_SAME, slots_per_gpu=4, lookahead=2)
    eng.set_align_period(4)
    eng.set_trace(True)
    t = 41
    for _ in range(8):
        t, _ = eng.decode_step(t)
    time.sleep(0.2)
    ev = eng.trace()
    st = eng.stats()
    eng.close()
    nxt = [e for e in ev if e["type"] == "LoadIssue" and e["aux"] == 3]
    assert nxt and len(nxt) == st["early_loads"]
    for e in ev:
        if e["type"] == "LoadIssue":
            assert e["layer"] <= max(e["l_cur"], 0) + 2, e
    for e in nxt:
        assert e["layer"] >= TINY.L   # window position of the next token's layer
    ends = {(e["step"], e["layer"], e["expert"]): e for e in ev if e["type"] == "LoadEnd"}
    for e in ev:
        if e["type"] == "ComputeStart":
            assert ends[(e["step"], e["layer"], e["expert"])]["bytes"] == BLOB


def test_alignment_period_option_errors(od):
    eng = engine(od, predictor=od.PRED_NONE, slots_per_gpu=2)
    with pytest.raises(od.OdmoeError):
        eng.set_align_period(2)           # no shadow in this ctx
    eng.set_align_period(1)
    eng.close()
    eng = engine(od, predictor=od.PRED_SHADOW_INT8, slots_per_gpu=2)
    with pytest.raises(od.OdmoeError):
        eng.set_align_period(0)
    eng.set_align_period(2)
    t = 3
    for _ in range(3):
        t, _ = eng.decode_step(t)
    eng.set_predictor(od.PRED_NONE)       # abandons the speculation: its early loads are dropped
    t2, _ = eng.decode_step(t)
    eng.set_predictor(od.PRED_SHADOW_INT8)
    eng.decode_step(t2)
    eng.close()
