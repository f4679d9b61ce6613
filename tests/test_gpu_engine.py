"""The stateful decode engine through the C ABI vs the CPU oracle (-m gpu).

Parity is teacher-forced per layer (SURVEY §8(c) protocol): the engine's debug capture exports
h_l, u_l, logits, ids, w and the per-expert outputs of every layer; the oracle recomputes each
layer from the GPU's own inputs. Because the hot path has no attention/KV state, a decode step
is a pure function of its input token, so feeding the GPU's previous token to the oracle is the
token-level teacher forcing."""
import numpy as np
import pytest

import oracle as O
from inputs import MIXTRAL, TINY, gen_expert, gen_model_weights, gen_prompt
from tests.gpu_util import TOL_BF16, TOL_FP32, assert_close, ids_match, l2rel, token_match, torch

pytestmark = pytest.mark.gpu
SEED = 2512


@pytest.fixture(scope="module")
def od():
    t = torch()
    assert t.cuda.is_available(), "gpu tests need a B200"
    from paper_2512_03927_b200 import odmoe
    return odmoe


def engine(od, shape, dtype="bf16", **kw):
    args = dict(dtype=od.BF16 if dtype == "bf16" else od.FP32, weight_seed=SEED)
    args.update(kw)
    return od.Engine(shape.L, shape.E, shape.k, shape.d, shape.F, shape.V, **args)


def read_f32(eng, what, layer, n):
    return np.frombuffer(eng.debug_read(what, layer, 4 * n), dtype=np.float32).astype(np.float64)


def read_u(eng, what, layer, d, dtype):
    if dtype == "bf16":
        b = np.frombuffer(eng.debug_read(what, layer, 2 * d), dtype=np.uint16)
        return (b.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    return read_f32(eng, what, layer, d)


def read_i32(eng, what, layer, n):
    return np.frombuffer(eng.debug_read(what, layer, 4 * n), dtype=np.int32)


def check_step_teacher_forced(eng, W, shape, dtype, token_in, token_out, shadow_W=None):
    """Per-layer teacher-forced comparison of one captured decode step. Returns #excused."""
    L, E, k, d = shape.L, shape.E, shape.k, shape.d
    tol = TOL_BF16 if dtype == "bf16" else TOL_FP32
    excused = 0
    h0 = read_f32(eng, "H_IN", 0, d)
    assert np.array_equal(h0.astype(np.float32), np.asarray(W["emb"][token_in], dtype=np.float32))
    for l in range(L):
        h = read_f32(eng, "H_IN", l, d)
        u = read_u(eng, "U", l, d, dtype)
        u_ref = O.rms_norm(h)
        utol = 2.0 ** -8 if dtype == "bf16" else 1e-6
        assert np.all(np.abs(u - u_ref) <= utol * np.abs(u_ref) + 1e-6), l
        lg = read_f32(eng, "LOGITS", l, E)
        r_ref = O.router_logits(W["router"][l], u)
        assert np.allclose(lg, r_ref, rtol=0, atol=1e-5 * np.abs(r_ref).max() + 1e-7), l
        ids = read_i32(eng, "IDS", l, k)
        ok, diff = ids_match(ids, r_ref, k)
        assert ok, (l, ids, r_ref)
        excused += diff
        w = read_f32(eng, "W", l, k)
        assert np.allclose(w, O.mixture_weights(r_ref, list(ids)), atol=2e-6)
        yp = read_f32(eng, "Y_PART", l, k * d).reshape(k, d)
        y_ref_total = np.zeros(d)
        for j in range(k):
            W1, W3, W2 = W["experts"][l][int(ids[j])]
            yr = w[j] * O.expert_ffn(W1, W3, W2, u)
            assert_close(yp[j], yr, tol, what=("y", l, j))
            y_ref_total += yr
        h_next = read_f32(eng, "H_IN", l + 1, d) if l + 1 < L else read_f32(eng, "H_FINAL", 0, d)
        assert_close(h_next, h + y_ref_total, tol, what=("h", l))
    # LM head + argmax from the captured final hidden state
    hf = read_f32(eng, "H_FINAL", 0, d)
    z = read_f32(eng, "LM_LOGITS", 0, shape.V)
    z_ref = O.final_logits(W["lm_head"], hf)
    # the GPU feeds the LM head RMSNorm(h_L) rounded to the model dtype (as u): same decision here,
    # then element-wise fp32-order agreement (a missing or doubled norm fails this)
    x = O.rms_norm(hf)
    z_same = np.asarray(W["lm_head"], dtype=np.float64) @ (O.round_bf16(x) if dtype == "bf16" else x)
    assert_close(z, z_same, 1e-4, 1e-3, what="lm logits")  # 1e-3: a bf16 rounding flip of one input
    assert l2rel(z, z_ref) <= tol
    ok, exc = token_match(token_out, z_ref)
    assert ok, (token_out, O.greedy_argmax(z_ref))
    excused += exc
    if shadow_W is not None:
        for l in range(L):
            sh = read_f32(eng, "SH_H_IN", l, d)
            su = read_u(eng, "SH_U", l, d, "bf16")
            assert np.all(np.abs(su - O.rms_norm(sh)) <= 2.0 ** -8 * np.abs(O.rms_norm(sh)) + 1e-6)
            sr_ref = O.router_logits(shadow_W["router"][l], su)
            sids = read_i32(eng, "SH_IDS", l, k)
            ok, diff = ids_match(sids, sr_ref, k)
            assert ok, ("shadow", l, sids, sr_ref)
            excused += diff
        # the shadow starts from ITS embedding row of the main token (token alignment)
        assert np.allclose(read_f32(eng, "SH_H_IN", 0, d), shadow_W["emb"][token_in], rtol=1e-6, atol=1e-9)
    return excused


@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_tiny_decode_teacher_forced(od, dtype):
    W = gen_model_weights(TINY, SEED, dtype=dtype)
    SW = O.quantize_model_int8(W)
    eng = engine(od, TINY, dtype, predictor=od.PRED_SHADOW_INT8, slots_per_gpu=2, debug_capture=1)
    tok = int(gen_prompt(TINY, 1, 1)[0])
    excused = 0
    for n in range(16):
        nxt, recs = eng.decode_step(tok)
        excused += check_step_teacher_forced(eng, W, TINY, dtype, tok, nxt, SW)
        # recall accounting recomputed from the records (Eq. 3, exact)
        for l in range(TINY.L):
            S = set(recs[l].true_ids[: TINY.k])
            P = set(recs[l].pred_ids[: TINY.k])
            assert recs[l].correct == len(S & P)
        tok = nxt
    assert excused <= 3
    st = eng.stats()
    assert st["tokens"] == 16
    assert st["max_resident"] <= 2   # S:326 residency audit at 2 slots
    eng.close()


@pytest.mark.parametrize("dtype,slots", [("fp32", 1), ("bf16", 2)])
def test_expert_layer_period_teacher_forced(od, dtype, slots):
    """expert_layer_period P = 2: layer l's experts are layer (l mod 2)'s, the host pool holds 2 layers,
    every load still moves a whole blob. Teacher-forced per layer vs the oracle on the aliased model;
    fp32 with ONE slot is the paper's precision under the <1 GB budget."""
    P = 2
    W = gen_model_weights(TINY, SEED, dtype=dtype)
    W["experts"] = {l: W["experts"][l % P] for l in range(TINY.L)}
    SW = O.quantize_model_int8(W)
    eng = engine(od, TINY, dtype, predictor=od.PRED_SHADOW_INT8, slots_per_gpu=slots, debug_capture=1,
                 expert_layer_period=P)
    st0 = eng.stats()
    blob = 3 * TINY.F * TINY.d * (2 if dtype == "bf16" else 4)
    assert st0["pool_bytes"] == P * TINY.E * blob
    tok = int(gen_prompt(TINY, 1, 1)[0])
    excused = 0
    for n in range(8):
        b0 = eng.stats()["bytes_h2d"]
        nxt, recs = eng.decode_step(tok)
        excused += check_step_teacher_forced(eng, W, TINY, dtype, tok, nxt, SW)
        db = eng.stats()["bytes_h2d"] - b0
        assert db % blob == 0 and db >= TINY.L * TINY.k * blob   # whole blobs, aliased or not
        tok = nxt
    assert excused <= 2
    assert eng.stats()["max_resident"] <= slots
    eng.close()


def test_tiny_fp32_free_run_tokens(od):
    """fp32 path, 16 tokens x 4 prompts: every token equals the oracle's greedy token for the
    same input token (no KV state => per-token teacher forcing), barring near-ties."""
    W = gen_model_weights(TINY, SEED, dtype="fp32")
    eng = engine(od, TINY, "fp32", predictor=od.PRED_NONE, slots_per_gpu=2)
    bad = 0
    for q in range(4):
        tok = int(gen_prompt(TINY, q + 1, 1)[0])
        for _ in range(16):
            nxt, _ = eng.decode_step(tok)
            ref, _, z = O.decode_token(W, tok, TINY.k)
            if nxt != ref:
                zs = np.sort(z)[::-1]
                assert abs(zs[0] - zs[1]) < 1e-3 * abs(zs[0])
                bad += 1
            tok = nxt
    assert bad <= 1
    eng.close()


def _run(od, shape, n, first, dtype="bf16", **kw):
    eng = engine(od, shape, dtype, **kw)
    toks, routes, t = [], [], first
    for _ in range(n):
        t, recs = eng.decode_step(t)
        toks.append(t)
        routes.append([tuple(r.true_ids[: shape.k]) for r in recs])
    st = eng.stats()
    return eng, toks, routes, st


def test_output_invariance_across_predictors_slots_and_modes(od):
    """Placement, prediction and loading change time, never values: bitwise
    identical tokens and routing for every predictor, slot budget, lookahead and the
    fully-resident baseline."""
    first = int(gen_prompt(TINY, 3, 1)[0])
    base_eng, base, base_r, _ = _run(od, TINY, 12, first, predictor=od.PRED_NONE, slots_per_gpu=2)
    base_eng.close()
    for kw in (dict(predictor=od.PRED_SHADOW_INT8, slots_per_gpu=2),
               dict(predictor=od.PRED_SHADOW_INT8, slots_per_gpu=5, lookahead=3),
               dict(predictor=od.PRED_RANDOM, slots_per_gpu=3, lookahead=2),
               dict(predictor=od.PRED_SHADOW_SAME, slots_per_gpu=4, lookahead=2),
               dict(predictor=od.PRED_NONE, slots_per_gpu=-1),
               dict(predictor=od.PRED_SHADOW_INT8, slots_per_gpu=2, chunk_bytes=65536),
               dict(predictor=od.PRED_SHADOW_INT8, slots_per_gpu=4, lookahead=2, refine_depth=2),
               dict(predictor=od.PRED_SHADOW_INT8, slots_per_gpu=2, refine_depth=1),
               dict(predictor=od.PRED_GATE_REUSE, slots_per_gpu=4, lookahead=2),
               dict(predictor=od.PRED_SHADOW_INT8, slots_per_gpu=1),          # fewer slots than k:
               dict(predictor=od.PRED_RANDOM, slots_per_gpu=1, lookahead=3)):  # deferred loads
        eng, toks, routes, _ = _run(od, TINY, 12, first, **kw)
        assert toks == base, kw
        assert routes == base_r, kw
        eng.close()


def test_same_precision_shadow_recall_exactly_one(od):
    eng, toks, _, st = _run(od, TINY, 10, 5, predictor=od.PRED_SHADOW_SAME, slots_per_gpu=4, lookahead=2)
    assert st["predicted_total"] == 10 * TINY.L * TINY.k
    assert st["correct"] == st["predicted_total"]
    eng.close()


BLOB_TINY = 3 * TINY.d * TINY.F * 2   # bytes of one bf16 expert


def _sets(arr, k=8):
    return sorted(int(x) for x in arr[:k] if x >= 0)


def _step_loads(eng, tok):
    """One decode step; (token, records, loads issued, bytes copied) of that step."""
    st0 = eng.stats()
    nxt, recs = eng.decode_step(tok)
    st1 = eng.stats()
    return nxt, recs, st1["loads_issued"] - st0["loads_issued"], st1["bytes_h2d"] - st0["bytes_h2d"]


@pytest.mark.parametrize("pred", ["perfect", "same", "random", "shadow_int8"])
def test_loader_accounting_exact(od, pred):
    """Loader accounting (SURVEY §8(c) a6 <-> a12), per decode token:
    the loads the loader performed equal O.expected_loads(true ids, loads issued before the router)
    exactly; every layer's reload set is O.misprediction_reloads; wherever the prediction reached
    the host in time (always for PERFECT / RANDOM at N = 1, 2 slots, D = 1) the issued set IS the
    prediction. PERFECT and the same-precision shadow therefore give exactly L*k loads and
    L*k*blob bytes per token whenever their predictions were in time."""
    p = od.PREDICTORS["shadow_same" if pred == "same" else pred]
    eng = engine(od, TINY, predictor=p, slots_per_gpu=2, lookahead=1, aux_seed=5)
    L, k = TINY.L, TINY.k
    first = 19
    if pred == "perfect":  # record the routing once
        t = first
        for _ in range(6):
            t, _ = eng.decode_step(t)
    t, full = first, 0
    for n in range(6):
        t_next, recs, loads, nbytes = _step_loads(eng, t)
        S = [_sets(r.true_ids, k) for r in recs]
        I = [_sets(r.issued_ids) for r in recs]
        assert loads == O.expected_loads(S, I), (n, loads, S, I)
        for l, r in enumerate(recs):
            rel = O.misprediction_reloads(S[l], {e: 0 for e in I[l]})
            assert _sets(r.reload_ids) == sorted(e for e, _ in rel), (n, l)
            assert r.n_reloads == len(rel)
            if r.pred_in_time:
                assert I[l] == _sets(r.pred_ids, k), (n, l)
            assert r.correct_in_time == (r.correct if r.pred_in_time else 0)
        if pred in ("perfect", "random"):
            assert all(r.pred_in_time for r in recs)
        if pred in ("perfect", "same") and all(r.pred_in_time for r in recs):
            assert loads == L * k and nbytes == L * k * BLOB_TINY
            full += 1
        if pred == "shadow_int8":  # recall accounting from the records, Eq. 3 numerator
            assert sum(r.correct for r in recs) == sum(len(set(S[l]) & set(_sets(r.pred_ids, k))) for l, r in enumerate(recs))
        t = t_next
    if pred == "perfect":
        assert full == 6
    eng.close()


@pytest.mark.parametrize("kw", [dict(predictor=2, slots_per_gpu=4, lookahead=2),
                                dict(predictor=2, slots_per_gpu=2, lookahead=1),
                                dict(predictor=0, slots_per_gpu=5, lookahead=3),
                                dict(predictor=0, slots_per_gpu=4, lookahead=2, refine_depth=2)])
def test_lookahead_window_and_trace_consistency(od, kw):
    """Reading Q11: no load is ever issued for a layer beyond l_cur + D; the event trace
     is consistent: every issued load has start/end events, a landed load copied one
    blob, an expert starts only after its load ended and after its layer's routing is known, and
    the slot count audit holds."""
    eng = engine(od, TINY, **kw)
    eng.set_trace(True)
    D = kw["lookahead"]
    t = 23
    for _ in range(5):
        t, recs = eng.decode_step(t)
    ev = eng.trace()
    eng.close()
    issues = [e for e in ev if e["type"] == "LoadIssue"]
    assert issues
    for e in issues:
        assert e["layer"] <= max(e["l_cur"], 0) + D, e
    ends = {}
    for e in ev:
        if e["type"] == "LoadEnd":
            ends.setdefault((e["step"], e["layer"], e["expert"]), []).append(e)
    cancelled = {(e["step"], e["layer"], e["expert"]) for e in ev if e["type"] == "LoadCancel"}
    n_end = sum(1 for e in ev if e["type"] == "LoadEnd")
    assert n_end == len(issues) == sum(1 for e in ev if e["type"] == "LoadStart")
    router = {(e["step"], e["layer"]): e["t_us"] for e in ev if e["type"] == "RouterDone"}
    starts = {}
    for e in ev:
        if e["type"] == "LoadStart":
            starts.setdefault((e["step"], e["layer"], e["expert"]), []).append(e["t_us"])
    cend = {(e["step"], e["layer"], e["expert"]): e["t_us"] for e in ev if e["type"] == "ComputeEnd"}
    for e in ev:
        if e["type"] == "ComputeStart":   # (fused kernel: after the whole blob; split: after W13)
            key = (e["step"], e["layer"], e["expert"])
            landed = [x for x in ends[key] if x["bytes"] == BLOB_TINY]
            assert landed, key
            assert e["t_us"] >= max(starts[key]) - 2.0, key   # event resolution ~0.5 us
            assert cend[key] >= max(x["t_us"] for x in landed) - 2.0, key
            assert e["t_us"] >= router[(e["step"], e["layer"])] - 2.0
    for key, es in ends.items():
        for x in es:
            assert x["bytes"] == BLOB_TINY or key in cancelled, (key, x)
    assert sum(1 for e in ev if e["type"] == "StepEnd") == 5


def test_predict_ahead_cache_follows_decode(od):
    """odmoe_predict_ahead caches one shadow pass per token; a decode step in between overwrites the
    shadow's buffers, so predict_ahead(a), decode_step(b), predict_ahead(a) must recompute."""
    eng = engine(od, TINY, predictor=od.PRED_SHADOW_INT8, slots_per_gpu=2)
    a, b = 33, 71
    Pa = eng.predict_ahead(a)
    _, recs_b = eng.decode_step(b)
    assert eng.predict_ahead(a) == Pa
    Pb = eng.predict_ahead(b)
    assert [sorted(x) for x in Pb] == [sorted(r.pred_ids[: TINY.k]) for r in recs_b]
    eng.close()


def test_random_predictor_recall_closed_form(od):
    """random prefetch recall ~ k/E = 0.25 (closed form for uniform k-subsets)."""
    n = 64
    eng, _, _, st = _run(od, TINY, n, 7, predictor=od.PRED_RANDOM, slots_per_gpu=2, aux_seed=11)
    r = st["correct"] / st["predicted_total"]
    p = TINY.k / TINY.E
    sigma = (p * (1 - p) / (TINY.k * TINY.L * n)) ** 0.5
    assert abs(r - p) < 4 * sigma * 1.5, r
    eng.close()


def test_perfect_predictor_replays_routing(od):
    eng = engine(od, TINY, predictor=od.PRED_PERFECT, slots_per_gpu=4, lookahead=2)
    t = 9
    seq = []
    for _ in range(6):
        t, _ = eng.decode_step(t)
        seq.append(t)
    eng.reset_stats()
    t = 9
    for _ in range(6):
        t, recs = eng.decode_step(t)
    st = eng.stats()
    assert st["correct"] == st["predicted_total"] == 6 * TINY.L * TINY.k
    eng.close()


def test_loader_roundtrip_bytes(od):
    """odmoe_load / load_wait / evict: the slot holds exactly the generator's bytes (H2D path)."""
    from tests.gpu_util import d2h, w13_interleaved
    eng = engine(od, TINY, predictor=od.PRED_NONE, slots_per_gpu=2)
    F, d = TINY.F, TINY.d
    n = 3 * F * d
    for (l, e) in [(0, 0), (3, 7), (2, 5)]:
        eng.load(l, e)
        p13, p2 = eng.load_wait(l, e)
        assert p2 - p13 == 2 * 2 * F * d
        raw = np.frombuffer(d2h(p13, 2 * n), dtype=np.uint16)
        got = (raw.astype(np.uint32) << 16).view(np.float32)
        W1, W3, W2 = gen_expert(TINY, SEED, l, e, "bf16")
        assert np.array_equal(got[: 2 * F * d].reshape(F, 2, d), w13_interleaved(W1, W3))
        assert np.array_equal(got[2 * F * d:].reshape(d, F), W2)
        eng.evict(l, e)
    with pytest.raises(od.OdmoeError):
        eng.evict(0, 0)
    eng.load(1, 1)
    eng.load(1, 2)
    with pytest.raises(od.OdmoeError):
        eng.load(1, 3)  # E_BUDGET: both slots occupied
    eng.close()


def test_predict_ahead_matches_decode_records(od):
    eng = engine(od, TINY, predictor=od.PRED_SHADOW_INT8, slots_per_gpu=2)
    P = eng.predict_ahead(33)
    nxt, recs = eng.decode_step(33)
    for l in range(TINY.L):
        assert sorted(P[l]) == sorted(recs[l].pred_ids[: TINY.k])
    assert eng.predict_ahead(33, 1, 2) == P[1:3]
    eng.close()


def test_config_errors(od):
    with pytest.raises(od.OdmoeError) as ei:
        od.Engine(4, 8, 9, 256, 512, 1024)
    assert ei.value.status == 1
    with pytest.raises(od.OdmoeError):
        od.Engine(4, 8, 2, 250, 512, 1024)
    with pytest.raises(od.OdmoeError):
        od.Engine(4, 8, 2, 256, 512, 1024, world_size=3, rank=0)
    eng = engine(od, TINY, predictor=od.PRED_NONE)
    with pytest.raises(od.OdmoeError) as ei:
        eng.decode_step(TINY.V)
    assert ei.value.status == 2
    eng.close()


# ------------------------------------------------------------------ Mixtral shape (full size)
@pytest.mark.slow
def test_mixtral_decode_sampled_layers(od):
    """BASELINE.json configs[1] shape in the bench's launch configuration (1 GPU, 2 slots,
    INT8 shadow): two decode steps; teacher-forced oracle checks on sampled layers (the oracle
    regenerates those experts itself from the seed)."""
    shape = MIXTRAL
    eng = engine(od, shape, "bf16", predictor=od.PRED_SHADOW_INT8, slots_per_gpu=2, debug_capture=1)
    tok = int(gen_prompt(shape, 1, 1)[0])
    W = gen_model_weights(shape, SEED, dtype="bf16", layers=[])  # emb + LM head (+ no layers)
    from inputs import KIND_ROUTER, tensor_id, weight_fp32, bf16_bits_to_f32, f32_to_bf16_bits
    for step in range(2):
        nxt, recs = eng.decode_step(tok)
        d, k, E = shape.d, shape.k, shape.E
        h0 = read_f32(eng, "H_IN", 0, d)
        assert np.array_equal(h0.astype(np.float32), W["emb"][tok])
        for l in ([0, 31] if step == 0 else [17]):
            Wg = bf16_bits_to_f32(f32_to_bf16_bits(weight_fp32(SEED, tensor_id(KIND_ROUTER, l), E, d, d))).reshape(E, d)
            h = read_f32(eng, "H_IN", l, d)
            u = read_u(eng, "U", l, d, "bf16")
            assert np.all(np.abs(u - O.rms_norm(h)) <= 2.0 ** -8 * np.abs(O.rms_norm(h)) + 1e-6)
            r_ref = O.router_logits(Wg, u)
            ids = read_i32(eng, "IDS", l, k)
            assert ids_match(ids, r_ref, k)[0]
            w = read_f32(eng, "W", l, k)
            yp = read_f32(eng, "Y_PART", l, k * d).reshape(k, d)
            for j in range(k):
                W1, W3, W2 = gen_expert(shape, SEED, l, int(ids[j]), "bf16")
                assert l2rel(yp[j], w[j] * O.expert_ffn(W1, W3, W2, u)) <= 1e-5
        z = read_f32(eng, "LM_LOGITS", 0, shape.V)
        z_ref = O.final_logits(W["lm_head"], read_f32(eng, "H_FINAL", 0, d))
        assert np.allclose(z, z_ref, rtol=0, atol=2e-2 * np.abs(z_ref).max())
        zs = np.sort(z_ref)[::-1]
        assert nxt == O.greedy_argmax(z_ref) or abs(zs[0] - zs[1]) < 1e-3 * abs(zs[0])
        tok = nxt
    st = eng.stats()
    assert st["max_resident"] <= 2 and st["resident_bytes"] < 1e9  # < 1 GB of experts per GPU
    eng.close()


@pytest.mark.slow
def test_mixtral_fp32_one_slot_sampled_layers(od):
    """The FP32 bench leg's launch configuration (`bench.py --dtype fp32`: the paper's precision,
    P:173; ONE 704.6 MB slot under the 1 GB budget; expert_layer_period 16, INT8
    shadow): two decode steps, teacher-forced oracle checks on sampled layers, including layers >= 16
    whose experts are those of layer l - 16 (fp32 tolerance 1e-5)."""
    shape = MIXTRAL
    P = 16
    eng = engine(od, shape, "fp32", predictor=od.PRED_SHADOW_INT8, slots_per_gpu=1, debug_capture=1,
                 expert_layer_period=P)
    tok = int(gen_prompt(shape, 1, 1)[0])
    W = gen_model_weights(shape, SEED, dtype="fp32", layers=[])
    from inputs import KIND_ROUTER, tensor_id, weight_fp32
    blob = 3 * shape.d * shape.F * 4
    for step in range(2):
        b0 = eng.stats()["bytes_h2d"]
        nxt, recs = eng.decode_step(tok)
        assert eng.stats()["bytes_h2d"] - b0 >= shape.L * shape.k * blob  # every load a whole fp32 blob
        d, k, E = shape.d, shape.k, shape.E
        for l in ([3, 19] if step == 0 else [31]):
            Wg = weight_fp32(SEED, tensor_id(KIND_ROUTER, l), E, d, d).reshape(E, d).astype(np.float64)
            h = read_f32(eng, "H_IN", l, d)
            u = read_u(eng, "U", l, d, "fp32")
            assert np.all(np.abs(u - O.rms_norm(h)) <= 1e-6 * np.abs(O.rms_norm(h)) + 1e-6)
            r_ref = O.router_logits(Wg, u)
            ids = read_i32(eng, "IDS", l, k)
            assert ids_match(ids, r_ref, k)[0]
            w = read_f32(eng, "W", l, k)
            yp = read_f32(eng, "Y_PART", l, k * d).reshape(k, d)
            for j in range(k):
                W1, W3, W2 = gen_expert(shape, SEED, l % P, int(ids[j]), "fp32")
                assert l2rel(yp[j], w[j] * O.expert_ffn(W1, W3, W2, u)) <= 1e-5
        z = read_f32(eng, "LM_LOGITS", 0, shape.V)
        z_ref = O.final_logits(W["lm_head"], read_f32(eng, "H_FINAL", 0, d))
        assert np.allclose(z, z_ref, rtol=0, atol=1e-4 * np.abs(z_ref).max())
        zs = np.sort(z_ref)[::-1]
        assert nxt == O.greedy_argmax(z_ref) or abs(zs[0] - zs[1]) < 1e-3 * abs(zs[0])
        tok = nxt
    st = eng.stats()
    assert st["max_resident"] <= 1 and st["resident_bytes"] < 1e9  # one fp32 slot < 1 GB
    eng.close()


@pytest.mark.slow
def test_mixtral_shadow_sampled_layers(od):
    """The INT8 shadow at BASELINE.json configs[1] shape in the bench's launch configuration (the
    one-launch-per-phase multi-expert kernel over the quantised experts): on sampled layers its
    router input, routing and expert output (h_{l+1} - h_l of the shadow's own residual stream)
    vs the oracle's int8-row shadow (quantize_model_int8 applied to the regenerated weights)."""
    from inputs import KIND_ROUTER, tensor_id, weight_fp32, bf16_bits_to_f32, f32_to_bf16_bits
    shape = MIXTRAL
    d, k, E = shape.d, shape.k, shape.E
    dq = lambda M: O.dequantize_int8_rows(*O.quantize_int8_rows(M))  # noqa: E731
    eng = engine(od, shape, "bf16", predictor=od.PRED_SHADOW_INT8, slots_per_gpu=2, debug_capture=1)
    tok = int(gen_prompt(shape, 2, 1)[0])
    eng.decode_step(tok)
    for l in (0, 13):
        Wg = bf16_bits_to_f32(f32_to_bf16_bits(weight_fp32(SEED, tensor_id(KIND_ROUTER, l), E, d, d))).reshape(E, d)
        sh = read_f32(eng, "SH_H_IN", l, d)
        su = read_u(eng, "SH_U", l, d, "bf16")
        assert np.all(np.abs(su - O.rms_norm(sh)) <= 2.0 ** -8 * np.abs(O.rms_norm(sh)) + 1e-6)
        sr_ref = O.router_logits(dq(Wg), su)
        sl = read_f32(eng, "SH_LOGITS", l, E)
        assert np.allclose(sl, sr_ref, rtol=0, atol=1e-5 * np.abs(sr_ref).max() + 1e-7), l
        sids = read_i32(eng, "SH_IDS", l, k)
        assert ids_match(sids, sr_ref, k)[0], (l, sids, sr_ref)
        w = O.mixture_weights(sr_ref, [int(i) for i in sids])
        y_ref = np.zeros(d)
        for j in range(k):
            W1, W3, W2 = gen_expert(shape, SEED, l, int(sids[j]), "bf16")
            y_ref += w[j] * O.expert_ffn(dq(W1), dq(W3), dq(W2), su)
        y = read_f32(eng, "SH_H_IN", l + 1, d) - sh
        assert l2rel(y, y_ref) <= 1e-4, (l, l2rel(y, y_ref))
    eng.close()


def test_runtime_options_switch_predictor_and_lookahead(od):
    """odmoe_set_option: switching predictor / lookahead between steps changes time and recall
    accounting only; tokens stay identical."""
    first = 21
    eng = engine(od, TINY, predictor=od.PRED_SHADOW_INT8, slots_per_gpu=4, lookahead=1)
    seqs = []
    for pred, D in ((od.PRED_SHADOW_INT8, 1), (od.PRED_NONE, 2), (od.PRED_PERFECT, 3), (od.PRED_RANDOM, 1),
                    (od.PRED_SHADOW_INT8, 3)):
        eng.set_predictor(pred)
        eng.set_lookahead(D)
        eng.reset_stats()
        t, toks = first, []
        for _ in range(6):
            t, _ = eng.decode_step(t)
            toks.append(t)
        seqs.append(toks)
        st = eng.stats()
        if pred == od.PRED_PERFECT:
            assert st["correct"] == st["predicted_total"] > 0
        if pred == od.PRED_NONE:
            assert st["predicted_total"] == 0
    assert all(s == seqs[0] for s in seqs)
    with pytest.raises(od.OdmoeError):
        eng.set_predictor(od.PRED_SHADOW_SAME)  # no such shadow in this ctx
    with pytest.raises(od.OdmoeError):
        eng.set_lookahead(0)
    eng.close()


def test_sep_refinement_improves_prediction_accuracy(od):
    """Refinement ("Mode B"): predictions re-anchored at the main model's exact
    state are at least as accurate as the token-start shadow (Mode A) and never change outputs."""
    eng = engine(od, TINY, predictor=od.PRED_SHADOW_INT8, slots_per_gpu=4, lookahead=2, refine_depth=2)
    t = 5
    for _ in range(24):
        t, recs = eng.decode_step(t)
    st = eng.stats()
    assert st["refine_total"] > 0
    ra = st["correct"] / st["predicted_total"]
    rb = st["refine_correct"] / st["refine_total"]
    assert rb >= ra - 0.02, (ra, rb)
    eng.set_refine_depth(0)
    eng.reset_stats()
    t = 5
    for _ in range(4):
        t, _ = eng.decode_step(t)
    assert eng.stats()["refine_total"] == 0
    eng.close()


def test_gate_reuse_predictor(od):
    """Prior-work next-layer gate reuse as an ablation predictor: predictions
    exist for layers >= 1, recall is recomputed exactly from the records, outputs unchanged."""
    eng = engine(od, TINY, predictor=od.PRED_GATE_REUSE, slots_per_gpu=4, lookahead=2)
    t, hits, tot = 13, 0, 0
    for _ in range(12):
        t, recs = eng.decode_step(t)
        for l in range(TINY.L):
            if recs[l].pred_available:
                S, P = set(recs[l].true_ids[:2]), set(recs[l].pred_ids[:2])
                assert recs[l].correct == len(S & P)
                hits += recs[l].correct
                tot += 2
        assert not recs[0].pred_available  # nothing precedes layer 0
    st = eng.stats()
    assert st["predicted_total"] == tot > 0 and st["correct"] == hits
    eng.close()


def test_bf16_shadow_of_fp32_model(od):
    """SEP with a BF16 shadow of the FP32 main model (the paper's FP16 shadow, P:86, P:164;
    reading Q26): teacher-forced shadow routing vs the oracle's bf16-rounded model, recall at
    least the INT8 shadow's on the same tokens, outputs identical to the no-predictor run."""
    W = gen_model_weights(TINY, SEED, dtype="fp32")
    SW = O.shadow_model_bf16(W)
    eng = engine(od, TINY, "fp32", predictor=od.PRED_SHADOW_BF16, slots_per_gpu=2, debug_capture=1)
    tok = int(gen_prompt(TINY, 2, 1)[0])
    first, toks, excused = tok, [], 0
    for _ in range(12):
        nxt, _ = eng.decode_step(tok)
        excused += check_step_teacher_forced(eng, W, TINY, "fp32", tok, nxt, SW)
        toks.append(nxt)
        tok = nxt
    assert excused <= 3
    st = eng.stats()
    r_bf16 = st["correct"] / st["predicted_total"]
    assert st["shadow_bytes"] < 0.6 * 4 * (TINY.L * TINY.E * 3 * TINY.d * TINY.F)
    eng.close()
    e8, toks8, _, st8 = _run(od, TINY, 12, first, dtype="fp32", predictor=od.PRED_SHADOW_INT8, slots_per_gpu=2)
    e8.close()
    en, toksn, _, _ = _run(od, TINY, 12, first, dtype="fp32", predictor=od.PRED_NONE, slots_per_gpu=2)
    en.close()
    assert toks == toks8 == toksn
    assert r_bf16 >= st8["correct"] / st8["predicted_total"] - 0.01, r_bf16
    assert r_bf16 >= 0.95, r_bf16
    with pytest.raises(od.OdmoeError):
        engine(od, TINY, "bf16", predictor=od.PRED_SHADOW_BF16)   # BF16 shadow needs an FP32 main model


@pytest.mark.parametrize("fmt", ["nf4", "fp8"])
@pytest.mark.parametrize("dims", [(256, 512), (1024, 2048)])
def test_lowbit_shadow_predictor(od, dims, fmt):
    """SEP with the NF4 shadow (reading Q27) and the FP8 shadow (Q28). TINY rows take
    the warp-per-row kernel, d=1024/F=2048 the flat one. Shadow routing teacher-forced against the
    oracle's quantised model (ids from the GPU's own shadow state), outputs identical to the
    no-predictor run, recall accounting exact."""
    d, F = dims
    shape = type(TINY)(TINY.L, TINY.E, TINY.k, d, F, TINY.V)
    W = gen_model_weights(shape, SEED, dtype="bf16")
    SW = O.quantize_model_nf4(W) if fmt == "nf4" else O.quantize_model_fp8(W)
    pred = od.PRED_SHADOW_NF4 if fmt == "nf4" else od.PRED_SHADOW_FP8
    eng = engine(od, shape, "bf16", predictor=pred, slots_per_gpu=2, debug_capture=1)
    tok = int(gen_prompt(shape, 4, 1)[0])
    first, toks, excused = tok, [], 0
    for _ in range(10):
        nxt, recs = eng.decode_step(tok)
        excused += check_step_teacher_forced(eng, W, shape, "bf16", tok, nxt, SW)
        for l in range(shape.L):
            assert recs[l].correct == len(set(recs[l].true_ids[:2]) & set(recs[l].pred_ids[:2]))
        toks.append(nxt)
        tok = nxt
    assert excused <= 3
    st = eng.stats()
    expert_bytes = shape.L * shape.E * 3 * d * F
    per_weight = 0.6 if fmt == "nf4" else 1.01                          # ~0.56 / ~1.0 B per weight
    assert st["shadow_bytes"] < per_weight * expert_bytes + 8 * shape.V * d
    eng.close()
    en, toksn, _, _ = _run(od, shape, 10, first, predictor=od.PRED_NONE, slots_per_gpu=2)
    en.close()
    assert toks == toksn
    print(fmt, "shadow recall", dims, st["correct"] / st["predicted_total"])


def test_resident_graph_replay_and_timer_levels(od):
    """The fully-resident 1-GPU step is captured into a CUDA graph on its second call and replayed;
    switching the timer level drops and recaptures it. Tokens equal the on-demand run throughout,
    and level 1 times exactly the expert launches (k per layer)."""
    first = 11
    ref_eng, ref, _, _ = _run(od, TINY, 10, first, predictor=od.PRED_NONE, slots_per_gpu=2)
    ref_eng.close()
    eng = engine(od, TINY, predictor=od.PRED_NONE, slots_per_gpu=-1, time_kernels=1)
    t, toks = first, []
    for i in range(10):
        if i == 5:
            st = eng.stats()
            assert st["n_w13"] == 5 * TINY.L * TINY.k and st["n_router"] == 0  # level 1: experts only
            eng.set_time_kernels(2)
        t, _ = eng.decode_step(t)
        toks.append(t)
    assert toks == ref
    assert eng.stats()["n_router"] > 0                                      # level 2: every family
    eng.close()


MID = type(TINY)(L=4, E=8, k=2, d=1024, F=2048, V=2048)   # rows of whole 512-byte groups: flat engine


def test_mid_shape_flat_engine_teacher_forced(od):
    """A shape whose rows are whole 512-byte groups, so every expert GEMV takes the flat engine:
    the fused cooperative bf16 expert kernel, the INT8 shadow's one-launch-per-phase multi-expert
    kernel, the refinement. Teacher-forced per layer vs the oracle, main and shadow."""
    W = gen_model_weights(MID, SEED, dtype="bf16")
    SW = O.quantize_model_int8(W)
    eng = engine(od, MID, "bf16", predictor=od.PRED_SHADOW_INT8, slots_per_gpu=2, refine_depth=2,
                 debug_capture=1)
    tok = int(gen_prompt(MID, 2, 1)[0])
    excused = 0
    for _ in range(4):
        nxt, recs = eng.decode_step(tok)
        excused += check_step_teacher_forced(eng, W, MID, "bf16", tok, nxt, SW)
        for l in range(MID.L):
            assert recs[l].correct == len(set(recs[l].true_ids[: MID.k]) & set(recs[l].pred_ids[: MID.k]))
        tok = nxt
    assert excused <= 2
    eng.close()


_MULTI_PROBE = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
from paper_2512_03927_b200 import odmoe as od
from inputs import gen_prompt
L, E, k, d, F, V = 4, 8, 2, 1024, 2048, 2048
eng = od.Engine(L, E, k, d, F, V, dtype=od.BF16, weight_seed=2512, predictor=od.PRED_SHADOW_INT8,
                slots_per_gpu=2, refine_depth=2, debug_capture=1)
tok, out = 7, []
for _ in range(3):
    tok, recs = eng.decode_step(tok)
    out.append(str(tok))
    for l in range(L):
        out.append(eng.debug_read("SH_LOGITS", l, 4 * E).hex())
        out.append(",".join(str(x) for x in recs[l].pred_ids[:k]))
eng.close()
print("|".join(out))
"""


@pytest.mark.parametrize("mma", ["0", "1"])
def test_shadow_multi_launch_equals_per_expert_launches(od, mma):
    """ODMOE_MULTI=0 (one launch per shadow expert) vs the default one launch per phase for the k
    experts. CUDA-core flat engine (ODMOE_SHADOW_MMA=0): every CTA takes the one-expert kernel's row
    range, so logits and predictions are bitwise identical. Tensor-core path: the k experts are one
    unit stream split evenly over the CTAs, so the fp32 summation order differs: identical
    predictions, logits within fp32 rounding."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for multi in ("0", "1"):
        env = dict(os.environ, ODMOE_MULTI=multi, ODMOE_SHADOW_MMA=mma)
        p = subprocess.run([sys.executable, "-c", _MULTI_PROBE.format(root=root)], env=env, capture_output=True,
                           text=True, timeout=600)
        assert p.returncode == 0, p.stderr[-2000:]
        res[multi] = p.stdout.strip().splitlines()[-1]
    if mma == "0":
        assert res["0"] == res["1"]
        return
    a, b = res["0"].split("|"), res["1"].split("|")
    assert len(a) == len(b)
    for x, y in zip(a, b):
        if len(x) == 64:   # shadow logits (8 fp32, hex)
            fx = np.frombuffer(bytes.fromhex(x), dtype=np.float32)
            fy = np.frombuffer(bytes.fromhex(y), dtype=np.float32)
            assert np.max(np.abs(fx - fy)) <= 2e-4 * np.max(np.abs(fx)) + 1e-7   # 12 chained shadow layers
        else:              # tokens and predicted ids
            assert x == y
