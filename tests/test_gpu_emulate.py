"""The multi-GPU expert arithmetic on ONE GPU (engine option emulate_world; SURVEY §8(e), §8(f)3;
P:104-126) teacher-forced per layer against the CPU oracle, element by element (-m gpu).

Sliced placement: every routed expert is computed as N F/N slices (O.sliced_expert_partials), each
emulated rank sums its k gated partials in router rank order and the N partials are summed in rank
order -- the launches, grids and summation order a real N-GPU run uses, so this checks the N > 1
data path on the driver's 1-GPU box. Paper's groups: each emulated rank of layer l's group
(l mod N_G) owns the experts the sorted pairing gives it (O.assign_experts)."""
import numpy as np
import pytest

import oracle as O
from inputs import TINY, gen_model_weights, gen_prompt
from tests.gpu_util import TOL_BF16, TOL_FP32, assert_close, ids_match, torch

pytestmark = pytest.mark.gpu
SEED = 2512
MID = type(TINY)(L=4, E=8, k=2, d=1024, F=2048, V=2048)


@pytest.fixture(scope="module")
def od():
    t = torch()
    assert t.cuda.is_available(), "gpu tests need a B200"
    from paper_2512_03927_b200 import odmoe
    return odmoe


def f32(eng, what, layer, n):
    return np.frombuffer(eng.debug_read(what, layer, 4 * n), dtype=np.float32).astype(np.float64)


def u_of(eng, layer, d, dtype):
    if dtype == "bf16":
        b = np.frombuffer(eng.debug_read("U", layer, 2 * d), dtype=np.uint16)
        return (b.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    return f32(eng, "U", layer, d)


def check_emulated_step(eng, W, shape, dtype, N, placement, G=None):
    L, k, d = shape.L, shape.k, shape.d
    tol = TOL_BF16 if dtype == "bf16" else TOL_FP32
    excused = 0
    for l in range(L):
        h = f32(eng, "H_IN", l, d)
        u = u_of(eng, l, d, dtype)
        r_ref = O.router_logits(W["router"][l], u)
        ids = [int(x) for x in np.frombuffer(eng.debug_read("IDS", l, 4 * k), dtype=np.int32)]
        ok, exc = ids_match(ids, r_ref, k)
        assert ok, (l, ids)
        excused += exc
        w = f32(eng, "W", l, k)
        yr = f32(eng, "Y_RANK", l, N * d).reshape(N, d)
        ref_rank = np.zeros((N, d))
        if placement == "sliced":
            for j, e in enumerate(ids):   # router rank order, as each rank sums
                parts = O.sliced_expert_partials(*W["experts"][l][e], u, N)
                for r in range(N):
                    ref_rank[r] += w[j] * parts[r]
        else:
            NG = N // G
            g = O.assign_layer(l, NG)
            owner = O.assign_experts(ids, O.plan_groups(N, G)[g])
            for j, e in enumerate(ids):
                ref_rank[owner[e]] += w[j] * O.expert_ffn(*W["experts"][l][e], u)
        for r in range(N):
            if np.any(ref_rank[r]):
                assert_close(yr[r], ref_rank[r], tol, what=("rank partial", l, r))
            else:
                assert not np.any(yr[r]), (l, r)
        y = f32(eng, "Y", l, d)
        assert_close(y, ref_rank.sum(axis=0), tol, what=("combined", l))
        h_next = f32(eng, "H_IN", l + 1, d) if l + 1 < L else f32(eng, "H_FINAL", 0, d)
        assert_close(h_next, h + ref_rank.sum(axis=0), tol, what=("h", l))
        # the combine itself is exactly the rank-order sum of the GPU's own partials (fp32, in order)
        s = yr[0].astype(np.float32)
        for r in range(1, N):
            s = (s + yr[r].astype(np.float32)).astype(np.float32)
        assert np.array_equal(s, y.astype(np.float32)), l
    return excused


@pytest.mark.parametrize("shape,dtype,N", [(TINY, "bf16", 2), (TINY, "bf16", 4), (TINY, "fp32", 4), (MID, "bf16", 2)])
def test_emulated_sliced_teacher_forced(od, shape, dtype, N):
    W = gen_model_weights(shape, SEED, dtype=dtype)
    eng = od.Engine(shape.L, shape.E, shape.k, shape.d, shape.F, shape.V, dtype=od.BF16 if dtype == "bf16" else od.FP32,
                    weight_seed=SEED, predictor=od.PRED_SHADOW_INT8, slots_per_gpu=2, debug_capture=1,
                    placement=od.PLACE_SLICED, emulate_world=N)
    tok, excused = int(gen_prompt(shape, 1, 1)[0]), 0
    for _ in range(4):
        nxt, recs = eng.decode_step(tok)
        excused += check_emulated_step(eng, W, shape, dtype, N, "sliced")
        tok = nxt
    st = eng.stats()
    eng.close()
    assert excused <= 2
    assert st["max_resident"] <= 2


@pytest.mark.parametrize("N,G", [(2, 2), (4, 2), (2, 1), (4, 1)])
def test_emulated_groups_teacher_forced(od, N, G):
    W = gen_model_weights(TINY, SEED, dtype="bf16")
    eng = od.Engine(TINY.L, TINY.E, TINY.k, TINY.d, TINY.F, TINY.V, dtype=od.BF16, weight_seed=SEED,
                    predictor=od.PRED_RANDOM, aux_seed=3, slots_per_gpu=2, debug_capture=1,
                    placement=od.PLACE_GROUPS, group_size=G, emulate_world=N)
    tok, excused = int(gen_prompt(TINY, 2, 1)[0]), 0
    for _ in range(4):
        nxt, _ = eng.decode_step(tok)
        excused += check_emulated_step(eng, W, TINY, "bf16", N, "groups", G)
        tok = nxt
    eng.close()
    assert excused <= 2


def test_emulated_groups_equal_single_gpu_bitwise(od):
    """The paper's placement at k = 2 combines two whole experts: a commutative two-term sum, so the
    emulated N = 2 / 4 runs give the 1-GPU run's tokens and final states bit for bit."""
    first = int(gen_prompt(TINY, 3, 1)[0])
    outs = []
    for N in (0, 2, 4):
        eng = od.Engine(TINY.L, TINY.E, TINY.k, TINY.d, TINY.F, TINY.V, dtype=od.BF16, weight_seed=SEED,
                        predictor=od.PRED_NONE, slots_per_gpu=2, debug_capture=1, placement=od.PLACE_GROUPS,
                        emulate_world=N)
        t, toks, hs = first, [], []
        for _ in range(6):
            t, _ = eng.decode_step(t)
            toks.append(t)
            hs.append(eng.debug_read("H_FINAL", 0, 4 * TINY.d))
        eng.close()
        outs.append((toks, hs))
    assert outs[1] == outs[0] and outs[2] == outs[0]


def test_emulate_world_config_errors(od):
    with pytest.raises(od.OdmoeError):
        od.Engine(TINY.L, TINY.E, TINY.k, TINY.d, TINY.F, TINY.V, emulate_world=3)
    with pytest.raises(od.OdmoeError):
        od.Engine(TINY.L, TINY.E, TINY.k, TINY.d, TINY.F, TINY.V, emulate_world=2, slots_per_gpu=-1)
    eng = od.Engine(TINY.L, TINY.E, TINY.k, TINY.d, TINY.F, TINY.V, emulate_world=2, placement=od.PLACE_SLICED,
                    predictor=od.PRED_NONE)
    with pytest.raises(od.OdmoeError):
        eng.prefill([1, 2, 3])
    eng.close()
