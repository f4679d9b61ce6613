"""Stateless kernels through the C ABI vs the CPU oracle (-m gpu).

Sizes: the tiny shape (several tiles + ragged tails) and the Mixtral shape (d=4096, F=14336,
E=8, V=32000) at BASELINE.json's full sizes for single experts/routers."""
import numpy as np
import pytest

import oracle as O
from inputs import (MIXTRAL, TINY, KIND_EMB, KIND_ROUTER, KIND_W1, KIND_W2, KIND_W3, bf16_bits_to_f32,
                    f32_to_bf16_bits, gen_expert, gen_hidden, tensor_id, weight_fp32, weight_bf16_bits)
from tests.gpu_util import TOL_BF16, TOL_FP32, assert_close, host, ids_match, l2rel, to_dev, torch, w13_interleaved

pytestmark = pytest.mark.gpu

SEED = 2512


@pytest.fixture(scope="module")
def od():
    t = torch()
    assert t.cuda.is_available(), "gpu tests need a B200"
    from paper_2512_03927_b200 import odmoe
    return odmoe


def stored(x, dtype):
    return bf16_bits_to_f32(f32_to_bf16_bits(x)).reshape(x.shape) if dtype == "bf16" else x


# ------------------------------------------------------------------ generator (shared recipe)
@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_generator_matches_inputs_module(od, dtype):
    t = torch()
    dt = od.BF16 if dtype == "bf16" else od.FP32
    # a plain tensor (router of layer 3) and the interleaved expert blob of (1, 5), tiny shape
    E, d, F = TINY.E, TINY.d, TINY.F
    out = t.empty((E, d), dtype=t.bfloat16 if dtype == "bf16" else t.float32, device="cuda")
    od.gen_weights(out, 2, layer=3, rows=E, cols=d, fan_in=d, seed=SEED, dtype=dt)
    ref = weight_fp32(SEED, tensor_id(KIND_ROUTER, 3), E, d, d)
    assert np.array_equal(host(out), stored(ref, dtype))
    blob = t.empty(3 * F * d, dtype=out.dtype, device="cuda")
    od.gen_weights(blob, 0, layer=1, expert=5, d=d, F=F, seed=SEED, dtype=dt)
    W1, W3, W2 = gen_expert(TINY, SEED, 1, 5, dtype)
    b = host(blob)
    assert np.array_equal(b[: 2 * F * d].reshape(F, 2, d), w13_interleaved(W1, W3))
    assert np.array_equal(b[2 * F * d:].reshape(d, F), W2)


# ------------------------------------------------------------------ quantiser (integer: bit-exact)
@pytest.mark.parametrize("shape", [(37, 256), (64, 4096), (4096, 14336)])
def test_quantizer_bit_exact(od, shape):
    t = torch()
    R, C = shape
    W = weight_bf16_bits(SEED, tensor_id(KIND_W2, 0, R % 7), R, C, C)
    Wf = bf16_bits_to_f32(W).reshape(R, C).copy()
    Wf[3 % R] = 0.0  # a zero row: q = 0, s = 1
    if R > 5:
        Wf[5, :3] = [Wf[5].max() * 2, -Wf[5].max() * 2, Wf[5].max()]  # exact half ties after scaling
    q_ref, s_ref = O.quantize_int8_rows(Wf.astype(np.float64))
    wd = to_dev(Wf, "bf16")
    q = t.empty((R, C), dtype=t.int8, device="cuda")
    s = t.empty(R, dtype=t.float32, device="cuda")
    od.quantize_int8_rows(wd, q, s)
    t.cuda.synchronize()
    assert np.array_equal(q.cpu().numpy(), q_ref)
    assert np.array_equal(s.cpu().numpy(), s_ref)


# ------------------------------------------------------------------ router
def _router_case(od, shape, dtype, m, n_add, seed):
    t = torch()
    E, d, k = shape.E, shape.d, shape.k
    dt = od.BF16 if dtype == "bf16" else od.FP32
    Wg = stored(weight_fp32(SEED, tensor_id(KIND_ROUTER, seed), E, d, d), dtype)
    h = gen_hidden(seed, m, d, 1.0)
    ys = [gen_hidden(seed + 100 + i, m, d, 0.3) for i in range(n_add)]
    hd = t.from_numpy(h.copy()).cuda()
    yd = [t.from_numpy(y.copy()).cuda() for y in ys]
    u = t.empty((m, d), dtype=t.bfloat16 if dtype == "bf16" else t.float32, device="cuda")
    ids = t.empty((m, k), dtype=t.int32, device="cuda")
    w = t.empty((m, k), dtype=t.float32, device="cuda")
    lg = t.empty((m, E), dtype=t.float32, device="cuda")
    flag = t.zeros(1, dtype=t.int32, device="cuda")
    keep = od.route_topk(hd, to_dev(Wg, dtype), k, u, ids, w, lg, y_add=yd, dtype=dt, flag=flag)
    t.cuda.synchronize()
    del keep
    return h, ys, Wg, host(hd), host(u), ids.cpu().numpy(), host(w), host(lg), int(flag.item())


@pytest.mark.parametrize("shape,dtype,m", [(TINY, "bf16", 300), (TINY, "fp32", 300),
                                           (MIXTRAL, "bf16", 2000), (MIXTRAL, "fp32", 200)])
def test_route_topk_parity(od, shape, dtype, m):
    k = shape.k
    h, ys, Wg, h_new, u, ids, w, lg, flag = _router_case(od, shape, dtype, m, 2, 7)
    assert flag == 0
    # residual: h + (y0 + y1), exactly as the fp32 adds
    want_h = (h + (ys[0] + ys[1]).astype(np.float32)).astype(np.float32)
    assert np.array_equal(h_new.astype(np.float32), want_h)
    excused = 0
    for r in range(m):
        u_ref = O.rms_norm(h_new[r])
        tol = 2.0 ** -8 if dtype == "bf16" else 1e-6
        assert np.all(np.abs(u[r] - u_ref) <= tol * np.abs(u_ref) + 1e-6), r
        # teacher forcing: logits from the GPU's rounded u
        r_ref = O.router_logits(Wg, u[r])
        assert np.allclose(lg[r], r_ref, rtol=0, atol=1e-5 * np.abs(r_ref).max() + 1e-7)
        ok, diff = ids_match(ids[r], r_ref, k)
        assert ok, (r, ids[r], r_ref)
        excused += diff
        w_ref = O.mixture_weights(r_ref, list(ids[r]))
        assert np.allclose(w[r], w_ref, atol=2e-6)
        assert abs(w[r].sum() - 1.0) < 1e-6
    assert excused <= max(2, m // 200)


@pytest.mark.parametrize("E,k,d,dtype,n_add", [(8, 2, 4096, "bf16", 2), (8, 2, 256, "bf16", 0), (8, 2, 4096, "fp32", 1),
                                               (64, 8, 1024, "bf16", 2), (64, 1, 512, "bf16", 2), (16, 4, 2048, "fp32", 3),
                                               (2, 2, 256, "bf16", 2)])
def test_decode_router_parity(od, E, k, d, dtype, n_add):
    """The decode step's router (m = 1: the 8-CTA cluster kernel with DSMEM reductions and warp-shuffle
    top-k) at the limits the ABI allows (E up to 64, k up to 8, k = E, k = 1): residual bit-exact, u
    within bf16 rounding of RMSNorm(h), logits element-wise, ids by the near-tie rule, mixture weights;
    40 independent rows (one launch each)."""
    t = torch()
    shape = type(TINY)(TINY.L, E, k, d, TINY.F, TINY.V)
    excused = 0
    for seed in range(40):
        h, ys, Wg, h_new, u, ids, w, lg, flag = _router_case(od, shape, dtype, 1, n_add, 300 + seed)
        assert flag == 0
        want = h.copy()
        if n_add:
            s = ys[0].astype(np.float32)
            for y in ys[1:]:
                s = (s + y.astype(np.float32)).astype(np.float32)
            want = (h + s).astype(np.float32)
        assert np.array_equal(h_new.astype(np.float32), want.astype(np.float32))
        u_ref = O.rms_norm(h_new[0])
        tol = 2.0 ** -8 if dtype == "bf16" else 1e-6
        assert np.all(np.abs(u[0] - u_ref) <= tol * np.abs(u_ref) + 1e-6)
        r_ref = O.router_logits(Wg, u[0])
        assert np.allclose(lg[0], r_ref, rtol=0, atol=1e-5 * np.abs(r_ref).max() + 1e-7)
        ok, exc = ids_match(ids[0], r_ref, k)
        assert ok, (seed, ids[0], r_ref)
        excused += exc
        assert np.allclose(w[0], O.mixture_weights(r_ref, list(ids[0])), atol=2e-6)
    assert excused <= 2


def test_decode_router_ties_and_nonfinite(od):
    """m = 1: exact ties go to the lower expert index; a non-finite logit sets the flag."""
    t = torch()
    E, d, k = 8, 1024, 2
    Wg = stored(weight_fp32(SEED, tensor_id(KIND_ROUTER, 11), E, d, d), "bf16")
    Wg[5] = Wg[2]
    Wg[7] = Wg[2]
    for seed in range(16):
        h = gen_hidden(40 + seed, 1, d)
        hd = t.from_numpy(h.copy()).cuda()
        u = t.empty((1, d), dtype=t.bfloat16, device="cuda")
        ids = t.empty((1, k), dtype=t.int32, device="cuda")
        w = t.empty((1, k), dtype=t.float32, device="cuda")
        od.route_topk(hd, to_dev(Wg, "bf16"), k, u, ids, w)
        t.cuda.synchronize()
        ref = O.top_k(O.router_logits(Wg, host(u)[0]), k)
        assert list(ids.cpu().numpy()[0]) == ref
    h = gen_hidden(7, 1, d)
    h[0, 3] = np.inf
    hd = t.from_numpy(h.copy()).cuda()
    flag = t.zeros(1, dtype=t.int32, device="cuda")
    od.route_topk(hd, to_dev(Wg, "bf16"), k, u, ids, w, flag=flag)
    t.cuda.synchronize()
    assert int(flag.item()) == 1


def test_route_topk_constructed_ties(od):
    t = torch()
    E, d, k = 8, 256, 2
    Wg = stored(weight_fp32(SEED, tensor_id(KIND_ROUTER, 9), E, d, d), "bf16")
    Wg[5] = Wg[2]  # exact tie between experts 2 and 5
    Wg[7] = Wg[2]
    h = gen_hidden(3, 64, d)
    hd = t.from_numpy(h.copy()).cuda()
    u = t.empty((64, d), dtype=t.bfloat16, device="cuda")
    ids = t.empty((64, k), dtype=t.int32, device="cuda")
    w = t.empty((64, k), dtype=t.float32, device="cuda")
    od.route_topk(hd, to_dev(Wg, "bf16"), k, u, ids, w)
    t.cuda.synchronize()
    ids = ids.cpu().numpy()
    uh = host(u)
    for r in range(64):
        ref = O.top_k(O.router_logits(Wg, uh[r]), k)
        assert list(ids[r]) == ref
        if 2 in ids[r]:
            assert 5 not in ids[r] or list(ids[r]) == [2, 5]


# ------------------------------------------------------------------ expert FFN
@pytest.mark.parametrize("shape,dtype", [(TINY, "bf16"), (TINY, "fp32"), (MIXTRAL, "bf16"), (MIXTRAL, "fp32")])
def test_expert_ffn_parity(od, shape, dtype):
    t = torch()
    d, F = shape.d, shape.F
    dt = od.BF16 if dtype == "bf16" else od.FP32
    W1, W3, W2 = gen_expert(shape, SEED, 2, 3, dtype)
    w13 = to_dev(w13_interleaved(W1, W3), dtype)
    w2 = to_dev(W2, dtype)
    errs = []
    for trial in range(3):
        u_f = stored(O.rms_norm(gen_hidden(50 + trial, 1, d)[0]).astype(np.float32), dtype)
        ud = to_dev(u_f, dtype)
        gate = t.tensor([0.25, 0.75], dtype=t.float32, device="cuda")
        a = t.empty(F, dtype=t.float32, device="cuda")
        y = t.empty(d, dtype=t.float32, device="cuda")
        od.expert_ffn(w13, w2, ud, a, y, gate_w=gate, gate_idx=1, dtype=dt)
        t.cuda.synchronize()
        ref = 0.75 * O.expert_ffn(W1, W3, W2, u_f)
        e = l2rel(host(y), ref)
        errs.append(e)
        assert e <= (TOL_BF16 if dtype == "bf16" else TOL_FP32), e
        # the design keeps a in fp32 and accumulates in fp32: far inside the bf16 bound
        assert e <= 1e-5
    # zero in -> zero out
    ud = to_dev(np.zeros(d, dtype=np.float32), dtype)
    od.expert_ffn(w13, w2, ud, a, y, dtype=dt)
    t.cuda.synchronize()
    assert float(y.abs().max()) == 0.0
    print("expert_ffn l2rel", shape, dtype, errs)


@pytest.mark.parametrize("shape", [TINY, MIXTRAL])
def test_shadow_expert_ffn_parity(od, shape):
    t = torch()
    d, F = shape.d, shape.F
    W1, W3, W2 = gen_expert(shape, SEED, 1, 6, "bf16")
    W13 = w13_interleaved(W1, W3).reshape(2 * F, d)
    q13, s13 = O.quantize_int8_rows(W13)
    q2, s2 = O.quantize_int8_rows(W2)
    u_f = stored(O.rms_norm(gen_hidden(77, 1, d)[0]).astype(np.float32), "bf16")
    a = t.empty(F, dtype=t.float32, device="cuda")
    y = t.empty(d, dtype=t.float32, device="cuda")
    cu = lambda x: t.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
    od.shadow_expert_ffn(cu(q13), cu(s13), cu(q2), cu(s2), to_dev(u_f, "bf16"), a, y)
    t.cuda.synchronize()
    dq13 = O.dequantize_int8_rows(q13, s13)
    ref = O.expert_ffn(dq13[0::2], dq13[1::2], O.dequantize_int8_rows(q2, s2), u_f)
    assert l2rel(host(y), ref) <= 1e-5


@pytest.mark.parametrize("dF", [(256, 512), (1024, 2048), (4096, 14336)])
def test_packed_shadow_expert_ffn_parity(od, dF):
    """The engine's INT8 shadow path on the tensor cores (reading Q32): the oracle's quantiser codes,
    packed into the mma fragment layout, give the dequantised oracle expert element by element
    (q exact in f16, x split hi/lo, fp32 accumulation)."""
    t = torch()
    d, F = dF
    shape = type(TINY)(TINY.L, TINY.E, TINY.k, d, F, TINY.V)
    W1, W3, W2 = gen_expert(shape, SEED, 2, 3, "bf16")
    W13 = w13_interleaved(W1, W3).reshape(2 * F, d)
    q13, s13 = O.quantize_int8_rows(W13)
    q2, s2 = O.quantize_int8_rows(W2)
    u_f = stored(O.rms_norm(gen_hidden(78, 1, d)[0]).astype(np.float32), "bf16")
    cu = lambda x: t.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
    p13 = t.empty(2 * F * d, dtype=t.uint8, device="cuda")
    p2 = t.empty(d * F, dtype=t.uint8, device="cuda")
    od.pack_int8_frag(cu(q13), p13, True)
    od.pack_int8_frag(cu(q2), p2, False)
    a = t.empty(F, dtype=t.float32, device="cuda")
    y = t.empty(d, dtype=t.float32, device="cuda")
    gw = t.tensor([0.25, 0.75], dtype=t.float32, device="cuda")
    od.shadow_expert_ffn_packed(p13, cu(s13), p2, cu(s2), to_dev(u_f, "bf16"), a, y, d, F, gate_w=gw, gate_idx=1)
    t.cuda.synchronize()
    dq13 = O.dequantize_int8_rows(q13, s13)
    a_ref = O.silu(dq13[0::2] @ u_f) * (dq13[1::2] @ u_f)
    ref = 0.75 * O.expert_ffn(dq13[0::2], dq13[1::2], O.dequantize_int8_rows(q2, s2), u_f)
    # a_scratch holds the SwiGLU activation in the tensor cores' B-fragment form (f16 hi + lo per
    # element, mma_gemv.cu store_frag): decode it
    hv = a.cpu().numpy().view(np.float16).astype(np.float64)
    p = np.arange(F)
    kb, c = p >> 4, p & 15
    tq, w, hf = (c & 7) >> 1, c >> 3, c & 1
    a_got = hv[((kb * 8 + tq) * 2 + w) * 2 + hf] + hv[((kb * 8 + 4 + tq) * 2 + w) * 2 + hf]
    assert_close(a_got, a_ref, 1e-5, what="a")
    assert_close(host(y), ref, 1e-5, what="y")


# ------------------------------------------------------------------ NF4 shadow (reading Q27)
@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
@pytest.mark.parametrize("shape", [(40, 256), (96, 4096 + 192), (28672, 4096)])
def test_nf4_quantizer_bit_exact(od, shape, dtype):
    """Codes and absmax identical to the oracle (integer decisions taken in fp64 on both sides)."""
    t = torch()
    R, C = shape
    Wf = stored(weight_fp32(SEED, tensor_id(KIND_W2, 1, R % 5), R, C, C), dtype).reshape(R, C).copy()
    Wf[1, 64:128] = 0.0                                    # an all-zero block -> code 7
    cb = np.asarray(O.NF4_CODEBOOK, dtype=np.float32)
    Wf[2, :64] = np.tile(cb, 4) * np.float32(0.25)         # codebook points (exact in bf16? kept as stored)
    Wf[2, :64] = stored(Wf[2, :64], dtype)
    q_ref, a_ref = O.quantize_nf4_blocks(Wf.astype(np.float64))
    packed_ref = (q_ref[:, 0::2] | (q_ref[:, 1::2] << 4)).astype(np.uint8)
    q = t.empty((R, C // 2), dtype=t.uint8, device="cuda")
    a = t.empty((R, C // 64), dtype=t.float32, device="cuda")
    od.quantize_nf4(to_dev(Wf, dtype), q, a, dtype=od.BF16 if dtype == "bf16" else od.FP32)
    t.cuda.synchronize()
    assert np.array_equal(a.cpu().numpy(), a_ref)
    assert np.array_equal(q.cpu().numpy(), packed_ref)


@pytest.mark.parametrize("dF", [(256, 512), (1024, 2048), (4096, 14336)])
def test_nf4_shadow_expert_ffn_parity(od, dF):
    """NF4 expert FFN vs the oracle's dequantised weights. (256, 512): warp-per-row kernel (fp32
    codebook, tol 1e-5); flat kernel: the codebook is held as fp16 pairs in shared memory
    (relative error <= 2^-11 per weight), tol 2^-10 on the l2-relative output."""
    t = torch()
    d, F = dF
    shape = type(TINY)(1, 8, 2, d, F, 1024)
    W1, W3, W2 = gen_expert(shape, SEED, 0, 3, "bf16")
    W13 = w13_interleaved(W1, W3).reshape(2 * F, d)
    q13, a13 = O.quantize_nf4_blocks(W13)
    q2, a2 = O.quantize_nf4_blocks(W2)
    pk = lambda q: np.ascontiguousarray((q[:, 0::2] | (q[:, 1::2] << 4)).astype(np.uint8))  # noqa: E731
    u_f = stored(O.rms_norm(gen_hidden(78, 1, d)[0]).astype(np.float32), "bf16")
    a = t.empty(F, dtype=t.float32, device="cuda")
    y = t.empty(d, dtype=t.float32, device="cuda")
    gw = t.tensor([0.75, 0.25], dtype=t.float32, device="cuda")
    cu = lambda x: t.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
    od.shadow_expert_ffn_nf4(cu(pk(q13)), cu(a13), cu(pk(q2)), cu(a2), to_dev(u_f, "bf16"), a, y, gate_w=gw, gate_idx=1)
    t.cuda.synchronize()
    dq13 = O.dequantize_nf4_blocks(q13, a13)
    ref = 0.25 * O.expert_ffn(dq13[0::2], dq13[1::2], O.dequantize_nf4_blocks(q2, a2), u_f)
    tol = 1e-5 if d % 1024 else 2.0 ** -10
    assert l2rel(host(y), ref) <= tol, l2rel(host(y), ref)


# ------------------------------------------------------------------ FP8 shadow (reading Q28)
@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
@pytest.mark.parametrize("shape", [(37, 256), (64, 4096), (4096, 14336)])
def test_fp8_quantizer_bit_exact(od, shape, dtype):
    t = torch()
    R, C = shape
    Wf = stored(weight_fp32(SEED, tensor_id(KIND_W1, 2, R % 3), R, C, C), dtype).reshape(R, C).copy()
    Wf[1] = 0.0
    q_ref, s_ref = O.quantize_fp8_rows(Wf.astype(np.float64))
    q = t.empty((R, C), dtype=t.uint8, device="cuda")
    s = t.empty(R, dtype=t.float32, device="cuda")
    od.quantize_fp8_rows(to_dev(Wf, dtype), q, s, dtype=od.BF16 if dtype == "bf16" else od.FP32)
    t.cuda.synchronize()
    assert np.array_equal(s.cpu().numpy(), s_ref)
    assert np.array_equal(q.cpu().numpy(), q_ref)


@pytest.mark.parametrize("dF", [(256, 512), (4096, 14336)])
def test_fp8_shadow_expert_ffn_parity(od, dF):
    """E4M3 values are exact in fp16, so the dequantisation is exact on both kernels: tol 1e-5."""
    t = torch()
    d, F = dF
    shape = type(TINY)(1, 8, 2, d, F, 1024)
    W1, W3, W2 = gen_expert(shape, SEED, 0, 5, "bf16")
    W13 = w13_interleaved(W1, W3).reshape(2 * F, d)
    q13, s13 = O.quantize_fp8_rows(W13)
    q2, s2 = O.quantize_fp8_rows(W2)
    u_f = stored(O.rms_norm(gen_hidden(79, 1, d)[0]).astype(np.float32), "bf16")
    a = t.empty(F, dtype=t.float32, device="cuda")
    y = t.empty(d, dtype=t.float32, device="cuda")
    cu = lambda x: t.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
    od.shadow_expert_ffn_fp8(cu(q13), cu(s13), cu(q2), cu(s2), to_dev(u_f, "bf16"), a, y)
    t.cuda.synchronize()
    dq13 = O.dequantize_fp8_rows(q13, s13)
    ref = O.expert_ffn(dq13[0::2], dq13[1::2], O.dequantize_fp8_rows(q2, s2), u_f)
    assert l2rel(host(y), ref) <= 1e-5, l2rel(host(y), ref)


def test_shadow_router_parity(od):
    t = torch()
    E, d, k = 8, 4096, 2
    Wg = stored(weight_fp32(SEED, tensor_id(KIND_ROUTER, 4), E, d, d), "bf16")
    q, s = O.quantize_int8_rows(Wg)
    m = 500
    h = gen_hidden(5, m, d)
    hd = t.from_numpy(h.copy()).cuda()
    u = t.empty((m, d), dtype=t.bfloat16, device="cuda")
    ids = t.empty((m, k), dtype=t.int32, device="cuda")
    w = t.empty((m, k), dtype=t.float32, device="cuda")
    lg = t.empty((m, E), dtype=t.float32, device="cuda")
    od.shadow_route_topk(hd, t.from_numpy(q).cuda(), t.from_numpy(s).cuda(), k, u, ids, w, lg)
    t.cuda.synchronize()
    uh, idsh, lgh = host(u), ids.cpu().numpy(), host(lg)
    Q = O.dequantize_int8_rows(q, s)
    for r in range(m):
        r_ref = O.router_logits(Q, uh[r])
        assert np.allclose(lgh[r], r_ref, rtol=0, atol=1e-5 * np.abs(r_ref).max())
        assert ids_match(idsh[r], r_ref, k)[0]


# ------------------------------------------------------------------ LM head + argmax
@pytest.mark.parametrize("shape,dtype", [(TINY, "bf16"), (MIXTRAL, "bf16"), (MIXTRAL, "fp32")])
def test_lm_head_argmax(od, shape, dtype):
    t = torch()
    V, d = shape.V, shape.d
    dt = od.BF16 if dtype == "bf16" else od.FP32
    W = stored(weight_fp32(SEED, tensor_id(6), V, d, d), dtype)
    Wd = to_dev(W, dtype)
    scratch = t.zeros(16 * 4096, dtype=t.uint8, device="cuda")
    tok = t.empty(1, dtype=t.int32, device="cuda")
    lg = t.empty(V, dtype=t.float32, device="cuda")
    for trial in range(4):
        h = gen_hidden(90 + trial, 1, d, 2.0)[0]
        od.lm_head_argmax(t.from_numpy(h.copy()).cuda(), Wd, tok, scratch, logits=lg, dtype=dt)
        t.cuda.synchronize()
        u = O.rms_norm(h)
        if dtype == "bf16":
            u = stored(u.astype(np.float32), "bf16").astype(np.float64)
        z = W.astype(np.float64) @ u
        assert np.allclose(host(lg), z, rtol=0, atol=1e-5 * np.abs(z).max())
        ref = O.greedy_argmax(z)
        if int(tok.item()) != ref:
            zs = np.sort(z)[::-1]
            assert abs(zs[0] - zs[1]) < 1e-3 * abs(zs[0]), (int(tok.item()), ref)
    # constructed tie: duplicate the winning row at a lower and a higher id
    W2 = W.copy()
    h = gen_hidden(99, 1, d, 2.0)[0]
    od.lm_head_argmax(t.from_numpy(h.copy()).cuda(), to_dev(W2, dtype), tok, scratch, dtype=dt)
    t.cuda.synchronize()
    win = int(tok.item())
    lo, hi = (1, V - 1) if win not in (1, V - 1) else (2, V - 2)
    W2[lo] = W2[win]
    W2[hi] = W2[win]
    od.lm_head_argmax(t.from_numpy(h.copy()).cuda(), to_dev(W2, dtype), tok, scratch, dtype=dt)
    t.cuda.synchronize()
    assert int(tok.item()) == min(lo, win)
