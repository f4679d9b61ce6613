"""Counter-based synthetic weight / prompt generator (numpy only).

Recipe (also in DESIGN.md §3):

* splitmix64(z): z += 0x9E3779B97F4A7C15; z = (z ^ z>>30) * 0xBF58476D1CE4E5B9;
  z = (z ^ z>>27) * 0x94D049BB133111EB; return z ^ z>>31   (all mod 2^64).
* stream base  b = splitmix64(splitmix64(seed) ^ tensor_id).
* element i    x_i = splitmix64(b + i);  u24 = x_i >> 40  (24 random bits).
* uniform      v_i = (2*u24 - (2^24 - 1)) * 2^-24   -- an odd multiple of 2^-24 in (-1, 1),
               exact in fp32, symmetric, never 0.
* weight       w_i = fl32(v_i * s), s = fl32(1/sqrt(fan_in)), one IEEE fp32 multiply (RNE);
               bf16 storage = round-to-nearest-even of w_i's fp32 bits.
* tensor_id    = kind << 40 | layer << 20 | expert.

Scales: U(+-1/sqrt(fan_in)) per matrix (reading Q23): embedding,
router, W1, W3 and LM head use fan_in = d; W2 uses fan_in = F.
Prompts: uniform ids in [1, V), id = 1 + (x_i >> 11) mod (V - 1).
"""
from __future__ import annotations

import dataclasses

import numpy as np

GOLDEN = 0x9E3779B97F4A7C15
_M1 = 0xBF58476D1CE4E5B9
_M2 = 0x94D049BB133111EB
MASK64 = (1 << 64) - 1

KIND_EMB = 1
KIND_ROUTER = 2
KIND_W1 = 3
KIND_W3 = 4
KIND_W2 = 5
KIND_LM_HEAD = 6
KIND_PROMPT = 7
KIND_HIDDEN = 8  # random test hidden states (router / expert unit tests)
KIND_WQ = 9      # attention projections (reading Q29): fan_in = d for all four
KIND_WK = 10
KIND_WV = 11
KIND_WO = 12


@dataclasses.dataclass(frozen=True)
class ModelShape:
    L: int
    E: int
    k: int
    d: int
    F: int
    V: int
    H: int = 0    # attention query heads (0 = no attention block, the round-1 hot path)
    Hkv: int = 0  # key/value heads (GQA); head_dim = d / H


# BASELINE.json configs[0] (V=1024 is SURVEY.md's proposal; BASELINE gives no vocab)
TINY = ModelShape(L=4, E=8, k=2, d=256, F=512, V=1024)
# Mixtral-8x7B shape (SURVEY.md §0 "Mixtral shape")
MIXTRAL = ModelShape(L=32, E=8, k=2, d=4096, F=14336, V=32000)
# with Mixtral's attention block (32 query heads, 8 KV heads, head_dim 128; reading Q29)
TINY_ATTN = ModelShape(L=4, E=8, k=2, d=256, F=512, V=1024, H=4, Hkv=2)
MIXTRAL_ATTN = ModelShape(L=32, E=8, k=2, d=4096, F=14336, V=32000, H=32, Hkv=8)


def splitmix64(z):
    """splitmix64 finaliser on a numpy uint64 array (wrapping arithmetic) or a Python int."""
    if isinstance(z, (int, np.integer)):
        z = (int(z) + GOLDEN) & MASK64
        z = ((z ^ (z >> 30)) * _M1) & MASK64
        z = ((z ^ (z >> 27)) * _M2) & MASK64
        return z ^ (z >> 31)
    z = z.astype(np.uint64, copy=True)
    with np.errstate(over="ignore"):
        z += np.uint64(GOLDEN)
        z ^= z >> np.uint64(30)
        z *= np.uint64(_M1)
        z ^= z >> np.uint64(27)
        z *= np.uint64(_M2)
        z ^= z >> np.uint64(31)
    return z


def tensor_id(kind: int, layer: int = 0, expert: int = 0) -> int:
    return (kind << 40) | (layer << 20) | expert


def _base(seed: int, tid: int) -> int:
    return splitmix64(splitmix64(seed) ^ tid)


def _u24_block(base, start, s, e, out):
    with np.errstate(over="ignore"):
        idx = np.arange(start + s, start + e, dtype=np.uint64) + base
    out[s:e] = (splitmix64(idx) >> np.uint64(40)).astype(np.uint32)


def stream_u24(seed: int, tid: int, n: int, start: int = 0, block: int = 1 << 22) -> np.ndarray:
    """u24 = splitmix64(base + i) >> 40 for i in [start, start+n), as uint32. Large tensors are
    generated block-parallel on a thread pool (numpy releases the GIL); the values do not depend
    on the blocking."""
    base = np.uint64(_base(seed, tid))
    out = np.empty(n, dtype=np.uint32)
    blocks = [(s, min(n, s + block)) for s in range(0, n, block)]
    if len(blocks) <= 2:
        for s, e in blocks:
            _u24_block(base, start, s, e, out)
        return out
    import concurrent.futures
    import os
    with concurrent.futures.ThreadPoolExecutor(max_workers=min(32, os.cpu_count() or 1)) as ex:
        list(ex.map(lambda se: _u24_block(base, start, se[0], se[1], out), blocks))
    return out


def uniform_pm1(seed: int, tid: int, n: int, start: int = 0) -> np.ndarray:
    """Odd multiples of 2^-24 in (-1, 1), exact in float32."""
    u = stream_u24(seed, tid, n, start).astype(np.int64)
    return ((2 * u - ((1 << 24) - 1)).astype(np.float32) * np.float32(2.0 ** -24)).astype(np.float32)


def fan_in_scale(fan_in: int) -> np.float32:
    return np.float32(1.0 / np.sqrt(np.float64(fan_in)))


def weight_fp32(seed: int, tid: int, rows: int, cols: int, fan_in: int) -> np.ndarray:
    v = uniform_pm1(seed, tid, rows * cols)
    return (v * fan_in_scale(fan_in)).astype(np.float32).reshape(rows, cols)


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16 bit pattern (uint16). Inputs are finite."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    r = ((u >> np.uint32(16)) & np.uint32(1)) + np.uint32(0x7FFF)
    return ((u + r) >> np.uint32(16)).astype(np.uint16)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.ascontiguousarray(b, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def weight_bf16_bits(seed: int, tid: int, rows: int, cols: int, fan_in: int) -> np.ndarray:
    return f32_to_bf16_bits(weight_fp32(seed, tid, rows, cols, fan_in))


def _stored(seed, tid, rows, cols, fan_in, dtype, block: int = 1 << 22):
    """Stored weight values (fp32, or bf16-rounded fp32). Same arithmetic as weight_fp32 +
    f32_to_bf16_bits, evaluated block-parallel on a thread pool."""
    n = rows * cols
    base = np.uint64(_base(seed, tid))
    scale = fan_in_scale(fan_in)
    out = np.empty(n, dtype=np.float32)

    def work(se):
        s_, e_ = se
        with np.errstate(over="ignore"):
            idx = np.arange(s_, e_, dtype=np.uint64) + base
        u = (splitmix64(idx) >> np.uint64(40)).astype(np.int64)
        w = ((2 * u - ((1 << 24) - 1)).astype(np.float32) * np.float32(2.0 ** -24)).astype(np.float32) * scale
        w = w.astype(np.float32)
        if dtype == "bf16":
            w = bf16_bits_to_f32(f32_to_bf16_bits(w))
        out[s_:e_] = w

    blocks = [(s_, min(n, s_ + block)) for s_ in range(0, n, block)]
    if len(blocks) <= 2:
        for b in blocks:
            work(b)
    else:
        import concurrent.futures
        import os
        with concurrent.futures.ThreadPoolExecutor(max_workers=min(32, os.cpu_count() or 1)) as ex:
            list(ex.map(work, blocks))
    return out.reshape(rows, cols)


def gen_expert(shape: ModelShape, seed: int, layer: int, expert: int, dtype: str = "bf16"):
    """(W1 [F,d], W3 [F,d], W2 [d,F]) as float32 arrays holding the STORED values
    (bf16-representable when dtype == 'bf16')."""
    d, F = shape.d, shape.F
    W1 = _stored(seed, tensor_id(KIND_W1, layer, expert), F, d, d, dtype)
    W3 = _stored(seed, tensor_id(KIND_W3, layer, expert), F, d, d, dtype)
    W2 = _stored(seed, tensor_id(KIND_W2, layer, expert), d, F, F, dtype)
    return W1, W3, W2


def gen_attention(shape: ModelShape, seed: int, layer: int, dtype: str = "bf16"):
    """(Wq [H*hd, d], Wk [Hkv*hd, d], Wv [Hkv*hd, d], Wo [d, H*hd]) stored values, hd = d / H."""
    d, hd = shape.d, shape.d // shape.H
    Wq = _stored(seed, tensor_id(KIND_WQ, layer), shape.H * hd, d, d, dtype)
    Wk = _stored(seed, tensor_id(KIND_WK, layer), shape.Hkv * hd, d, d, dtype)
    Wv = _stored(seed, tensor_id(KIND_WV, layer), shape.Hkv * hd, d, d, dtype)
    Wo = _stored(seed, tensor_id(KIND_WO, layer), d, shape.H * hd, d, dtype)
    return Wq, Wk, Wv, Wo


def gen_model_weights(shape: ModelShape, seed: int, dtype: str = "bf16", layers=None):
    """Dict of stored weights (float32 arrays): emb [V,d], router[l] [E,d],
    experts[l][e] = (W1, W3, W2), lm_head [V,d]; with shape.H > 0 also attn[l] = (Wq, Wk, Wv, Wo).
    gamma is 1 (reading Q7)."""
    d = shape.d
    layers = range(shape.L) if layers is None else layers
    w = {
        "emb": _stored(seed, tensor_id(KIND_EMB), shape.V, d, d, dtype),
        "lm_head": _stored(seed, tensor_id(KIND_LM_HEAD), shape.V, d, d, dtype),
        "router": {},
        "experts": {},
    }
    for l in layers:
        w["router"][l] = _stored(seed, tensor_id(KIND_ROUTER, l), shape.E, d, d, dtype)
        w["experts"][l] = {e: gen_expert(shape, seed, l, e, dtype) for e in range(shape.E)}
    if shape.H > 0:
        w["attn"] = {l: gen_attention(shape, seed, l, dtype) for l in layers}
        w["heads"] = (shape.H, shape.Hkv)
    return w


def gen_prompt(shape: ModelShape, aux_seed: int, length: int) -> np.ndarray:
    """Uniform token ids in [1, V) (prompts avoid EOS id 0)."""
    base = np.uint64(_base(aux_seed, tensor_id(KIND_PROMPT)))
    with np.errstate(over="ignore"):
        x = splitmix64(np.arange(length, dtype=np.uint64) + base)
    return (1 + (x >> np.uint64(11)) % np.uint64(shape.V - 1)).astype(np.int32)


def gen_hidden(seed: int, m: int, d: int, scale: float = 1.0) -> np.ndarray:
    """Random fp32 hidden states [m, d] for unit tests (uniform in (-scale, scale))."""
    return (uniform_pm1(seed, tensor_id(KIND_HIDDEN, 0, m), m * d) * np.float32(scale)).reshape(m, d)
