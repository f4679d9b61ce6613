"""Helpers for the -m gpu parity tests: move seeded inputs to the GPU and read results back.
Tolerances (north_star, BASELINE.json): ids exact except oracle near-ties (1e-3 relative gap),
hidden states l2-relative <= 2e-2 (bf16 path) / 1e-5 (fp32 path)."""
import numpy as np

import oracle as O
from inputs import f32_to_bf16_bits

TOL_BF16 = 2e-2
TOL_FP32 = 1e-5


def torch():
    import torch as t
    return t


def to_dev(x_f32: np.ndarray, dtype: str):
    """Stored (bf16-representable or fp32) float32 array -> CUDA tensor of that dtype."""
    t = torch()
    if dtype == "bf16":
        bits = f32_to_bf16_bits(np.ascontiguousarray(x_f32, dtype=np.float32))
        return t.from_numpy(bits.view(np.int16).copy()).cuda().view(t.bfloat16)
    return t.from_numpy(np.ascontiguousarray(x_f32, dtype=np.float32)).cuda()


def w13_interleaved(W1, W3):
    """[F, 2, d]: row 2f = W1 row f (gate), 2f+1 = W3 row f (up) -- the blob layout."""
    F, d = W1.shape
    out = np.empty((F, 2, d), dtype=np.float32)
    out[:, 0, :] = W1
    out[:, 1, :] = W3
    return out


def host(t):
    tt = torch()
    if t.dtype == tt.bfloat16:
        return t.float().cpu().numpy().astype(np.float64)
    return t.cpu().numpy().astype(np.float64)


def l2rel(x, ref):
    x = np.asarray(x, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    n = np.linalg.norm(ref)
    return float(np.linalg.norm(x - ref) / (n if n > 0 else 1.0))


def ids_match(gpu_ids, ref_logits, k):
    """(ok, excused): the GPU's top-k equals the oracle's, or differs from it only by swapping
    members of the tied run at the k/k+1 boundary (O.ids_excusable, pinned by
    tests/golden/near_tie_cases.json)."""
    return O.ids_excusable([int(x) for x in gpu_ids], ref_logits, k)


def token_match(gpu_token, ref_logits):
    """Greedy token: the oracle's argmax, or a member of the tied run at the top (k = 1 rule)."""
    return O.ids_excusable([int(gpu_token)], ref_logits, 1)


def maxabs_rel(x, ref):
    """max |x - ref| / max |ref| (SURVEY §8(c) Parity 3, reported beside the l2 error)."""
    x = np.asarray(x, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    m = np.max(np.abs(ref))
    return float(np.max(np.abs(x - ref)) / (m if m > 0 else 1.0))


# Element-wise bound for vectors whose inputs are teacher-forced bit for bit (bf16 or fp32 weights
# and u identical on both sides; the GPU accumulates in fp32 in another order): fp32 rounding only.
# One wrong output element out of d = 4096 moves max-abs by O(1), l2 only by 1/64.
TOL_ELEM = 1e-4


def assert_close(x, ref, tol_l2, tol_max=TOL_ELEM, what=""):
    e2, em = l2rel(x, ref), maxabs_rel(x, ref)
    assert e2 <= tol_l2 and em <= tol_max, (what, e2, em)
    return e2, em


def d2h(ptr: int, nbytes: int) -> bytes:
    """Synchronous device->host copy of a raw device pointer (ctx-owned memory), via the same
    CUDA runtime torch uses (shares the primary context)."""
    import ctypes
    import glob
    import os
    t = torch()
    lib = glob.glob(os.path.join(os.path.dirname(t.__file__), "..", "nvidia", "cuda_runtime", "lib", "libcudart.so*"))[0]
    rt = ctypes.CDLL(lib)
    buf = ctypes.create_string_buffer(nbytes)
    t.cuda.synchronize()
    assert rt.cudaMemcpy(buf, ctypes.c_void_p(ptr), ctypes.c_size_t(nbytes), 2) == 0
    return buf.raw
