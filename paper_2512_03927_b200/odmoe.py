"""Thin ctypes binding of libodmoe.so (include/odmoe.h). Argument marshalling only: every step
of the hot path runs in the library's CUDA kernels / C++ runtime. PyTorch tensors are used
only as device-memory holders (``data_ptr()``) and for the current CUDA stream.

There is no fallback: if the library is missing the import raises.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ODMOE_LIB") or os.path.join(_HERE, "libodmoe.so")

BF16, FP32 = 0, 1
(PRED_SHADOW_INT8, PRED_NONE, PRED_RANDOM, PRED_PERFECT, PRED_SHADOW_SAME, PRED_GATE_REUSE, PRED_SHADOW_BF16,
 PRED_SHADOW_NF4, PRED_SHADOW_FP8) = range(9)
PLACE_GROUPS, PLACE_SLICED = 0, 1
PREDICTORS = {"shadow_int8": 0, "none": 1, "random": 2, "perfect": 3, "shadow_same": 4, "gate_reuse": 5,
              "shadow_bf16": 6, "shadow_nf4": 7, "shadow_fp8": 8}

STATUS = {0: "OK", 1: "E_CONFIG", 2: "E_RANGE", 3: "E_NONFINITE", 4: "E_BUDGET", 5: "E_STATE",
          6: "E_PLAN", 7: "E_NOMEM", 8: "E_CUDA", 9: "E_NCCL"}

# debug_read fields
DBG = dict(H_IN=0, U=1, LOGITS=2, IDS=3, W=4, Y=5, Y_PART=6, SH_H_IN=7, SH_U=8, SH_LOGITS=9,
           SH_IDS=10, H_FINAL=11, LM_LOGITS=12, H_PRE=13, SH_H_FINAL=14, SH_TOK=15, SH_LM_LOGITS=16, Y_RANK=17)


class OdmoeError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run `make -C paper_2512_03927_b200` "
                          "(or __graft_entry__.build()); there is no CPU fallback")
    return ctypes.CDLL(LIB_PATH)


_lib = _load()


class Config(ctypes.Structure):
    _fields_ = [("L", ctypes.c_int32), ("E", ctypes.c_int32), ("k", ctypes.c_int32), ("d", ctypes.c_int32),
                ("F", ctypes.c_int32), ("V", ctypes.c_int32), ("dtype", ctypes.c_int32),
                ("predictor", ctypes.c_int32), ("lookahead", ctypes.c_int32),
                ("slots_per_gpu", ctypes.c_int32), ("rms_eps", ctypes.c_float),
                ("weight_seed", ctypes.c_uint64), ("aux_seed", ctypes.c_uint64),
                ("rank", ctypes.c_int32), ("world_size", ctypes.c_int32), ("group_size", ctypes.c_int32),
                ("device", ctypes.c_int32), ("chunk_bytes", ctypes.c_int64),
                ("debug_capture", ctypes.c_int32), ("time_kernels", ctypes.c_int32),
                ("pool_threads", ctypes.c_int32), ("refine_depth", ctypes.c_int32),
                ("placement", ctypes.c_int32), ("n_heads", ctypes.c_int32), ("n_kv_heads", ctypes.c_int32),
                ("max_seq", ctypes.c_int32), ("emulate_world", ctypes.c_int32), ("expert_layer_period", ctypes.c_int32),
                ("nccl_id", ctypes.c_void_p)]


class LayerRecord(ctypes.Structure):
    _fields_ = [("true_ids", ctypes.c_int32 * 8), ("pred_ids", ctypes.c_int32 * 8),
                ("weights", ctypes.c_float * 8), ("pred_available", ctypes.c_int32),
                ("correct", ctypes.c_int32), ("n_reloads", ctypes.c_int32),
                ("load_wait_us", ctypes.c_float), ("pred_in_time", ctypes.c_int32),
                ("correct_in_time", ctypes.c_int32), ("issued_ids", ctypes.c_int32 * 8),
                ("reload_ids", ctypes.c_int32 * 8)]


class TraceEvent(ctypes.Structure):
    _fields_ = [("type", ctypes.c_int32), ("step", ctypes.c_int32), ("layer", ctypes.c_int32),
                ("expert", ctypes.c_int32), ("slot", ctypes.c_int32), ("l_cur", ctypes.c_int32),
                ("aux", ctypes.c_int32), ("rank", ctypes.c_int32), ("bytes", ctypes.c_int64),
                ("t_us", ctypes.c_double)]


EV_NAMES = ["StepStart", "LoadIssue", "LoadStart", "LoadEnd", "LoadCancel", "RouterDone", "ComputeStart",
            "ComputeEnd", "Mispredict", "StepEnd"]


class Stats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in (
        "tokens", "loads_issued", "loads_completed", "loads_cancelled", "reloads", "bytes_h2d",
        "kernel_launches", "max_resident", "resident_bytes", "shadow_bytes", "pool_bytes")] + [
        ("pool_build_s", ctypes.c_double)] + [
        (n, ctypes.c_double) for n in ("ms_router", "ms_w13", "ms_w2", "ms_shadow", "ms_lm_head", "ms_embed")] + [
        (n, ctypes.c_int64) for n in ("n_router", "n_w13", "n_w2", "n_shadow", "n_lm_head", "n_embed")] + [
        ("wait_us", ctypes.c_double), ("correct", ctypes.c_int64), ("predicted_total", ctypes.c_int64),
        ("refine_corrections", ctypes.c_int64), ("refine_correct", ctypes.c_int64), ("refine_total", ctypes.c_int64),
        ("ms_attn", ctypes.c_double), ("n_attn", ctypes.c_int64), ("correct_in_time", ctypes.c_int64),
        ("spec_steps", ctypes.c_int64), ("early_loads", ctypes.c_int64), ("ms_sh_w13", ctypes.c_double),
        ("ms_sh_w2", ctypes.c_double), ("n_sh_w13", ctypes.c_int64), ("n_sh_w2", ctypes.c_int64),
        ("ms_sh_pass", ctypes.c_double), ("n_sh_pass", ctypes.c_int64)]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


_P = ctypes.c_void_p
_I = ctypes.c_int
_F = ctypes.c_float
_I64 = ctypes.c_int64


def _sig(name, args, res=ctypes.c_int):
    f = getattr(_lib, name)
    f.argtypes = args
    f.restype = res
    return f


_abi_version = _sig("odmoe_abi_version", [], ctypes.c_int32)
_create = _sig("odmoe_create", [ctypes.POINTER(Config), ctypes.POINTER(ctypes.c_void_p)])
_destroy = _sig("odmoe_destroy", [_P], None)
_last_error = _sig("odmoe_last_error", [_P], ctypes.c_char_p)
_get_stats = _sig("odmoe_get_stats", [_P, ctypes.POINTER(Stats)])
_reset_stats = _sig("odmoe_reset_stats", [_P])
_nccl_uid = _sig("odmoe_nccl_unique_id", [_P])
_route = _sig("odmoe_route_topk", [_P, _P, _I, _P, _P, _I, _I, _I, _I, _I, _F, _P, _P, _P, _P, _P, _P])
_sh_route = _sig("odmoe_shadow_route_topk", [_P, _P, _I, _P, _P, _I, _I, _I, _I, _F, _P, _P, _P, _P, _P, _P])
_ffn = _sig("odmoe_expert_ffn", [_P, _P, _P, _P, _I, _I, _I, _I, _P, _P, _P])
_sh_ffn = _sig("odmoe_shadow_expert_ffn", [_P, _P, _P, _P, _P, _P, _I, _I, _I, _P, _P, _P])
_lm = _sig("odmoe_lm_head_argmax", [_P, _P, _I, _I, _I, _F, _P, _P, _P, _P])
_quant = _sig("odmoe_quantize_int8_rows", [_P, _I64, _I64, _I, _P, _P, _P])
_sh_ffn_packed = _sig("odmoe_shadow_expert_ffn_packed", [_P, _P, _P, _P, _P, _P, _I, _I, _I, _P, _P, _P])
_pack_frag = _sig("odmoe_pack_int8_frag", [_P, _I64, _I64, _I, _P, _P])
_sh_ffn_nf4 = _sig("odmoe_shadow_expert_ffn_nf4", [_P, _P, _P, _P, _P, _P, _I, _I, _I, _P, _P, _P])
_quant_nf4 = _sig("odmoe_quantize_nf4", [_P, _I64, _I64, _I, _P, _P, _P])
_sh_ffn_fp8 = _sig("odmoe_shadow_expert_ffn_fp8", [_P, _P, _P, _P, _P, _P, _I, _I, _I, _P, _P, _P])
_quant_fp8 = _sig("odmoe_quantize_fp8_rows", [_P, _I64, _I64, _I, _P, _P, _P])
_gen = _sig("odmoe_gen_weights", [_P, _I, _I, _I, _I64, _I64, _I64, _I, _I, ctypes.c_uint64, _I, _P])
_load_ = _sig("odmoe_load", [_P, _I, _I])
_load_wait = _sig("odmoe_load_wait", [_P, _I, _I, ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_void_p)])
_evict = _sig("odmoe_evict", [_P, _I, _I])
_predict = _sig("odmoe_predict_ahead", [_P, ctypes.c_int32, _I, _I, _P])
_decode = _sig("odmoe_decode_step", [_P, ctypes.c_int32, ctypes.POINTER(ctypes.c_int32), _P])
_prefill = _sig("odmoe_prefill", [_P, _P, _I, ctypes.POINTER(ctypes.c_int32), _P])
_dbg = _sig("odmoe_debug_read", [_P, _I, _I, _P, _I64])
_tensor_ptr = _sig("odmoe_tensor_ptr", [_P, _I, _I, ctypes.POINTER(ctypes.c_void_p)])

_ffn_grouped = _sig("odmoe_expert_ffn_grouped", [_P, _P, _I, _P, _P, _P, _I, _I, _P, _P, _P, _I64, _P])
_prefill_group = _sig("odmoe_prefill_group", [_P, _P, _I, _I, _I, _P, _P, _P, _P, _P])
_prefill_dbg = _sig("odmoe_prefill_debug_read", [_P, _I, _I, _P, _I64])
_set_option = _sig("odmoe_set_option", [_P, _I, _I64])
_trace_read = _sig("odmoe_trace_read", [_P, _P, ctypes.c_int32, ctypes.POINTER(ctypes.c_int32)])
_plan_layer = _sig("odmoe_plan_layer", [_I, _I, _I, _I, _P, _I, _P, ctypes.POINTER(ctypes.c_int32)])
_plan_pool = _sig("odmoe_plan_pool_holds", [_I, _I, _I, _I, _I, _I, _I], ctypes.c_int32)

EXPORTED = ["odmoe_set_option", "odmoe_expert_ffn_grouped", "odmoe_prefill_group", "odmoe_prefill_debug_read",
            "odmoe_plan_layer", "odmoe_plan_pool_holds", "odmoe_abi_version", "odmoe_create", "odmoe_destroy", "odmoe_last_error", "odmoe_get_stats",
            "odmoe_reset_stats", "odmoe_nccl_unique_id", "odmoe_route_topk", "odmoe_expert_ffn",
            "odmoe_shadow_expert_ffn", "odmoe_shadow_route_topk", "odmoe_lm_head_argmax",
            "odmoe_quantize_int8_rows", "odmoe_gen_weights", "odmoe_load", "odmoe_load_wait",
            "odmoe_evict", "odmoe_predict_ahead", "odmoe_decode_step", "odmoe_prefill",
            "odmoe_debug_read", "odmoe_tensor_ptr", "odmoe_shadow_expert_ffn_nf4", "odmoe_quantize_nf4",
            "odmoe_shadow_expert_ffn_fp8", "odmoe_quantize_fp8_rows", "odmoe_trace_read",
            "odmoe_shadow_expert_ffn_packed", "odmoe_pack_int8_frag"]


def abi_version() -> int:
    return int(_abi_version())


def _check(st: int, ctx=None):
    if st != 0:
        msg = _last_error(ctx).decode(errors="replace") if ctx is not None or st else ""
        raise OdmoeError(st, msg)


def _ptr(t) -> Optional[int]:
    return None if t is None else t.data_ptr()


def _stream(stream):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _ptr_array(tensors: Sequence, device):
    import torch
    return torch.tensor([t.data_ptr() for t in tensors], dtype=torch.int64, device=device)


# ------------------------------------------------------------------ stateless kernels
def route_topk(h, w_gate, k: int, u_out, ids, w, logits=None, y_add=(), gamma=None, eps=1e-5,
               dtype=BF16, flag=None, stream=None):
    """h [m,d] fp32 (updated in place by the residual add), w_gate [E,d] (bf16 or fp32)."""
    m, d = h.shape
    E = w_gate.shape[0]
    yp = _ptr_array(y_add, h.device) if len(y_add) else None
    _check(_route(_ptr(h), _ptr(yp), len(y_add), _ptr(gamma), _ptr(w_gate), m, E, d, k, dtype, eps,
                  _ptr(u_out), _ptr(ids), _ptr(w), _ptr(logits), _ptr(flag), _stream(stream)))
    return yp  # keep the pointer array alive until the stream passes


def shadow_route_topk(h, q_gate, s_gate, k: int, u_out, ids, w, logits=None, y_add=(), eps=1e-5,
                      flag=None, stream=None):
    m, d = h.shape
    E = q_gate.shape[0]
    yp = _ptr_array(y_add, h.device) if len(y_add) else None
    _check(_sh_route(_ptr(h), _ptr(yp), len(y_add), _ptr(q_gate), _ptr(s_gate), m, E, d, k, eps,
                     _ptr(u_out), _ptr(ids), _ptr(w), _ptr(logits), _ptr(flag), _stream(stream)))
    return yp


def expert_ffn(w13, w2, u, a_scratch, y, gate_w=None, gate_idx=0, dtype=BF16, stream=None):
    """w13 [F,2,d] (or [2F,d]), w2 [d,F], u [d]; y [d] fp32 = gate_w[gate_idx] * FFN(u)."""
    d = w2.shape[0]
    F = w2.shape[1]
    _check(_ffn(_ptr(w13), _ptr(w2), _ptr(u), _ptr(gate_w), gate_idx, d, F, dtype, _ptr(a_scratch),
                _ptr(y), _stream(stream)))


def shadow_expert_ffn(q13, s13, q2, s2, u, a_scratch, y, gate_w=None, gate_idx=0, stream=None):
    d, F = q2.shape
    _check(_sh_ffn(_ptr(q13), _ptr(s13), _ptr(q2), _ptr(s2), _ptr(u), _ptr(gate_w), gate_idx, d, F,
                   _ptr(a_scratch), _ptr(y), _stream(stream)))


def pack_int8_frag(q, out, pair_rows: bool, stream=None):
    """int8 codes q [R, C] -> the tensor-core fragment-packed layout (uint8 [R*C])."""
    R, C = q.shape
    _check(_pack_frag(_ptr(q), R, C, int(pair_rows), _ptr(out), _stream(stream)))


def shadow_expert_ffn_packed(q13p, s13, q2p, s2, u, a_scratch, y, d, F, gate_w=None, gate_idx=0, stream=None):
    """INT8 shadow expert on the tensor cores: q13p / q2p from pack_int8_frag (W13 pair_rows=True)."""
    _check(_sh_ffn_packed(_ptr(q13p), _ptr(s13), _ptr(q2p), _ptr(s2), _ptr(u), _ptr(gate_w), gate_idx, d, F,
                          _ptr(a_scratch), _ptr(y), _stream(stream)))


def shadow_expert_ffn_nf4(q13, a13, q2, a2, u, a_scratch, y, gate_w=None, gate_idx=0, stream=None):
    """NF4 shadow expert: q13 uint8 [2F, d/2], a13 fp32 [2F, d/64], q2 uint8 [d, F/2], a2 fp32 [d, F/64]."""
    d = q2.shape[0]
    F = 2 * q2.shape[1]
    _check(_sh_ffn_nf4(_ptr(q13), _ptr(a13), _ptr(q2), _ptr(a2), _ptr(u), _ptr(gate_w), gate_idx, d, F,
                       _ptr(a_scratch), _ptr(y), _stream(stream)))


def shadow_expert_ffn_fp8(q13, s13, q2, s2, u, a_scratch, y, gate_w=None, gate_idx=0, stream=None):
    """FP8 shadow expert: q13 uint8 E4M3 [2F, d], s13 [2F], q2 [d, F], s2 [d]."""
    d, F = q2.shape
    _check(_sh_ffn_fp8(_ptr(q13), _ptr(s13), _ptr(q2), _ptr(s2), _ptr(u), _ptr(gate_w), gate_idx, d, F,
                       _ptr(a_scratch), _ptr(y), _stream(stream)))


def prefill_group(ids, w, E: int, offsets, src_pair, inv, gate_perm, stream=None):
    """ids [T,k] int32, w [T,k] fp32 -> offsets [E+1], src_pair/inv [T*k] int32, gate_perm [T*k]."""
    T, k = ids.shape
    _check(_prefill_group(_ptr(ids), _ptr(w), T, k, E, _ptr(offsets), _ptr(src_pair), _ptr(inv),
                          _ptr(gate_perm), _stream(stream)))


def expert_ffn_grouped(w13s, w2s, x_perm, offsets: Sequence[int], gate_perm, a2_scratch, y_perm, tiles_scratch,
                       stream=None):
    """Grouped SwiGLU FFN on tcgen05: w13s/w2s lists of bf16 device tensors (one per expert),
    offsets host list [E+1]. Synchronous on the stream."""
    n = len(w13s)
    d = w2s[0].shape[0]
    F = w2s[0].shape[1]
    a13 = (ctypes.c_void_p * n)(*[t.data_ptr() for t in w13s])
    a2 = (ctypes.c_void_p * n)(*[t.data_ptr() for t in w2s])
    off = (ctypes.c_int32 * (n + 1))(*offsets)
    _check(_ffn_grouped(a13, a2, n, _ptr(x_perm), off, _ptr(gate_perm), d, F, _ptr(a2_scratch), _ptr(y_perm),
                        _ptr(tiles_scratch), tiles_scratch.numel() * tiles_scratch.element_size(), _stream(stream)))


def lm_head_argmax(h, lm_head, token_out, scratch, logits=None, eps=1e-5, dtype=BF16, stream=None):
    V, d = lm_head.shape
    _check(_lm(_ptr(h), _ptr(lm_head), V, d, dtype, eps, _ptr(token_out), _ptr(logits), _ptr(scratch),
               _stream(stream)))


def quantize_int8_rows(w, q, s, dtype=BF16, stream=None):
    R, C = w.shape
    _check(_quant(_ptr(w), R, C, dtype, _ptr(q), _ptr(s), _stream(stream)))


def quantize_nf4(w, q, absmax, dtype=BF16, stream=None):
    """w [R, C] -> q uint8 [R, C/2] (two codes per byte, low nibble = even column), absmax [R, C/64]."""
    R, C = w.shape
    _check(_quant_nf4(_ptr(w), R, C, dtype, _ptr(q), _ptr(absmax), _stream(stream)))


def quantize_fp8_rows(w, q, s, dtype=BF16, stream=None):
    """w [R, C] -> q uint8 E4M3 codes [R, C], s [R]."""
    R, C = w.shape
    _check(_quant_fp8(_ptr(w), R, C, dtype, _ptr(q), _ptr(s), _stream(stream)))


def gen_weights(out, kind, layer=0, expert=0, rows=0, cols=0, fan_in=1, d=0, F=0, seed=2512, dtype=BF16,
                stream=None):
    _check(_gen(_ptr(out), kind, layer, expert, rows, cols, fan_in, d, F, seed, dtype, _stream(stream)))


def plan_layer(k: int, world_size: int, layer: int, ids: Sequence[int], rank: int, group_size: int = 0):
    """Experts of `layer` computed by `rank` (host-only placement plan)."""
    arr = (ctypes.c_int32 * k)(*ids)
    out = (ctypes.c_int32 * k)()
    n = ctypes.c_int32(0)
    _check(_plan_layer(k, world_size, group_size, layer, arr, rank, out, ctypes.byref(n)))
    return list(out[: n.value])


def plan_pool_holds(E: int, k: int, world_size: int, layer: int, expert: int, rank: int, group_size: int = 0) -> bool:
    r = _plan_pool(E, k, world_size, group_size, layer, expert, rank)
    if r < 0:
        raise OdmoeError(1, "invalid plan sizes")
    return bool(r)


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    if _nccl_uid(buf) != 0:
        raise OdmoeError(9, "ncclGetUniqueId failed")
    return buf.raw


# ------------------------------------------------------------------ stateful engine
class Engine:
    """One decode engine per process/GPU (odmoe_create ... odmoe_destroy)."""

    def __init__(self, L, E, k, d, F, V, dtype=BF16, predictor=PRED_SHADOW_INT8, lookahead=1,
                 slots_per_gpu=2, rms_eps=1e-5, weight_seed=2512, aux_seed=1, rank=0, world_size=1,
                 group_size=0, device=0, chunk_bytes=0, debug_capture=0, time_kernels=0,
                 nccl_id: Optional[bytes] = None, refine_depth=0, placement=0, n_heads=0, n_kv_heads=0,
                 max_seq=0, emulate_world=0, expert_layer_period=0):
        self.cfg = Config(L=L, E=E, k=k, d=d, F=F, V=V, dtype=dtype, predictor=predictor,
                          lookahead=lookahead, slots_per_gpu=slots_per_gpu, rms_eps=rms_eps,
                          weight_seed=weight_seed, aux_seed=aux_seed, rank=rank, world_size=world_size,
                          group_size=group_size, device=device, chunk_bytes=chunk_bytes,
                          debug_capture=debug_capture, time_kernels=time_kernels, pool_threads=0,
                          refine_depth=refine_depth, placement=placement, n_heads=n_heads,
                          n_kv_heads=n_kv_heads, max_seq=max_seq, emulate_world=emulate_world,
                          expert_layer_period=expert_layer_period)
        self._uid = ctypes.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        self.cfg.nccl_id = ctypes.cast(self._uid, ctypes.c_void_p) if self._uid is not None else None
        self.L, self.E, self.k, self.d, self.F, self.V = L, E, k, d, F, V
        self.rank = rank
        h = ctypes.c_void_p()
        st = _create(ctypes.byref(self.cfg), ctypes.byref(h))
        if st != 0:
            raise OdmoeError(st, _last_error(None).decode(errors="replace"))
        self.ctx = h

    def close(self):
        if getattr(self, "ctx", None):
            _destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _ck(self, st):
        if st != 0:
            raise OdmoeError(st, _last_error(self.ctx).decode(errors="replace"))

    def decode_step(self, token: int, records: bool = True):
        out = ctypes.c_int32(-1)
        recs = (LayerRecord * self.L)() if records else None
        self._ck(_decode(self.ctx, int(token), ctypes.byref(out), recs))
        return out.value, recs

    def predict_ahead(self, token: int, from_layer: int = 0, depth: Optional[int] = None):
        depth = self.L - from_layer if depth is None else depth
        buf = (ctypes.c_int32 * (depth * self.k))()
        self._ck(_predict(self.ctx, int(token), from_layer, depth, buf))
        return [list(buf[i * self.k:(i + 1) * self.k]) for i in range(depth)]

    def set_lookahead(self, D: int):
        self._ck(_set_option(self.ctx, 1, int(D)))

    def set_predictor(self, p: int):
        self._ck(_set_option(self.ctx, 2, int(p)))

    def set_refine_depth(self, R: int):
        self._ck(_set_option(self.ctx, 3, int(R)))

    def set_kv_align(self, on: bool):
        """Attention + shadow ctx: 1 = the shadow reads the main model's KV cache (KV1), 0 = its own (KV0)."""
        self._ck(_set_option(self.ctx, 5, int(bool(on))))

    def set_time_kernels(self, level: int):
        """0 = no CUDA events, 1 = around the expert launches, 2 = around every kernel family."""
        self._ck(_set_option(self.ctx, 6, int(level)))

    def set_trace(self, on: bool):
        """Event trace on/off (LoadIssue/Start/End/Cancel, RouterDone, ComputeStart/End, Mispredict)."""
        self._ck(_set_option(self.ctx, 7, int(bool(on))))

    def set_align_period(self, period: int):
        """Token alignment period T_p of the shadow (1 = Mode A; > 1 = cross-token speculation)."""
        self._ck(_set_option(self.ctx, 8, int(period)))

    def trace(self, cap: int = 1 << 16):
        """Resolved trace events since the last call, as dicts (t_us = device µs, NaN = host-only)."""
        out = []
        buf = (TraceEvent * cap)()
        while True:
            n = ctypes.c_int32(0)
            self._ck(_trace_read(self.ctx, buf, cap, ctypes.byref(n)))
            for i in range(n.value):
                e = buf[i]
                out.append(dict(type=EV_NAMES[e.type], step=e.step, layer=e.layer, expert=e.expert, slot=e.slot,
                                l_cur=e.l_cur, aux=e.aux, rank=e.rank, bytes=e.bytes, t_us=e.t_us))
            if n.value < cap:
                return out

    def set_pass_timing(self, on: bool):
        """CUDA events around every whole shadow pass (stats ms_sh_pass / n_sh_pass)."""
        self._ck(_set_option(self.ctx, 9, int(bool(on))))

    def set_position(self, pos: int):
        """Attention ctx: KV-cache position of the next decode step (0 = new sequence)."""
        self._ck(_set_option(self.ctx, 4, int(pos)))

    def load(self, layer, expert):
        self._ck(_load_(self.ctx, layer, expert))

    def load_wait(self, layer, expert):
        a, b = ctypes.c_void_p(), ctypes.c_void_p()
        self._ck(_load_wait(self.ctx, layer, expert, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    def evict(self, layer, expert):
        self._ck(_evict(self.ctx, layer, expert))

    def prefill(self, tokens):
        arr = (ctypes.c_int32 * len(tokens))(*tokens)
        out = ctypes.c_int32(-1)
        counts = (ctypes.c_int32 * (self.L * self.E))()
        self._ck(_prefill(self.ctx, arr, len(tokens), ctypes.byref(out), counts))
        return out.value, list(counts)

    def prefill_debug_read(self, what: int, layer: int, nbytes: int) -> bytes:
        buf = ctypes.create_string_buffer(nbytes)
        self._ck(_prefill_dbg(self.ctx, what, layer, buf, nbytes))
        return buf.raw

    def debug_read(self, what: str, layer: int, nbytes: int) -> bytes:
        buf = ctypes.create_string_buffer(nbytes)
        self._ck(_dbg(self.ctx, DBG[what], layer, buf, nbytes))
        return buf.raw

    def tensor_ptr(self, what: int, index: int = 0) -> int:
        p = ctypes.c_void_p()
        self._ck(_tensor_ptr(self.ctx, what, index, ctypes.byref(p)))
        return p.value

    def stats(self) -> dict:
        s = Stats()
        self._ck(_get_stats(self.ctx, ctypes.byref(s)))
        return s.as_dict()

    def reset_stats(self):
        self._ck(_reset_stats(self.ctx))
