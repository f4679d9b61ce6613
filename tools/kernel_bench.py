"""Microbenchmark of the hot kernels through the C ABI (stateless calls, small memory footprint,
suitable for ncu): expert SwiGLU GEMV pair (bf16 / int8 shadow), router, LM head, grouped GEMM.
Times with CUDA events on the launching stream, L2 flushed (256 MB write) before every launch.

    python tools/kernel_bench.py [--iters 20] [--only gemv]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2512_03927_b200 import odmoe  # noqa: E402

d, F, E, V = 4096, 14336, 8, 32000


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}


GAP_S = 0.0
DIRTY = False
GAP_MODE = "idle"   # idle: host sleep (GPU idle); spin: one-CTA spin kernel fills the gap; busy: HBM writes fill it


def timeit(fn, iters, flush):
    ts = []
    s = torch.cuda.current_stream()
    for i in range(iters + 3):
        if DIRTY:
            flush.add_(1)  # write 256 MB: L2 full of DIRTY lines (like just after an H2D load)
        else:
            flush.sum()  # read 256 MB (> 126 MB L2): evicts the weights with CLEAN lines
        if GAP_S > 0 and GAP_MODE == "idle":
            torch.cuda.synchronize()
            import time as _t
            _t.sleep(GAP_S)  # idle GPU before the launch (like the on-demand path waiting on PCIe)
        elif GAP_S > 0 and GAP_MODE == "spin":
            torch.cuda.synchronize()
            torch.cuda._sleep(int(GAP_S * 1.9e9))  # one CTA spins for the gap on this stream
        elif GAP_S > 0 and GAP_MODE == "busy":
            torch.cuda.synchronize()
            for _ in range(max(1, int(GAP_S / 40e-6))):
                flush.add_(1)  # the whole GPU streams HBM for the gap (256 MB writes, ~40 us each)
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b) * 1e-3)
    ts.sort()
    return ts[len(ts) // 2], ts[0]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--only", default="")
    ap.add_argument("--gap-ms", type=float, default=0.0)
    ap.add_argument("--dirty", action="store_true")
    ap.add_argument("--gap-mode", default="idle", choices=["idle", "spin", "busy"])
    args = ap.parse_args()
    global GAP_S, DIRTY, GAP_MODE
    GAP_S = args.gap_ms * 1e-3
    DIRTY = args.dirty
    GAP_MODE = args.gap_mode
    dev = torch.device("cuda", 0)
    flush = torch.zeros(64 << 20, dtype=torch.float32, device=dev)
    pk = peaks()
    out = {}
    bf = torch.bfloat16
    if args.only == "bf16":  # the main bf16 expert alone (ncu target; ODMOE_MAIN_MMA=0/1 A/B)
        blob = torch.empty(3 * F * d, dtype=bf, device=dev)
        odmoe.gen_weights(blob, 0, layer=0, expert=0, d=d, F=F, seed=2512)
        w13, w2 = blob[: 2 * F * d], blob[2 * F * d:].view(d, F)
        u = (torch.rand(d, device=dev) - 0.5).to(bf)
        a = torch.empty(F, device=dev)
        y = torch.empty(d, device=dev)
        gw = torch.ones(2, device=dev)
        med, best = timeit(lambda: odmoe.expert_ffn(w13, w2, u, a, y, gate_w=gw), args.iters, flush)
        nbytes = 3 * F * d * 2
        out["expert_ffn_bf16"] = dict(us_median=med * 1e6, us_best=best * 1e6, GBps=nbytes / med / 1e9,
                                      frac_hbm=nbytes / med / 1e9 / pk["hbm_gbs"], bytes=nbytes,
                                      engine="mma" if os.environ.get("ODMOE_MAIN_MMA", "0") == "1" else "ffma2")
        del blob
    if args.only in ("", "gemv", "shadow"):
        blob = torch.empty(3 * F * d, dtype=bf, device=dev)
        odmoe.gen_weights(blob, 0, layer=0, expert=0, d=d, F=F, seed=2512)
        w13, w2 = blob[: 2 * F * d], blob[2 * F * d:].view(d, F)
        u = (torch.rand(d, device=dev) - 0.5).to(bf)
        a = torch.empty(F, device=dev)
        y = torch.empty(d, device=dev)
        gw = torch.ones(2, device=dev)
        if args.only != "shadow":  # --only shadow: the low-bit shadow experts alone (ncu target)
            med, best = timeit(lambda: odmoe.expert_ffn(w13, w2, u, a, y, gate_w=gw), args.iters, flush)
            nbytes = 3 * F * d * 2
            out["expert_ffn_bf16"] = dict(us_median=med * 1e6, us_best=best * 1e6, GBps=nbytes / med / 1e9,
                                          frac_hbm=nbytes / med / 1e9 / pk["hbm_gbs"], bytes=nbytes)
        # int8 shadow expert
        q = torch.empty((3 * F * d,), dtype=torch.int8, device=dev)
        sc = torch.empty(2 * F + d, device=dev)
        odmoe.quantize_int8_rows(w13.view(2 * F, d), q[: 2 * F * d].view(2 * F, d), sc[: 2 * F])
        odmoe.quantize_int8_rows(w2, q[2 * F * d:].view(d, F), sc[2 * F:])
        med, best = timeit(lambda: odmoe.shadow_expert_ffn(q[: 2 * F * d], sc[: 2 * F], q[2 * F * d:].view(d, F),
                                                           sc[2 * F:], u, a, y, gate_w=gw), args.iters, flush)
        nb = 3 * F * d + (2 * F + d) * 4
        out["expert_ffn_int8"] = dict(us_median=med * 1e6, us_best=best * 1e6, GBps=nb / med / 1e9,
                                      frac_hbm=nb / med / 1e9 / pk["hbm_gbs"], bytes=nb)
        # the same expert on the tensor cores (fragment-packed codes; the engine's shadow path)
        p13 = torch.empty(2 * F * d, dtype=torch.uint8, device=dev)
        p2 = torch.empty(d * F, dtype=torch.uint8, device=dev)
        odmoe.pack_int8_frag(q[: 2 * F * d].view(2 * F, d), p13, True)
        odmoe.pack_int8_frag(q[2 * F * d:].view(d, F), p2, False)
        med, best = timeit(lambda: odmoe.shadow_expert_ffn_packed(p13, sc[: 2 * F], p2, sc[2 * F:], u, a, y, d, F,
                                                                  gate_w=gw), args.iters, flush)
        out["expert_ffn_int8_mma"] = dict(us_median=med * 1e6, us_best=best * 1e6, GBps=nb / med / 1e9,
                                          frac_hbm=nb / med / 1e9 / pk["hbm_gbs"], bytes=nb)
        del p13, p2
        # NF4 shadow expert (reading Q27): codes + block absmax
        q4 = torch.empty((3 * F * d // 2,), dtype=torch.uint8, device=dev)
        a4 = torch.empty(3 * F * d // 64, device=dev)
        odmoe.quantize_nf4(w13.view(2 * F, d), q4[: F * d].view(2 * F, d // 2), a4[: 2 * F * d // 64].view(2 * F, d // 64))
        odmoe.quantize_nf4(w2, q4[F * d:].view(d, F // 2), a4[2 * F * d // 64:].view(d, F // 64))
        med, best = timeit(lambda: odmoe.shadow_expert_ffn_nf4(q4[: F * d].view(2 * F, d // 2), a4[: 2 * F * d // 64],
                                                               q4[F * d:].view(d, F // 2), a4[2 * F * d // 64:],
                                                               u, a, y, gate_w=gw), args.iters, flush)
        nb = 3 * F * d // 2 + 3 * F * d // 64 * 4
        out["expert_ffn_nf4"] = dict(us_median=med * 1e6, us_best=best * 1e6, GBps=nb / med / 1e9,
                                     frac_hbm=nb / med / 1e9 / pk["hbm_gbs"], bytes=nb)
        # FP8 shadow expert (reading Q28)
        q8 = torch.empty((3 * F * d,), dtype=torch.uint8, device=dev)
        odmoe.quantize_fp8_rows(w13.view(2 * F, d), q8[: 2 * F * d].view(2 * F, d), sc[: 2 * F])
        odmoe.quantize_fp8_rows(w2, q8[2 * F * d:].view(d, F), sc[2 * F:])
        med, best = timeit(lambda: odmoe.shadow_expert_ffn_fp8(q8[: 2 * F * d], sc[: 2 * F], q8[2 * F * d:].view(d, F),
                                                               sc[2 * F:], u, a, y, gate_w=gw), args.iters, flush)
        nb = 3 * F * d + (2 * F + d) * 4
        out["expert_ffn_fp8"] = dict(us_median=med * 1e6, us_best=best * 1e6, GBps=nb / med / 1e9,
                                     frac_hbm=nb / med / 1e9 / pk["hbm_gbs"], bytes=nb)
        del blob, q, q4, q8
    if args.only in ("read",):
        # read-only ceiling: torch's reduction over the same byte counts (one and two experts)
        for nb in (3 * F * d * 2, 6 * F * d * 2, 1 << 30):
            t = torch.empty(nb // 2, dtype=bf, device=dev).normal_()
            med, best = timeit(lambda: t.sum(dtype=torch.float32), args.iters, flush)
            out[f"torch_sum_{nb >> 20}MiB"] = dict(us_median=med * 1e6, GBps=nb / med / 1e9,
                                                   frac_hbm=nb / med / 1e9 / pk["hbm_gbs"], bytes=nb)
            del t
    if args.only in ("", "lm"):
        W = torch.empty((V, d), dtype=bf, device=dev)
        odmoe.gen_weights(W, 6, rows=V, cols=d, fan_in=d, seed=2512)
        h = torch.randn(d, device=dev)
        tok = torch.empty(1, dtype=torch.int32, device=dev)
        scratch = torch.zeros(16 * 4096, dtype=torch.uint8, device=dev)
        med, best = timeit(lambda: odmoe.lm_head_argmax(h, W, tok, scratch), args.iters, flush)
        nb = V * d * 2
        out["lm_head_argmax"] = dict(us_median=med * 1e6, us_best=best * 1e6, GBps=nb / med / 1e9,
                                     frac_hbm=nb / med / 1e9 / pk["hbm_gbs"], bytes=nb)
        del W
    if args.only in ("", "router"):
        Wg = torch.empty((E, d), dtype=bf, device=dev)
        odmoe.gen_weights(Wg, 2, rows=E, cols=d, fan_in=d, seed=2512)
        h = torch.randn(1, d, device=dev)
        y0 = torch.randn(1, d, device=dev) * 0.1
        y1 = torch.randn(1, d, device=dev) * 0.1
        uo = torch.empty(1, d, dtype=bf, device=dev)
        ids = torch.empty(1, 2, dtype=torch.int32, device=dev)
        w = torch.empty(1, 2, device=dev)
        med, best = timeit(lambda: odmoe.route_topk(h, Wg, 2, uo, ids, w, y_add=[y0, y1]), args.iters, flush)
        out["router_topk"] = dict(us_median=med * 1e6, us_best=best * 1e6)
    if args.only in ("", "grouped"):
        import numpy as np
        rng = np.random.default_rng(3)
        ids = np.stack([rng.choice(E, size=2, replace=False) for _ in range(512)])
        counts = np.bincount(ids.reshape(-1), minlength=E)
        off = [0] + [int(v) for v in np.cumsum(counts)]
        M = int(off[-1])
        blobs = []
        for e in range(E):
            b = torch.empty(3 * F * d, dtype=bf, device=dev)
            odmoe.gen_weights(b, 0, layer=0, expert=e, d=d, F=F, seed=2512)
            blobs.append(b)
        w13s = [b[: 2 * F * d] for b in blobs]
        w2s = [b[2 * F * d:].view(d, F) for b in blobs]
        x = (torch.rand(M, d, device=dev) - 0.5).to(bf)
        gate = torch.rand(M, device=dev)
        a2 = torch.empty(M, F, dtype=bf, device=dev)
        y = torch.empty(M, d, device=dev)
        tiles = torch.empty(16 * ((M // 128 + E + 1) * (2 * F // 128 + d // 128)), dtype=torch.uint8, device=dev)
        med, best = timeit(lambda: odmoe.expert_ffn_grouped(w13s, w2s, x, off, gate, a2, y, tiles), max(5, args.iters // 4), flush)
        flops = 2.0 * M * 3 * d * F
        nb = E * 3 * F * d * 2
        out["grouped_ffn_T512"] = dict(ms_median=med * 1e3, TFLOPs=flops / med / 1e12, GBps=nb / med / 1e9,
                                       frac_tensor=flops / med / 1e12 / pk["bf16_tflops"],
                                       frac_hbm=nb / med / 1e9 / pk["hbm_gbs"], rows=M,
                                       note="includes the host tile-list build + a stream sync")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
