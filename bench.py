"""OD-MoE decode benchmark (BASELINE.json metric: decode tokens/s vs fully-resident, and
expert-prediction accuracy).

One step = one batch-1 decode iteration of the whole hot path:
embed -> 32 x [router/top-k -> prediction check -> just-in-time H2D expert loads -> SwiGLU
expert GEMVs -> combine] -> LM head -> argmax, with the INT8 shadow predictor running ahead.
Workload at N=1: BASELINE.json configs[1] (Mixtral-8x7B shape, bf16, 1 GPU, on-demand, 2 slots
= 705 MB of experts per GPU). At N>1 (torchrun): configs[3]/[2] layout, experts spread
round-robin over groups of 2 GPUs, lookahead D = N/2.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode tokens/s vs fully-resident (1/2/4/8 B200); expert-prediction accuracy"
UNIT = "tok/s"
SHAPE = dict(L=32, E=8, k=2, d=4096, F=14336, V=32000)
EXPERT_BYTES = 3 * SHAPE["d"] * SHAPE["F"] * 2          # 352,321,536 (bf16)
W13_BYTES = 2 * SHAPE["d"] * SHAPE["F"] * 2
W2_BYTES = SHAPE["d"] * SHAPE["F"] * 2
SEED = 2512


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=16)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--predictor", default="shadow_int8")
    ap.add_argument("--slots", type=int, default=0,
                    help="device expert slots per GPU; 0 => 2 (groups: whole experts) or 2k (sliced: 1/N slices)")
    ap.add_argument("--placement", default="sliced", choices=["groups", "sliced"],
                    help="N > 1: sliced loading (SURVEY §8(f)3; default: every link serves every layer, "
                         "measured 97.6 vs 93.6 %% of the link roofline at 4 GPUs) or the paper's worker "
                         "groups (P:104)")
    ap.add_argument("--refine", type=int, default=2,
                    help="SEP refinement depth R (DESIGN.md §7); 0 = the paper's token-aligned shadow only")
    ap.add_argument("--lookahead", type=int, default=0, help="0 => max(1, N/2) (groups) or 1 (sliced)")
    ap.add_argument("--no-resident", action="store_true", help="skip the fully-resident baseline")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--first-token", type=int, default=-1)
    ap.add_argument("--prefill", type=int, default=512,
                    help="prompt tokens prefilled (configs[4]: TTFT + grouped GEMM) before the decode warm-up; 0 = skip")
    ap.add_argument("--attention", action="store_true",
                    help="with Mixtral's attention block (32 q / 8 kv heads, RoPE; SURVEY §8(f)4, reading Q29)")
    ap.add_argument("--context", type=int, default=512,
                    help="--attention: decode starts at this KV-cache position (rows before it zero: synthetic context)")
    ap.add_argument("--align-period", type=int, default=1,
                    help="token alignment period T_p of the shadow (1 = every token, the paper's optimum "
                         "P:277; > 1 = cross-token speculation, SURVEY §8(f)2)")
    ap.add_argument("--group-size", type=int, default=0, help="groups placement: G (0 => min(k, N))")
    ap.add_argument("--no-r0", action="store_true", help="skip the paper-only SEP (refine 0) leg")
    ap.add_argument("--trace-steps", type=int, default=2, help="steps traced for the Eq. 1 analysis (0 = skip)")
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "fp32"],
                    help="main-model precision; fp32 = the paper's (P:173): 704.6 MB experts, 1 slot under the "
                         "1 GB budget (SURVEY §8(d) C4), no refinement / prefill (bf16 paths)")
    ap.add_argument("--layer-period", type=int, default=-1,
                    help="expert_layer_period P (odmoe.h): expert weights repeat every P layers so the host pool "
                         "holds P layers; loads and bytes per token unchanged. -1 => 16 for fp32 (the 180 GB "
                         "fp32 pool exceeds the box's host RAM), 0 otherwise")
    ap.add_argument("--chunk-mb", type=int, default=0, help="H2D copy chunk of the loader in MiB (0 = the engine's default)")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    if a.layer_period < 0:
        a.layer_period = 16 if a.dtype == "fp32" else 0
    if a.dtype == "fp32":
        global EXPERT_BYTES, W13_BYTES, W2_BYTES
        EXPERT_BYTES, W13_BYTES, W2_BYTES = 2 * EXPERT_BYTES, 2 * W13_BYTES, 2 * W2_BYTES
        a.refine, a.prefill = 0, 0
        if a.slots == 0:
            a.slots = 1
    return a


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                smax = float(p[2])
            except ValueError:
                continue
            for nm, v in zip(names, p[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def h2d_peak_gbs(torch, dev, barrier=None):
    """Host-link roofline measured in the same run: one expert blob (352 MB) copied from
    cudaHostAlloc'd pinned memory with cudaMemcpyAsync, whole and in the loader's 32 MiB chunks,
    best of 3 each (all ranks at once when N > 1, so it is the concurrent per-GPU figure)."""
    import ctypes
    import glob
    lib = glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib",
                                 "libcudart.so*"))[0]
    rt = ctypes.CDLL(lib)
    hp = ctypes.c_void_p()
    assert rt.cudaHostAlloc(ctypes.byref(hp), ctypes.c_size_t(EXPERT_BYTES), ctypes.c_uint(1)) == 0
    ctypes.memset(hp, 1, EXPERT_BYTES)
    dst = torch.empty(EXPERT_BYTES, dtype=torch.uint8, device=dev)
    st = torch.cuda.Stream(device=dev)
    best = 0.0
    for chunk in (EXPERT_BYTES, 32 << 20):
        for _ in range(3):
            if barrier is not None:
                barrier()
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(st)
            off = 0
            while off < EXPERT_BYTES:
                n = min(chunk, EXPERT_BYTES - off)
                rt.cudaMemcpyAsync(ctypes.c_void_p(dst.data_ptr() + off), ctypes.c_void_p(hp.value + off),
                                   ctypes.c_size_t(n), 1, ctypes.c_void_p(st.cuda_stream))
                off += n
            b.record(st)
            torch.cuda.synchronize()
            best = max(best, EXPERT_BYTES / (a.elapsed_time(b) * 1e-3) / 1e9)
    rt.cudaFreeHost(hp)
    del dst
    return best


# ---------------------------------------------------------------------------- CPU oracle leg
def _blas_threads():
    try:
        from threadpoolctl import threadpool_info
        return max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        return os.cpu_count()


class OracleWalk:
    """Walks the CPU oracle (as it stands) through the layers of one Mixtral-shape decode token.
    Only the oracle call (O.moe_layer) is timed; the synthetic weights it reads are generated
    beforehand (in the real system they already sit in host DRAM), and only the routed experts
    of each layer are generated."""

    def __init__(self, seed=SEED, first_token=1):
        import numpy as np
        import oracle as O
        from inputs import MIXTRAL, KIND_ROUTER, tensor_id
        from inputs.fixture import _stored
        self.np, self.O, self.shape = np, O, MIXTRAL
        self.seed = seed
        self._stored, self._tid, self._kr = _stored, tensor_id, KIND_ROUTER
        d = MIXTRAL.d
        self.emb_row = _stored(seed, tensor_id(1), MIXTRAL.V, d, d, "bf16")[first_token]
        self.h = np.asarray(self.emb_row, dtype=np.float64)
        self.layer = 0

    def step(self):
        """One layer (router + top-k + 2 SwiGLU experts + combine); returns timed seconds."""
        from inputs import gen_expert
        S_, O, np = self.shape, self.O, self.np
        l = self.layer % S_.L
        Wg = self._stored(self.seed, self._tid(self._kr, l), S_.E, S_.d, S_.d, "bf16")
        sel = O.top_k(O.router_logits(Wg, O.rms_norm(self.h)), S_.k)   # which experts to generate
        experts = {e: gen_expert(S_, self.seed, l, e, "bf16") for e in sel}
        t0 = time.perf_counter()
        out = O.moe_layer(self.h, Wg, experts, S_.k)
        dt = time.perf_counter() - t0
        self.h = out["h_next"] if self.layer + 1 < S_.L else self.np.asarray(self.emb_row, dtype=np.float64)
        self.layer += 1
        return dt

    def lm_head_seconds(self):
        S_, O = self.shape, self.O
        W = self._stored(self.seed, self._tid(6), S_.V, S_.d, S_.d, "bf16")
        t0 = time.perf_counter()
        O.greedy_argmax(O.final_logits(W, self.h))
        return time.perf_counter() - t0


def oracle_sample(n_layers=24):
    """cpu_baseline: the oracle on `n_layers` consecutive layers of one decode token plus the LM
    head, scaled to a 32-layer token."""
    walk = OracleWalk()
    t_layers = sum(walk.step() for _ in range(n_layers))
    t_lm = walk.lm_head_seconds()
    s_tok = t_layers / n_layers * walk.shape.L + t_lm
    return {"value": 1.0 / s_tok, "unit": UNIT, "cores": _blas_threads(), "kind": "oracle",
            "sample": f"layers 0-{n_layers - 1} of one Mixtral-shape decode token (router, top-k, 2 SwiGLU "
                      f"experts, combine; fp64 numpy on the bf16 weights) + LM head/argmax, scaled to 32 "
                      f"layers; {t_layers + t_lm:.1f} s of timed CPU work"}


def run_reference(args):
    """--impl reference: the CPU oracle as the reference arm, on our arm's metric/config. Each step
    is a bounded sample: ONE of the 32 MoE layers of a decode token (the steps walk the token's
    layers), so ms_per_step is the measured time of that sample and the timed region is
    steps x ms_per_step; the metric (tok/s) = 1 / (mean layer time x 32 + LM head)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        # torchrun pins OMP_NUM_THREADS=1 per rank; rank 0 runs alone here, so give the oracle the
        # host cores it has at N = 1
        try:
            import numpy  # noqa: F401  (threadpoolctl only sees BLAS libraries already loaded)
            from threadpoolctl import threadpool_limits
            threadpool_limits(limits=len(os.sched_getaffinity(0)))
        except Exception:
            pass
    walk = OracleWalk()
    for _ in range(args.warmup):
        walk.step()
    times = [walk.step() for _ in range(args.steps)]
    t_lm = walk.lm_head_seconds()
    s_tok = statistics.mean(times) * walk.shape.L + t_lm
    v = 1.0 / s_tok
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": statistics.mean(times) * 1e3,
            "step": "one of the 32 MoE layers of a decode token (1/32 of a token; the LM head timed once)",
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": workload_config(args, 1),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": _blas_threads(), "kind": "oracle",
                             "sample": "each step = one of the 32 Mixtral-shape MoE layers of a decode token "
                                       "(router, top-k, 2 SwiGLU experts; fp64), scaled x32 + LM head"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def attn_kw(args):
    ctx = max(args.context, args.prefill)
    return dict(n_heads=32, n_kv_heads=8, max_seq=ctx + args.warmup + args.steps + 8) if args.attention else {}


def sliced(args, n):
    return args.placement == "sliced" and n > 1


def n_slots(args, n):
    return args.slots or (2 * SHAPE["k"] if sliced(args, n) else 2)


def model_kw(args, odmoe):
    """Main-model precision and the expert-layer period (fp32 leg)."""
    return dict(dtype=odmoe.FP32 if args.dtype == "fp32" else odmoe.BF16, expert_layer_period=args.layer_period)


def lookahead(args, n):
    return args.lookahead or (1 if sliced(args, n) else max(1, n // 2))


def workload_config(args, n):
    ng = max(1, n // 2)
    if n == 1:
        wl = ("configs[1]: Mixtral-8x7B shape (L=32, E=8, top-2, d=4096, F=14336, V=32000), "
              "bf16, batch-1 decode, on-demand expert loading")
        if args.dtype == "fp32":
            wl = ("configs[3] at the paper's precision (P:173): Mixtral-8x7B shape, FP32, batch-1 decode, "
                  f"on-demand, {n_slots(args, n)} slot(s) of 704.6 MB under the 1 GB budget")
    elif sliced(args, n):
        wl = (f"configs[2]/[3]: Mixtral-8x7B shape, bf16, batch-1 decode, sliced loading: each of {n} GPUs "
              f"loads and computes 1/{n} of every routed expert, partials reduced on GPU 0, lookahead {lookahead(args, n)}")
    else:
        wl = (f"configs[2]/[3]: Mixtral-8x7B shape, bf16, batch-1 decode, experts round-robin "
              f"over {ng} groups of 2 GPUs, lookahead {lookahead(args, n)}")
    per_slot = EXPERT_BYTES // n if sliced(args, n) else EXPERT_BYTES
    return {"workload": wl, "placement": args.placement if n > 1 else "single",
            "predictor": args.predictor, "slots_per_gpu": n_slots(args, n), "refine_depth": args.refine,
            "expert_bytes_per_gpu": n_slots(args, n) * per_slot,
            "lookahead": lookahead(args, n), "weight_seed": SEED,
            "attention": (("Mixtral GQA 32q/8kv, head_dim 128, RoPE 1e6, bf16 KV cache; " +
                           (f"decode after the {args.prefill}-token prefill" if args.prefill > 0 else
                            f"decode from position {args.context} (earlier cache rows zero: synthetic context)"))
                          if args.attention else "none on the hot path (reading Q22)"),
            "l2": f"inputs larger than L2: every step streams 64 distinct {EXPERT_BYTES / 1e6:.1f} MB experts",
            "expert_layer_period": args.layer_period or None}


# ---------------------------------------------------------------------------- our arm
_T0 = time.time()


def log(rank, msg):
    """Phase log on stderr (locates a stall in a multi-rank run; never on stdout)."""
    print(f"[bench r{rank} +{time.time() - _T0:7.1f}s] {msg}", file=sys.stderr, flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    # stdout carries the JSON line alone: native banners written to fd 1 (NCCL's version line under
    # torchrun) go to stderr; the line itself is written to the saved descriptor.
    sys.stdout.flush()
    json_out = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    import faulthandler
    faulthandler.dump_traceback_later(480, repeat=True, file=sys.stderr)  # stack dump if a phase stalls
    import torch
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    n = world
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2512_03927_b200 import odmoe
    peaks, peak_src = measured_peaks()

    uid = None
    if world > 1:
        obj = [odmoe.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    D = lookahead(args, n)
    pred = odmoe.PREDICTORS[args.predictor]
    log(rank, "create engine")
    t_create = time.time()
    refine = args.refine if args.predictor.startswith("shadow") else 0
    eng = odmoe.Engine(device=local, rank=rank, world_size=world, nccl_id=uid, predictor=pred,
                       slots_per_gpu=n_slots(args, n), lookahead=D, time_kernels=2, weight_seed=SEED,
                       refine_depth=refine, placement=int(sliced(args, n)), group_size=args.group_size,
                       chunk_bytes=args.chunk_mb << 20, **SHAPE, **attn_kw(args), **model_kw(args, odmoe))
    if args.align_period > 1:
        eng.set_align_period(args.align_period)
    if args.attention and args.prefill <= 0:
        eng.set_position(args.context)  # no prompt: decode over a zero-filled synthetic context
    t_create = time.time() - t_create
    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    link = h2d_peak_gbs(torch, torch.device("cuda", local), barrier if dist is not None else None)

    tok = args.first_token if args.first_token >= 0 else 1
    prefill = None
    if args.prefill > 0:
        log(rank, f"prefill {args.prefill}")
        from inputs import MIXTRAL, gen_prompt
        prompt = [int(x) for x in gen_prompt(MIXTRAL, 1, args.prefill)]
        eng.prefill(prompt[:8])  # allocate the prefill buffers / slots outside the timed call
        eng.reset_stats()
        barrier()
        t0 = time.perf_counter()
        tok, counts = eng.prefill(prompt)
        ttft = time.perf_counter() - t0
        pst = eng.stats()
        gg_ms = (pst["ms_w13"] + pst["ms_w2"])
        flops = 2.0 * args.prefill * SHAPE["k"] * 3 * SHAPE["d"] * SHAPE["F"] * SHAPE["L"]
        prefill = {"tokens": args.prefill, "ttft_ms_rank": ttft * 1e3, "h2d_bytes": pst["bytes_h2d"],
                   "grouped_gemm_ms_total": gg_ms, "grouped_gemm_TFLOPs": flops / max(gg_ms, 1e-9) / 1e9 / n,
                   "experts_activated_per_layer": sum(1 for c in counts if c > 0) / SHAPE["L"],
                   "note": "host wall clock of odmoe_prefill (synchronous); GEMM time from CUDA events"}
    log(rank, "warmup")
    for _ in range(args.warmup):
        tok, _ = eng.decode_step(tok, records=False)
    eng.reset_stats()
    log(rank, "timed decode")
    recs_all = []
    clocks = ClockSampler(local)
    barrier()
    clocks.start()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    ev0.record()
    for _ in range(args.steps):
        tok, recs = eng.decode_step(tok, records=(rank == 0))
        if rank == 0:
            recs_all.append([(tuple(r.true_ids[:2]), tuple(r.pred_ids[:2]), r.correct) for r in recs])
    ev1.record()
    barrier()
    wall = time.perf_counter() - t0
    clk = clocks.stop()
    dev_s = ev0.elapsed_time(ev1) * 1e-3
    st = eng.stats()
    # paper-only SEP (refinement off: the token-aligned shadow alone) beside the default
    r0 = None
    if refine > 0 and not args.no_r0:
        log(rank, "SEP refine 0 leg")
        r0 = leg(eng, torch, barrier, dist, tok, min(args.steps, 8), refine=0, restore=refine)
        tok = r0.pop("tok")
    # Eq. 1 from a per-layer event trace of a few more steps
    trace_ev = None
    if args.trace_steps > 0:
        log(rank, "traced steps")
        eng.set_trace(True)
        for _ in range(args.trace_steps):
            tok, _ = eng.decode_step(tok, records=False)
        time.sleep(0.05)
        trace_ev = eng.trace()
        eng.set_trace(False)
    # the shadow's whole token-aligned pass alone (SEP Mode A, a4): one event pair per pass on the
    # shadow stream, 8 passes for distinct tokens (N = 1: at N > 1 a pass broadcasts its predictions)
    sh_pass = None
    if n == 1 and args.predictor.startswith("shadow") and args.attention is False:
        eng.set_time_kernels(0)
        eng.set_pass_timing(True)
        eng.predict_ahead(7)
        eng.reset_stats()
        for t in range(8):
            eng.predict_ahead(1000 + t)
        pst = eng.stats()
        eng.set_pass_timing(False)
        if pst["n_sh_pass"]:
            k_, d_, F_ = SHAPE["k"], SHAPE["d"], SHAPE["F"]
            sh_bytes = SHAPE["L"] * k_ * (3 * F_ * d_ + (2 * F_ + d_) * 4)
            us = pst["ms_sh_pass"] / pst["n_sh_pass"] * 1e3
            sh_pass = {"bound": "hbm", "kernel": "whole INT8 shadow pass (32 x [router, k expert W13+SwiGLU, W2+gate])",
                       "algorithmic_bytes": sh_bytes, "us": us, "GBps": sh_bytes / us / 1e3,
                       "peak": peaks["hbm_gbs"], "frac": sh_bytes / us / 1e3 / peaks["hbm_gbs"], "passes": pst["n_sh_pass"],
                       "note": "odmoe_predict_ahead for 8 distinct tokens, alone on the GPU; CUDA events around each "
                               "pass on the shadow stream; bytes = the k experts' int8 codes + row scales of 32 layers"}
    if dist is not None:
        # every rank's expert-kernel time (rank 0 shares its GPU with the shadow stream)
        g_rank = (st["ms_w13"] + st["ms_w2"]) / max(1, st["n_w13"]) * 1e3
        gl = [torch.zeros(1, dtype=torch.float64, device="cuda") for _ in range(world)]
        dist.all_gather(gl, torch.tensor([g_rank], dtype=torch.float64, device="cuda"))
        us_per_rank = [float(x[0]) for x in gl]
        tt = torch.tensor([dev_s, wall], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dev_s, wall = float(tt[0]), float(tt[1])
        agg = torch.tensor([st["bytes_h2d"], link], dtype=torch.float64, device="cuda")
        dist.all_reduce(agg, op=dist.ReduceOp.SUM)
        bytes_all, link_all = float(agg[0]), float(agg[1])
    else:
        bytes_all, link_all = float(st["bytes_h2d"]), link
        us_per_rank = None
    eng.close()
    del eng

    value = args.steps / dev_s
    e2e = args.steps / wall
    res = None
    if not args.no_resident:
        log(rank, "resident baseline")
        res = resident_baseline(odmoe, torch, args, local, rank, world, dist)

    if rank == 0:
        n_exp = max(1, st["n_w13"])
        gemv_ms = (st["ms_w13"] + st["ms_w2"]) / n_exp
        blob = EXPERT_BYTES // n if sliced(args, n) else EXPERT_BYTES   # bytes one launch pair streams
        achieved = blob / (gemv_ms * 1e-3) / 1e9 if gemv_ms > 0 else None
        traffic = None  # ncu dram bytes of one launch pair, captured at this slice size only
        prof = os.path.join(ROOT, "profiles", "ncu_expert_gemv_r02.json")
        if os.path.exists(prof) and not sliced(args, n) and args.dtype == "bf16":
            try:
                traffic = json.load(open(prof)).get("dram_bytes_per_expert")
            except Exception:
                traffic = None
        floor_us = None  # pure-read floor of one 352 MB launch (tools/pattern_bench.cu, measured)
        pf = os.path.join(ROOT, "profiles", "pattern_bench_r01.json")
        if os.path.exists(pf) and not sliced(args, n) and args.dtype == "bf16":
            try:
                floor_us = json.load(open(pf))["slices_336MB"]["us_mean"]
            except Exception:
                floor_us = None
        recall = st["correct"] / st["predicted_total"] if st["predicted_total"] else None
        recall_it = st["correct_in_time"] / st["predicted_total"] if st["predicted_total"] else None
        recall_ref = st["refine_correct"] / st["refine_total"] if st["refine_total"] else None
        roof_tok = link_all * 1e9 / (64 * EXPERT_BYTES)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": n, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dev_s / args.steps * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32" if args.dtype == "fp32" else "bf16",
            "data": "synthetic (counter-based splitmix64 weights, U(+-1/sqrt(fan_in)), seed 2512; "
                    "greedy token feedback)",
            "config": workload_config(args, n),
            "recall_eq3": recall,
            "recall_in_time": recall_it,
            "recall_refined": recall_ref,
            "recall_note": "recall_eq3 = Eq. 3 of the token-aligned INT8 shadow (the paper's SEP, prediction "
                           "accuracy); recall_in_time = the same with predictions that reached the host after "
                           "their layer's router scored 0 (S:197); recall_refined = predictions re-anchored at "
                           "the main model's state each layer (refine_depth, DESIGN.md §7), which drive the "
                           "loads when enabled",
            "roofline": {"bound": "hbm", "kernel": "expert SwiGLU GEMV (W13+SwiGLU, W2+gate)",
                         "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                         "frac": achieved / peaks["hbm_gbs"] if achieved else None, "traffic": traffic,
                         "peak_source": peak_src, "bytes_per_launch_pair": blob,
                         "avg_us_per_expert": gemv_ms * 1e3, "w13_us": st["ms_w13"] / n_exp * 1e3,
                         "w2_us": st["ms_w2"] / n_exp * 1e3,
                         "read_floor_us": floor_us,
                         "frac_of_read_floor": (floor_us / (gemv_ms * 1e3)) if (floor_us and gemv_ms > 0) else None,
                         "us_per_expert_by_rank": us_per_rank,
                         "note": "CUDA events around each on-demand launch in the timed step (includes the wait "
                                 "for the copy-stream event and the idle-to-busy ramp); read_floor_us = the same "
                                 "bytes streamed with no arithmetic in one launch (profiles/pattern_bench_r01.json); "
                                 "at N > 1 `achieved` is rank 0's, whose cooperative expert launches also wait for the "
                                 "shadow / refinement kernels sharing its GPU; us_per_expert_by_rank lists every rank"},
            "host_link": {"bound": "pcie_h2d", "achieved": bytes_all / dev_s / 1e9,
                          "peak": link_all, "unit": "GB/s", "frac": bytes_all / dev_s / 1e9 / link_all,
                          "roofline_tok_s": roof_tok, "frac_tok_s": value / roof_tok,
                          "bytes_h2d_per_step": bytes_all / args.steps,
                          "algorithmic_bytes_per_step": 64 * EXPERT_BYTES},
            "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": int(bytes_all / args.steps) + 4,
                    "d2h_bytes_per_step": 4 + (32 * 2 * 4 if True else 0),
                    "note": "odmoe_decode_step with a host token in/out; the H2D bytes are the "
                            "step's expert loads from the pinned host pool"},
            "gpu_launches": st["kernel_launches"],
            "clocks": clk,
            "engine": {"create_s": t_create, "pool_build_s": st["pool_build_s"],
                       "pool_bytes": st["pool_bytes"], "resident_expert_bytes": st["resident_bytes"],
                       "shadow_bytes": st["shadow_bytes"], "reloads": st["reloads"],
                       "loads_cancelled": st["loads_cancelled"], "max_resident": st["max_resident"],
                       "us_router": st["ms_router"] / max(1, st["n_router"]) * 1e3,
                       "us_shadow_per_step": st["ms_shadow"] / args.steps * 1e3,
                       "us_lm_head": st["ms_lm_head"] / max(1, st["n_lm_head"]) * 1e3,
                       "us_attention_per_step": st["ms_attn"] / args.steps * 1e3},
        }
        # GPU memory holding experts (slots on every GPU; + the INT8 shadow on GPU 0)
        # as fractions of the whole model's experts (the paper's "1/3 GPU memory", Q24)
        all_experts = SHAPE["L"] * SHAPE["E"] * EXPERT_BYTES
        slot_bytes = n * st["resident_bytes"]
        line["memory"] = {"expert_slot_bytes_all_gpus": slot_bytes, "all_experts_bytes": all_experts,
                          "slot_fraction": slot_bytes / all_experts, "shadow_bytes_gpu0": st["shadow_bytes"],
                          "with_shadow_fraction": (slot_bytes + st["shadow_bytes"]) / all_experts,
                          "resident_baseline_fraction": 1.0,
                          "note": "peak expert slots x blob on each of the N GPUs (the <1 GB budget per GPU), and "
                                  "that plus the INT8 shadow held by GPU 0, over all L x E experts"}
        # Eq. 1 (reading Q12): t_maxload = N_G t^M + (N_G - 1) t^W, validated per layer
        # against the event trace of the traced steps
        G = args.group_size or min(SHAPE["k"], n)
        ng = 1 if sliced(args, n) else max(1, n // G)
        if trace_ev is not None:
            line["eq1"] = eq1_from_trace(trace_ev, ng, SHAPE["L"], gemv_ms * 1e3 if gemv_ms > 0 else None,
                                         st["ms_router"] / max(1, st["n_router"]) * 1e3)
        sh_rf = shadow_roofline(st, args.steps, peaks["hbm_gbs"])
        if sh_rf is not None:
            sh_rf["note"] = ("per-phase CUDA events inside the decode step (the shadow stream shares the GPU with "
                             "the main model's kernels and copies; each event pair also cuts the PDL chain)")
            line["roofline_shadow"] = sh_rf
        if sh_pass is not None:
            line["roofline_shadow_pass"] = sh_pass
        if r0 is not None:
            line["sep_refine0"] = r0
        if prefill is not None:
            line["prefill"] = prefill
        if res is not None:
            line["resident"] = res
            line["ratio_vs_resident"] = value / res["value"]
            # the same kernel measured live inside the fully-resident decode step of this run
            # (back-to-back launches with PDL; no idle-to-busy ramp per expert)
            line["roofline_resident"] = {"bound": "hbm", "kernel": line["roofline"]["kernel"],
                                         "achieved": res["expert_gemv_GBps"], "peak": peaks["hbm_gbs"],
                                         "unit": "GB/s",
                                         "frac": (res["expert_gemv_GBps"] / peaks["hbm_gbs"]
                                                  if res["expert_gemv_GBps"] else None),
                                         "traffic": traffic, "avg_us_per_expert": res["expert_gemv_us"]}
        if not args.no_cpu_baseline and n == 1:
            log(rank, "cpu baseline (oracle sample)")
            try:
                line["cpu_baseline"] = oracle_sample(24)  # ~10-15 s of timed CPU work on the box
            except Exception as e:  # report, never hide
                line["cpu_baseline"] = {"value": None, "error": repr(e)}
        out = json.dumps(line)
        print(out, file=json_out, flush=True)
        if args.out:
            with open(args.out, "w") as f:
                f.write(out + "\n")
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    faulthandler.cancel_dump_traceback_later()
    log(rank, "done")
    return 0


def leg(eng, torch, barrier, dist, tok, steps, refine, restore):
    """A short extra on-demand leg on the same engine with another refinement depth (time_kernels
    stays on; CUDA-event time, max over ranks). Returns tokens/s, recall and the shadow's GPU time."""
    eng.set_refine_depth(refine)
    tok, _ = eng.decode_step(tok, records=False)
    eng.reset_stats()
    barrier()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        tok, _ = eng.decode_step(tok, records=False)
    b.record()
    barrier()
    sec = a.elapsed_time(b) * 1e-3
    if dist is not None:
        t = torch.tensor([sec], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        sec = float(t[0])
    st = eng.stats()
    out = {"refine_depth": refine, "steps": steps, "value": steps / sec, "unit": UNIT,
           "recall_eq3": st["correct"] / st["predicted_total"] if st["predicted_total"] else None,
           "recall_in_time": st["correct_in_time"] / st["predicted_total"] if st["predicted_total"] else None,
           "reloads_per_step": st["reloads"] / steps, "us_shadow_per_step": st["ms_shadow"] / steps * 1e3,
           "bytes_h2d_per_step": st["bytes_h2d"] / steps, "tok": tok}
    eng.set_refine_depth(restore)
    return out


def shadow_roofline(st, steps, peak):
    """The INT8 shadow's expert phases (one launch per phase for the k experts of a layer) against
    the HBM peak: algorithmic bytes = int8 codes + fp32 row scales of the k experts."""
    if not st.get("n_sh_w13"):
        return None
    k, d, F = SHAPE["k"], SHAPE["d"], SHAPE["F"]
    b13 = k * (2 * F * d + 2 * F * 4)
    b2 = k * (d * F + d * 4)
    if not st.get("n_sh_w2"):  # both phases in one (cooperative) launch per layer
        us = st["ms_sh_w13"] / (st["n_sh_w13"] / k) * 1e3
        return {"bound": "hbm", "kernel": "INT8 shadow expert layer (W13+SwiGLU, grid barrier, W2+gate) of the k "
                                          "experts in one cooperative launch",
                "layer": {"bytes": b13 + b2, "us": us, "GBps": (b13 + b2) / us / 1e3,
                          "frac": (b13 + b2) / us / 1e3 / peak},
                "peak": peak, "unit": "GB/s", "us_shadow_per_step": st["ms_shadow"] / steps * 1e3,
                "frac": (b13 + b2) / us / 1e3 / peak}
    us13 = st["ms_sh_w13"] / (st["n_sh_w13"] / k) * 1e3
    us2 = st["ms_sh_w2"] / (st["n_sh_w2"] / k) * 1e3
    out = {"bound": "hbm", "kernel": "INT8 shadow experts, one launch per phase for the layer's k experts",
           "w13": {"bytes": b13, "us": us13, "GBps": b13 / us13 / 1e3, "frac": b13 / us13 / 1e3 / peak},
           "w2": {"bytes": b2, "us": us2, "GBps": b2 / us2 / 1e3, "frac": b2 / us2 / 1e3 / peak},
           "peak": peak, "unit": "GB/s", "us_shadow_per_step": st["ms_shadow"] / steps * 1e3}
    out["frac"] = (b13 + b2) / (us13 + us2) / 1e3 / peak
    return out


def eq1_from_trace(ev, ng, L, t_w_kernel_us=None, t_m_kernel_us=None):
    """Eq. 1 (worked example P:137; reading Q12) against the measured per-layer trace of this
    rank: t^M_l = main-node time of layer l (previous layer's last expert end -> this layer's routing
    known), t^W_l = expert computation of layer l on this GPU, t_load = one expert load (LoadStart ->
    LoadEnd, landed loads). Eq. 1 predicts an I/O stall at layer l iff t_load > t^maxload = N_G t^M +
    (N_G - 1) t^W; the trace measures one when the expert start waited for its load (ComputeStart -
    RouterDone > 5 us)."""
    import math
    by = {}
    for e in ev:
        by.setdefault(e["type"], []).append(e)
    full = max((e["bytes"] for e in by.get("LoadEnd", [])), default=0)
    starts = {}
    for e in by.get("LoadStart", []):
        if not math.isnan(e["t_us"]):  # (a load stopped before its first chunk never started)
            starts.setdefault((e["step"], e["layer"], e["expert"]), []).append(e["t_us"])
    loads = []
    for e in by.get("LoadEnd", []):
        key = (e["step"], e["layer"], e["expert"])
        if e["bytes"] == full and key in starts and not math.isnan(e["t_us"]):
            loads.append(e["t_us"] - max(starts[key]))
    router = {(e["step"], e["layer"]): e["t_us"] for e in by.get("RouterDone", [])}
    cs, ce, cw = {}, {}, {}
    cstart = {(e["step"], e["layer"], e["expert"]): e["t_us"] for e in by.get("ComputeStart", [])}
    for e in by.get("ComputeStart", []):
        cs.setdefault((e["step"], e["layer"]), []).append(e["t_us"])
    for e in by.get("ComputeEnd", []):
        ce.setdefault((e["step"], e["layer"]), []).append(e["t_us"])
        key = (e["step"], e["layer"], e["expert"])
        if key in cstart:  # this expert's kernel time (its start event fires once its load has landed)
            cw[(e["step"], e["layer"])] = cw.get((e["step"], e["layer"]), 0.0) + e["t_us"] - cstart[key]
    step0 = {e["step"]: e["t_us"] for e in by.get("StepStart", [])}
    tM, tW, stalls = [], [], []
    for (s, l), tr in sorted(router.items()):
        prev = None
        for j in range(l - 1, -1, -1):
            if (s, j) in ce:
                prev = max(ce[(s, j)])
                break
        if prev is None:
            prev = step0.get(s)
        if prev is not None:
            tM.append(tr - prev)
        if (s, l) in cs and (s, l) in cw:
            # expert kernel time of the layer on this GPU: from the kernel timers when given (the
            # split W13 / W2 launches at N > 1 wait for the W2 part between ComputeStart and End)
            tw = t_w_kernel_us * len(cs[(s, l)]) if t_w_kernel_us else cw[(s, l)]
            tW.append(tw)
            # time the layer's expert work spent waiting for its loads once the routing was known
            stalls.append(max(ce[(s, l)]) - tr - tw)
    if not loads or not tM or not tW:
        return {"N_G": ng, "note": "trace incomplete on this rank"}
    mean = lambda v: sum(v) / len(v)  # noqa: E731
    # t^M: the main node's own work per layer. From the trace (previous expert end -> routing known)
    # when this rank computes every layer; with groups the previous layer ran on another GPU, so the
    # router kernel time (kernel timers) is used
    t_M = t_m_kernel_us if (ng > 1 and t_m_kernel_us) else mean(tM)
    t_W, t_load = mean(tW), mean(loads)
    t_max = ng * t_M + (ng - 1) * t_W
    pred_stall = t_load > t_max
    n_stall = sum(1 for x in stalls if x > 5.0)
    return {"N_G": ng, "t_M_us": t_M, "t_W_us": t_W, "t_load_us": t_load, "t_maxload_us": t_max,
            "io_bottlenecked": pred_stall, "layers_traced": len(stalls),
            "stalled_layers_measured": n_stall, "stalled_layers_predicted": len(stalls) if pred_stall else 0,
            "mean_stall_us": mean(stalls), "loads_traced": len(loads),
            "note": "this rank's layers; t^M = previous layer's last expert end -> routing known; t^W = this "
                    "GPU's expert kernel time of the layer; stall = (last expert end - routing known) - t^W, "
                    "the time the layer's expert work waited for its loads (P:124, Fig. 4); CUDA events, "
                    "S:350-358 trace"}


def resident_baseline(odmoe, torch, args, dev, rank, world, dist):
    """Fully-resident baseline (same kernels and placement; every expert a GPU can be assigned is
    preloaded in its HBM; routing consumed on the device, no per-layer host sync). Collective at
    N > 1 (its own NCCL communicator); timed like our arm (events, max over ranks)."""
    uid = None
    if world > 1:
        obj = [odmoe.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    eng = odmoe.Engine(device=dev, rank=rank, world_size=world, nccl_id=uid, predictor=odmoe.PRED_NONE,
                       slots_per_gpu=-1, time_kernels=1, weight_seed=SEED, placement=int(sliced(args, world)),
                       **SHAPE, **attn_kw(args), **model_kw(args, odmoe))
    if args.attention:
        eng.set_position(args.context)
    tok = 1

    def timed():
        nonlocal tok
        for _ in range(args.warmup):
            tok, _ = eng.decode_step(tok, records=False)
        eng.reset_stats()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(args.steps):
            tok, _ = eng.decode_step(tok, records=False)
        b.record()
        torch.cuda.synchronize()
        sec = a.elapsed_time(b) * 1e-3
        if dist is not None:
            t = torch.tensor([sec], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            sec = float(t[0])
        return sec

    # pass 1: CUDA events around the expert launches (the kernel's duration); pass 2: no events
    # (they cut the PDL chains), which gives the baseline's tokens/s
    timed()
    st = eng.stats()
    eng.set_time_kernels(0)
    if args.attention:
        eng.set_position(args.context)
    s = timed()
    eng.close()
    n_exp = max(1, st["n_w13"])
    gemv_ms = (st["ms_w13"] + st["ms_w2"]) / n_exp
    blob = EXPERT_BYTES // world if sliced(args, world) else EXPERT_BYTES
    return {"value": args.steps / s, "unit": UNIT, "ms_per_step": s / args.steps * 1e3,
            "expert_gemv_us": gemv_ms * 1e3,
            "expert_gemv_GBps": blob / (gemv_ms * 1e-3) / 1e9 if gemv_ms > 0 else None,
            "resident_expert_bytes_per_gpu": st["resident_bytes"],
            "hbm_roofline_tok_s_1gpu": measured_peaks()[0]["hbm_gbs"] * 1e9 / (64 * EXPERT_BYTES + SHAPE["V"] * SHAPE["d"] * EXPERT_BYTES // (3 * SHAPE["d"] * SHAPE["F"]))}


if __name__ == "__main__":
    sys.exit(main())
