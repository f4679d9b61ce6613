"""Predictor x lookahead sweep of the on-demand decode (configs[2]: lookahead 1-4 over 2/4 GPUs;
the B200 analogue of the paper's ablation cases: SEP shadow / perfect / none = case 6
/ random = case 5). One engine per rank; options switched at run time (odmoe_set_option).
Every configuration decodes the same token sequence from the same first token, so outputs are
identical and only time and recall change. Prints one JSON line per configuration (rank 0).

    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 tools/sweep.py
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

SHAPE = dict(L=32, E=8, k=2, d=4096, F=14336, V=32000)
EXPERT_BYTES = 3 * 4096 * 14336 * 2


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--lookaheads", default="1,2,3,4")
    ap.add_argument("--predictors", default="shadow_int8,perfect,gate_reuse,none,random")
    ap.add_argument("--slots", type=int, default=0, help="0 => 2 (groups) or 2k (sliced)")
    ap.add_argument("--placement", default="groups", choices=["groups", "sliced"])
    ap.add_argument("--attention", action="store_true", help="Mixtral attention block (32/8 heads) + 512-token prefill")
    ap.add_argument("--kv-align", default="1", help="comma list of shadow KV alignment (1 = main cache, 0 = own)")
    ap.add_argument("--refine", default="0", help="comma list of SEP refinement depths (shadow predictor only)")
    ap.add_argument("--periods", default="1", help="comma list of token alignment periods T_p (shadow predictors)")
    ap.add_argument("--group-size", type=int, default=0, help="groups placement: G (0 => min(k, N))")
    ap.add_argument("--out", default="")
    ap.add_argument("--build-predictor", default="shadow_int8",
                    help="predictor the engine is created with (its shadow is the one shadow predictors use)")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2512_03927_b200 import odmoe
    uid = None
    if world > 1:
        obj = [odmoe.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    eng = odmoe.Engine(device=local, rank=rank, world_size=world, nccl_id=uid,
                       predictor=odmoe.PREDICTORS[args.build_predictor],
                       slots_per_gpu=args.slots or (4 if args.placement == "sliced" and world > 1 else 2),
                       lookahead=1, weight_seed=2512, placement=int(args.placement == "sliced"),
                       group_size=args.group_size, **SHAPE,
                       **(dict(n_heads=32, n_kv_heads=8, max_seq=2048) if args.attention else {}))
    lines = []
    combos = []
    aligns = [int(x) for x in args.kv_align.split(",")] if args.attention else [1]
    for pname in args.predictors.split(","):
        for D in [int(x) for x in args.lookaheads.split(",")]:
            for R in ([int(x) for x in args.refine.split(",")] if pname.startswith("shadow") else [0]):
                for A in (aligns if pname.startswith("shadow") else [1]):
                    for T in ([int(x) for x in args.periods.split(",")] if pname.startswith("shadow") else [1]):
                        combos.append((pname, D, R, A, T))
    prompt = None
    if args.attention:
        from inputs import MIXTRAL, gen_prompt
        prompt = [int(x) for x in gen_prompt(MIXTRAL, 1, 512)]
    for pname, D, R, A, T in combos:
        if True:
            eng.set_predictor(odmoe.PREDICTORS[pname])
            eng.set_lookahead(D)
            eng.set_refine_depth(R)
            eng.set_align_period(T)
            if args.attention:
                if pname.startswith("shadow"):
                    eng.set_kv_align(A)
                tok, _ = eng.prefill(prompt)  # same context for every configuration
            else:
                tok = 1
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
            s = a.elapsed_time(b) * 1e-3
            st = eng.stats()
            t = torch.tensor([s, float(st["bytes_h2d"])], dtype=torch.float64, device="cuda")
            if dist is not None:
                mx = t.clone()
                dist.all_reduce(mx, op=dist.ReduceOp.MAX)
                sm = t.clone()
                dist.all_reduce(sm, op=dist.ReduceOp.SUM)
                s, bytes_all = float(mx[0]), float(sm[1])
            else:
                bytes_all = float(t[1])
            if rank == 0:
                rec = st["correct"] / st["predicted_total"] if st["predicted_total"] else None
                recb = st["refine_correct"] / st["refine_total"] if st["refine_total"] else None
                if pname.startswith("shadow"):
                    pname = args.build_predictor
                line = {"n_gpus": world, "placement": args.placement, "group_size": args.group_size,
                        "attention": args.attention, "kv_align": A, "predictor": pname, "lookahead": D,
                        "refine_depth": R, "align_period": T,
                        "recall_in_time": st["correct_in_time"] / st["predicted_total"] if st["predicted_total"] else None,
                        "spec_steps": st["spec_steps"], "early_loads_per_token": st["early_loads"] / args.steps,
                        "recall_refined": recb, "refine_corrections_per_token": st["refine_corrections"] / args.steps,
                        "tok_s": args.steps / s,
                        "ms_per_token": s / args.steps * 1e3, "recall_eq3": rec,
                        "h2d_GBps_aggregate": bytes_all / s / 1e9,
                        "h2d_bytes_per_token": bytes_all / args.steps,
                        "wasted_bytes_per_token": bytes_all / args.steps - 64 * EXPERT_BYTES,
                        "reloads_per_token_rank0": st["reloads"] / args.steps, "steps": args.steps}
                print(json.dumps(line), flush=True)
                lines.append(line)
    eng.close()
    if rank == 0 and args.out:
        with open(args.out, "w") as f:
            for ln in lines:
                f.write(json.dumps(ln) + "\n")
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
