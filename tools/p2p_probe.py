"""Per-expert kernel durations on every rank from the engine's event trace (N GPUs, on-demand, sliced):
which expert launches the fused P2P send slows, and by how much. Writes gpurun_out/p2p_probe_<tag>.json.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/p2p_probe.py --tag f1
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

SHAPE = dict(L=32, E=8, k=2, d=4096, F=14336, V=32000)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", default="x")
    ap.add_argument("--steps", type=int, default=3)
    args = ap.parse_args()
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    import torch.distributed as dist
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2512_03927_b200 import odmoe
    obj = [odmoe.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    eng = odmoe.Engine(device=local, rank=rank, world_size=world, nccl_id=obj[0], predictor=odmoe.PRED_SHADOW_INT8,
                       slots_per_gpu=4, lookahead=1, weight_seed=2512, refine_depth=2, placement=1, **SHAPE)
    tok = 1
    for _ in range(3):
        tok, _ = eng.decode_step(tok, records=False)
    eng.set_trace(True)
    for _ in range(args.steps):
        tok, _ = eng.decode_step(tok, records=False)
    torch.cuda.synchronize()
    ev = eng.trace()
    eng.close()
    cs = {(e["step"], e["layer"], e["expert"]): e["t_us"] for e in ev if e["type"] == "ComputeStart"}
    rows = []
    for e in ev:
        if e["type"] != "ComputeEnd":
            continue
        key = (e["step"], e["layer"], e["expert"])
        if key in cs:
            rows.append((e["step"], e["layer"], e["expert"], cs[key], e["t_us"]))
    by_layer = {}
    for s, l, x, t0, t1 in rows:
        by_layer.setdefault((s, l), []).append((t0, t1))
    first, last = [], []
    for v in by_layer.values():
        v.sort()
        if len(v) >= 2:
            first.append(v[0][1] - v[0][0])
            last.append(v[-1][1] - v[-1][0])
    res = {"rank": rank, "tag": args.tag, "layers": len(by_layer),
           "first_expert_us": sum(first) / max(1, len(first)), "last_expert_us": sum(last) / max(1, len(last)),
           "last_minus_first_us": (sum(last) - sum(first)) / max(1, len(last))}
    out = [None] * world
    dist.all_gather_object(out, res)
    if rank == 0:
        os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
        with open(os.path.join(ROOT, "gpurun_out", f"p2p_probe_{args.tag}.json"), "w") as f:
            json.dump(out, f, indent=1)
        print(json.dumps(out))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
