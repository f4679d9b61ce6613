"""Shadow-pass probe (Mixtral shape): builds an on-demand engine with the INT8 shadow and runs
odmoe_predict_ahead (one full token-aligned shadow pass, SEP Mode A) for distinct tokens; prints the
host time per pass. Used under ncu to capture the shadow's expert-phase kernels in isolation.

    python tools/shadow_probe.py [--passes 4]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2512_03927_b200 import odmoe  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--passes", type=int, default=4)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    eng = odmoe.Engine(32, 8, 2, 4096, 14336, 32000, dtype=odmoe.BF16, predictor=odmoe.PRED_SHADOW_INT8,
                       slots_per_gpu=2, weight_seed=2512)
    for t in range(1, args.passes + 1):
        t0 = time.perf_counter()
        eng.predict_ahead(100 + t)
        print(f"pass {t}: {(time.perf_counter() - t0) * 1e3:.2f} ms", flush=True)
    eng.close()


if __name__ == "__main__":
    main()
