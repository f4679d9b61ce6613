"""Host logic of bench.py (-m "not gpu"): the Eq. 1 analysis of an event trace (Eq. 1,
worked example P:137; reading Q12: t_maxload = N_G t^M + (N_G - 1) t^W) on hand-built traces, and the
argument handling of the FP32 leg (fp32 => one slot)."""
import importlib
import math
import sys

import pytest

import bench

NAN = float("nan")


def ev(type_, step, layer, expert, t_us, nbytes=0):
    return {"type": type_, "step": step, "layer": layer, "expert": expert, "t_us": t_us, "bytes": nbytes}


def two_layer_trace(full=352321536):
    """One step, two layers, two experts each. Layer 0's routing is known at 50 us; its loads land at
    6410 and 12810 us; each expert kernel takes 70 us. Layer 1's routing follows 10 us after layer 0's
    last expert ends."""
    t = [ev("StepStart", 0, -1, -1, 0.0)]
    # layer 0
    t += [ev("LoadIssue", 0, 0, 3, NAN), ev("LoadStart", 0, 0, 3, 10.0), ev("LoadEnd", 0, 0, 3, 6410.0, full)]
    t += [ev("LoadIssue", 0, 0, 5, NAN), ev("LoadStart", 0, 0, 5, 6410.0), ev("LoadEnd", 0, 0, 5, 12810.0, full)]
    t += [ev("RouterDone", 0, 0, -1, 50.0)]
    t += [ev("ComputeStart", 0, 0, 3, 6420.0), ev("ComputeEnd", 0, 0, 3, 6490.0)]
    t += [ev("ComputeStart", 0, 0, 5, 12820.0), ev("ComputeEnd", 0, 0, 5, 12890.0)]
    # layer 1: routing 10 us after layer 0's last expert; its loads ran during layer 0 and landed early
    t += [ev("LoadStart", 0, 1, 0, 12810.0), ev("LoadEnd", 0, 1, 0, 19210.0, full)]
    t += [ev("LoadStart", 0, 1, 1, 19210.0), ev("LoadEnd", 0, 1, 1, 25610.0, full)]
    # a load stopped before its first chunk: no start time, must be ignored
    t += [ev("LoadStart", 0, 1, 7, NAN), ev("LoadEnd", 0, 1, 7, NAN, 0)]
    t += [ev("RouterDone", 0, 1, -1, 12900.0)]
    t += [ev("ComputeStart", 0, 1, 0, 19220.0), ev("ComputeEnd", 0, 1, 0, 19290.0)]
    t += [ev("ComputeStart", 0, 1, 1, 25620.0), ev("ComputeEnd", 0, 1, 1, 25690.0)]
    return t


def test_eq1_single_group_matches_hand_values():
    r = bench.eq1_from_trace(two_layer_trace(), ng=1, L=2, t_w_kernel_us=70.0)
    # t^M: (50 - 0) and (12900 - 12890) -> mean 30; t^W: 2 experts x 70; t_load: 6400 for every landed load
    assert r["N_G"] == 1
    assert r["t_M_us"] == pytest.approx(30.0)
    assert r["t_W_us"] == pytest.approx(140.0)
    assert r["t_load_us"] == pytest.approx(6400.0)
    assert r["t_maxload_us"] == pytest.approx(30.0)          # N_G = 1: t^maxload = t^M
    assert r["loads_traced"] == 4                            # the never-started load is not counted
    assert r["io_bottlenecked"] is True
    # stall = (last expert end - routing known) - t^W: layer 0: 12890 - 50 - 140; layer 1: 25690 - 12900 - 140
    assert r["mean_stall_us"] == pytest.approx(((12890 - 50 - 140) + (25690 - 12900 - 140)) / 2)
    assert r["stalled_layers_measured"] == 2 and r["stalled_layers_predicted"] == 2


def test_eq1_groups_reading_q12():
    """N_G = 2 (the paper's worked example uses N_G groups): t^maxload = 2 t^M + t^W with t^M from
    the router kernel timer; a load shorter than that predicts no stall."""
    tr = two_layer_trace()
    r = bench.eq1_from_trace(tr, ng=2, L=2, t_w_kernel_us=70.0, t_m_kernel_us=7.0)
    assert r["t_M_us"] == pytest.approx(7.0)
    assert r["t_maxload_us"] == pytest.approx(2 * 7.0 + 140.0)
    # shrink every load to 100 us: now t_load < t^maxload, so Eq. 1 predicts no I/O stall
    short = []
    for e in tr:
        e = dict(e)
        if e["type"] == "LoadEnd" and not math.isnan(e["t_us"]) and e["bytes"]:
            starts = [x["t_us"] for x in tr if x["type"] == "LoadStart" and (x["layer"], x["expert"]) == (e["layer"], e["expert"])]
            e["t_us"] = starts[0] + 100.0
        short.append(e)
    r2 = bench.eq1_from_trace(short, ng=2, L=2, t_w_kernel_us=70.0, t_m_kernel_us=7.0)
    assert r2["t_load_us"] == pytest.approx(100.0)
    assert r2["io_bottlenecked"] is False and r2["stalled_layers_predicted"] == 0


def test_eq1_incomplete_trace_is_reported_not_guessed():
    r = bench.eq1_from_trace([ev("StepStart", 0, -1, -1, 0.0)], ng=1, L=2)
    assert "incomplete" in r["note"] and "t_maxload_us" not in r


def test_fp32_leg_arguments(monkeypatch):
    """--dtype fp32: 704.6 MB experts, ONE slot (< 1 GB), no refinement / prefill (bf16
    paths), expert_layer_period 16 by default; the bf16 default is untouched."""
    try:
        monkeypatch.setattr(sys, "argv", ["bench.py", "--dtype", "fp32"])
        a = bench.parse()
        assert a.slots == 1 and a.refine == 0 and a.prefill == 0 and a.layer_period == 16
        assert bench.EXPERT_BYTES == 2 * 3 * 4096 * 14336 * 2
        assert bench.n_slots(a, 1) * bench.EXPERT_BYTES < 1e9
    finally:
        importlib.reload(bench)
    monkeypatch.setattr(sys, "argv", ["bench.py"])
    b = bench.parse()
    assert b.dtype == "bf16" and b.layer_period == 0 and b.refine == 2 and bench.n_slots(b, 1) == 2
    assert bench.EXPERT_BYTES == 352321536


def test_reference_arm_prints_one_contract_line():
    """`bench.py --impl reference` (the oracle as the reference arm, on the host cores): exactly one JSON
    line on stdout with the contract keys, a bounded per-step sample and zero host<->device bytes."""
    import json
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [x for x in out.stdout.splitlines() if x.strip()]
    assert len(lines) == 1
    line = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "dtype", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["unit"] == "tok/s" and line["value"] > 0
    assert line["metric"] == bench.METRIC and line["higher_is_better"] is True
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    # a step is one of the 32 layers of a token: the token takes at least 32 steps' time
    assert 1.0 / line["value"] >= 32 * line["ms_per_step"] * 1e-3 * 0.99
