"""CPU: the shared-memory bank model and on-chip roofline (banksim.py), the
counterpart of the reference's declared pmg::banksim (banksim.hpp:112-139)."""

import importlib.util
import os

import pytest

from paper_2405_19004_b200 import banksim as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench():
    spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_conflict_free_and_broadcast():
    f64, f32 = B.BankConfig(word_bytes=8), B.BankConfig(word_bytes=4)
    # stride-1 warp: 2 wavefronts for 8-byte words (two half-warps), 1 for 4-byte
    assert B.instruction_wavefronts([(l, l) for l in range(32)], f64) == (2, 0)
    assert B.instruction_wavefronts([(l, l) for l in range(32)], f32) == (1, 0)
    # everybody reads one word: broadcast
    assert B.instruction_wavefronts([(l, 7) for l in range(32)], f64) == (2, 0)
    assert B.instruction_wavefronts([(l, 7) for l in range(32)], f32) == (1, 0)
    # odd strides are conflict-free, stride 16 (f64) / 32 (f32) serialise fully
    assert B.instruction_wavefronts([(l, 5 * l) for l in range(32)], f64)[1] == 0
    assert B.instruction_wavefronts([(l, 16 * l) for l in range(32)], f64) == (32, 30)
    assert B.instruction_wavefronts([(l, 32 * l) for l in range(32)], f32) == (32, 31)
    # stride 2 in f64: 2-way per half-warp
    assert B.instruction_wavefronts([(l, 2 * l) for l in range(32)], f64) == (4, 2)
    rep = B.count_conflicts([[(l, l) for l in range(32)], [(l, 16 * l) for l in range(32)]], f64)
    assert rep.total_wavefronts == 34 and rep.total_excess == 30


@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("k", range(1, 8))
def test_traffic_model_flops_match_reference_count(dim, k):
    """flops of the model == the instrumented count of the reference's
    contraction sequence (bench.flops_per_patch)."""
    c = B.shared_traffic_model("fused", k, dim, 8)
    assert c.flops == _bench().flops_per_patch(dim, k)
    s = B.shared_traffic_model("solver", k, dim, 8)
    assert 0 < s.flops < c.flops
    # smem intensity rises with the degree (SURVEY.md §8d quotes ~0.15 .. 1.65 flop/B in 3D f64)
    if dim == 3:
        inten = c.flops / (c.bytes_read + c.bytes_written)
        assert abs(inten - [0.149, 0.386, 0.619, 0.853, 1.087, 1.320, 1.553][k - 1]) < 2e-3


def test_onchip_roofline():
    assert abs(B.onchip_bandwidth_tbps(B.A100) - 17.145) < 1e-3
    b200 = B.onchip_bandwidth_tbps(B.B200)
    assert abs(b200 - 148 * 32 * 4 * 1.965e9 / 1.024e12) < 1e-9
    assert B.onchip_roofline(2.0, 1.0, 1.0, B.B200) == pytest.approx(b200)
    with pytest.raises(ValueError):
        B.shared_traffic_model("global", 2, 3, 8)


def test_pp_layout_tables_reproduce_their_modelled_wavefronts():
    """The ping-pong smoother's shared-memory layouts (csrc/smoother_pp_table.hpp)
    are what the bank model says they are: replaying every stage's warp
    accesses (tools/bank_search_pp.py) gives the wavefront count recorded in
    the table, within a bounded excess over the conflict-free ideal (the
    measured counters are in profiles/r02/: LDS/STS 1.07-1.35x, LDGSTS
    staging 2-3.8x)."""
    import re
    import sys

    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import bank_search_pp as B

    src = open(os.path.join(ROOT, "paper_2405_19004_b200", "csrc", "smoother_pp_table.hpp")).read()
    blocks = re.findall(r"modelled (\d+) wavefronts per CTA, ideal (\d+) \(PB=(\d+)\).*?struct PPLayout<(\d), (\d)>"
                        r".*?T\[6\]\[5\] = \{(.*?)\};.*?F\[7\] = \{(.*?)\};", src, re.S)
    assert len(blocks) == 10
    for modelled, ideal, PB, K, W, T, F in blocks:
        K, W, PB = int(K), int(W), int(PB)
        rows = [list(map(int, r.split(","))) for r in re.findall(r"\{([^{}]*)\}", T)]
        flips = list(map(int, F.split(",")))
        c = B.u_read_cost(K, PB, flips[0], W)
        for i, X in enumerate("ABCDEF"):
            s0, s1, s2, arrsep, WW = rows[i]
            c += B.tensor_cost(K, PB, X, flips[i], flips[i + 1], (s0, s1, s2, WW), arrsep, W)
        assert c == int(modelled), (K, W, c, modelled)
        assert B.ideal(K, PB, W) == int(ideal)
        assert c <= 1.3 * int(ideal), (K, W, c / int(ideal))
