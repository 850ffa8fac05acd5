"""The shared-memory bank-conflict model behind the mixed-radix layout
(scripts/tools/bank_sim.py; profiles/round2_mixed_radix.md).  CPU only: it
replays the exchange addresses of LineFFT::run_f (csrc/kernels/fft_core.cuh)."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scripts", "tools"))
import bank_sim as b  # noqa: E402


def pad16(p):
    return p + (p >> 4)


def ident(p):
    return p


def test_plans_match_the_kernels():
    assert b.plan(256) == (16, 16, [16, 16])
    assert b.plan(160) == (20, 8, [5, 4, 4, 2])
    assert b.plan(384) == (12, 32, [3, 4, 4, 4, 2])


def test_power_of_two_layout_is_conflict_free():
    tot, ideal = b.cost(256, (256 + 16) | 1, pad16)
    assert tot == ideal


def test_mixed_radix_layouts():
    # the old layout at 160: stores 3.2x, loads 2x the ideal wavefronts (ncu measured 3.4x / 2.0x)
    old, ideal = b.cost(160, (160 + 10) | 1, pad16)
    assert (old["st"], old["ld"]) == (384, 240) and ideal == {"st": 120, "ld": 120}
    # the chosen one: unpadded, row stride 8 mod 16 (fft_kernels.cuh row_stride<160>() = 168)
    new, _ = b.cost(160, 168, ident)
    assert (new["st"], new["ld"]) == (168, 120)
    new96, ideal96 = b.cost(96, 104, ident)
    assert new96["ld"] == ideal96["ld"] and new96["st"] < b.cost(96, (96 + 6) | 1, pad16)[0]["st"]
