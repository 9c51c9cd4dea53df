"""resolve_fallback on measured costs:
the crossover solver and the decision boundary, checked against the
oracle's restatement of the SPEC rule, on both sides of the crossover."""
import math

import pytest

from oracle import harvest_oracle as O


def _link(fc, bw):
    from paper_2602_00328_b200.interconnect import LinkKind, LinkSpec
    return LinkSpec(LinkKind.HOST_LINK, fc, bw, endpoints=(0, 1))


# host links and per-entry recompute rates of the magnitude measured on B200
# (fixed ~10 us, 55 GB/s; Llama-3-8B KV 131,072 B per entry)
CASES = [(10e-6, 55e9, 131072, 2.5e-6), (10e-6, 55e9, 131072, 3.1e-6), (40e-6, 20e9, 131072, 9e-6),
         (2e-6, 770e9, 131072, 2e-7), (10e-6, 55e9, 70272, 1.4e-6)]


@pytest.mark.parametrize("fc,bw,bpe,rate", CASES)
def test_linear_crossover_flips_exactly_at_the_closed_form(fc, bw, bpe, rate):
    """with host (alpha, B) and recompute rate r the decision
    flips where alpha + e*b/B = e*r.  Below e* Recompute, at and above it
    FetchFromHost -- for the product's solver, KVCacheManager's rule and the
    oracle alike."""
    from paper_2602_00328_b200.costs import fallback_crossover, fetch_wins
    link = _link(fc, bw)
    out = fallback_crossover(link, bpe, rate, max_entries=1 << 14)
    e_star = out["closed_form_e_star"]
    assert e_star is not None and e_star > 0
    lo, hi = math.floor(e_star), math.ceil(e_star)
    if lo == hi:
        lo -= 1
    for e, want in ((lo, "Recompute"), (hi, "FetchFromHost")):
        if e < 1:
            continue
        assert O.resolve_fallback(e, bpe, rate, fc, bw, backed=True) == want
        assert fetch_wins(link, e, bpe, rate) == (want == "FetchFromHost")
    if lo >= 1:
        assert out["flips"] == [{"last_entries_recompute": lo, "first_entries_fetch": hi}]
    else:
        assert out["flips"] == [] and out["decision_at_1"] == "FetchFromHost"


def test_no_crossover_when_recompute_is_cheaper_per_entry():
    """r <= b/B: recompute wins at every size (no flip), as the closed form says."""
    from paper_2602_00328_b200.costs import fallback_crossover
    out = fallback_crossover(_link(10e-6, 55e9), 131072, 1e-6)
    assert out["closed_form_e_star"] is None and out["flips"] == []
    assert out["decision_at_1"] == out["decision_at_max"] == "Recompute"
    assert O.resolve_fallback(5000, 131072, 1e-6, 10e-6, 55e9, backed=True) == "Recompute"


def test_measured_curve_crossover():
    """A measured recompute curve (weight-bound at small chunks, compute-bound
    at large ones) against a host link: the solver's flip points agree with
    evaluating both costs at every entry count."""
    from paper_2602_00328_b200.costs import RecomputeCost, fallback_crossover, fetch_wins
    curve = RecomputeCost([(1, 30e-6), (16, 40e-6), (256, 400e-6), (4096, 6e-3)])
    link = _link(20e-6, 10e9)
    out = fallback_crossover(link, 131072, curve, max_entries=8192)
    brute = [fetch_wins(link, e, 131072, curve) for e in range(1, 8193)]
    flips = [e + 1 for e in range(1, 8192) if brute[e] != brute[e - 1]]
    assert [f.get("first_entries_fetch", f.get("first_entries_recompute")) for f in out["flips"]] == flips
    assert curve(8) == pytest.approx(30e-6 + 10e-6 * 7 / 15)
    assert curve(8192) == pytest.approx(12e-3)


def test_kv_manager_uses_the_measured_costs():
    """KVCacheManager.resolve_fallback reads set_costs()' link and recompute
    (no GPU needed: the decision is host-side arithmetic)."""
    from paper_2602_00328_b200.kv import KVBlock, KVCacheManager, KVTier, LLAMA3_8B
    from paper_2602_00328_b200.runtime import Durability
    kv = KVCacheManager.__new__(KVCacheManager)
    kv.m = LLAMA3_8B
    kv.set_costs(host_link=_link(10e-6, 55e9), recompute=2.5e-6)
    e_star = 10e-6 / (2.5e-6 - 131072 / 55e9)
    for e in (math.floor(e_star), math.ceil(e_star)):
        b = KVBlock(0, 0, 0, e, Durability.BACKED, KVTier.NOT_MATERIALIZED, host_slot=3)
        want = O.resolve_fallback(e, 131072, 2.5e-6, 10e-6, 55e9, backed=True)
        assert kv.resolve_fallback(b) == want
    b = KVBlock(0, 0, 0, 16, Durability.LOSSY, KVTier.NOT_MATERIALIZED)
    assert kv.resolve_fallback(b) == "Recompute"


def test_layer_runs_coalesces_consecutive_blocks():
    """F.layer_runs: consecutive blocks contiguous in source and destination
    (same layer strides) become one run per layer; a break starts a new run;
    short average runs are left to the per-page kernel (None)."""
    import numpy as np
    from paper_2602_00328_b200 import fetch as F
    page, L = 4096, 3
    sb = [1000 * page + i * page for i in range(6)] + [5000 * page + i * page for i in range(4)]
    db = [i * page for i in range(10)]
    ss, ds = [64 * page] * 10, [16 * page] * 10
    src, dst, nb = F.layer_runs(sb, ss, db, ds, page, L, min_run_bytes=4 * page)
    assert len(src) == L * 2
    want = []
    for l in range(L):
        want += [(1000 * page + l * 64 * page, l * 16 * page, 6 * page),
                 (5000 * page + l * 64 * page, 6 * page + l * 16 * page, 4 * page)]
    assert sorted(zip(src.tolist(), dst.tolist(), nb.tolist())) == sorted(want)
    # every page is covered exactly once
    assert int(nb.sum()) == 10 * L * page
    assert F.layer_runs(sb, ss, db, ds, page, L, min_run_bytes=1 << 20) is None
    # a stride change breaks a run even when the bases are contiguous
    ss2 = list(ss)
    ss2[3] = 32 * page
    src2, _, nb2 = F.layer_runs(sb, ss2, db, ds, page, L, min_run_bytes=page)
    assert len(src2) == L * 4 and int(nb2.sum()) == 10 * L * page
