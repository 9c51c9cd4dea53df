"""Pin the CPU oracle before trusting it (CPU tier, no GPU).

* stable_hash64 / expert_content against values the reference produced
  (tests/golden/stable_hash64.json; runtime.py:38-44, moe.py:114-115);
* the splitmix64 content generator against the published known-answer vectors
  (Vigna, splitmix64.c, state 0) and a pure-Python restatement;
* best_fit / free_coalesce against the reference allocator's recorded runs
  (tests/golden/allocator.json; memalloc.py:90-138) and SPEC.md:56-58;
* stage_fetch_plan against the reference decode's recorded fetches
  (tests/golden/moe_fetch.json; moe.py:282-313);
* resolve_fallback against SPEC.md:417-425's examples.
"""
import json
import os

import numpy as np
import pytest

from oracle import harvest_oracle as O

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    with open(os.path.join(G, name)) as f:
        return json.load(f)


def test_stable_hash64_matches_reference():
    g = load("stable_hash64.json")
    for tag, val in zip(g["tags"], g["values"]):
        assert O.stable_hash64(*tag) == int(val)
    assert O.expert_seed("qwen2-moe", 3, 7) == int(g["expert_content_qwen2_3_7"])


def test_splitmix64_known_answers():
    # Vigna's splitmix64.c with x = 0: the first three next() outputs
    kat = [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]
    assert [O.content_word(0, i) for i in range(3)] == kat
    assert O.content_words_py(0, 3) == kat
    for seed in (1, 0xDEADBEEF, (1 << 64) - 1, O.expert_seed("m", 1, 2)):
        assert [O.content_word(seed, i) for i in range(64)] == O.content_words_py(seed, 64)


@pytest.mark.parametrize("n", [0, 1, 7, 8, 9, 4096, 65536 + 3])
def test_content_bytes_and_digest(n):
    seed = O.kv_seed(1, 2, 3)
    buf = O.content(seed, n)
    words = O.content_words_py(seed, (n + 7) // 8)
    want = b"".join(w.to_bytes(8, "little") for w in words)[:n]
    assert buf.tobytes() == want
    assert O.digest(buf) == O.content_digest(seed, n)
    if n:
        b2 = buf.copy()
        b2[n // 2] ^= 1
        assert O.digest(b2) != O.digest(buf)


def test_gather_restatement():
    rng = np.random.default_rng(0)
    src = rng.integers(0, 255, size=1 << 20, dtype=np.uint8)
    dst = np.zeros_like(src)
    sizes = [1000, 0, 12345, 65536, 7]
    offs = np.cumsum([0] + sizes[:-1])
    perm = [3, 0, 4, 1, 2]
    sp = [src.ctypes.data + int(offs[p]) for p in perm]
    doffs = np.cumsum([0] + [sizes[p] for p in perm][:-1])
    dp = [dst.ctypes.data + int(o) for o in doffs]
    O.gather(sp, dp, [sizes[p] for p in perm], threads=3)
    pos = 0
    for p in perm:
        assert np.array_equal(dst[pos:pos + sizes[p]], src[offs[p]:offs[p] + sizes[p]])
        pos += sizes[p]


def test_best_fit_matches_reference_runs():
    g = load("allocator.json")
    for case in g["cases"]:
        fl = [(0, case["usable"])]
        for kind, a, b, want in case["ops"]:
            if kind == "alloc":
                base, fl = O.best_fit(fl, a)
                assert base == want
            else:
                fl = O.free_coalesce(fl, a, b)
        assert [list(x) for x in fl] == case["free_list"]
    for ex in g["spec_examples"]:
        base, fl = O.best_fit([tuple(x) for x in ex["free_list"]], ex["size"])
        assert base == ex["base"] and [list(x) for x in fl] == ex["after"]


def test_select_device_spec_example():
    # free 10 GiB and 2 GiB, request 1.5 GiB -> the 2 GiB peer
    GiB = 1 << 30
    cands = [{"dev": 1, "free_list": [(0, 10 * GiB)], "allocated": 0, "ceiling": 10 * GiB},
             {"dev": 2, "free_list": [(0, 2 * GiB)], "allocated": 0, "ceiling": 2 * GiB}]
    assert O.select_device(cands, 3 * GiB // 2) == 2
    assert O.select_device(cands, 11 * GiB) is None
    assert O.select_device(cands, 1 << 20, "Locality", hops={1: 1, 2: 2}) == 1


def test_stage_fetch_plan_matches_reference_decode():
    g = load("moe_fetch.json")
    for name in ("qwen15_b32_peer50", "qwen15_b32_host100", "qwen15_b32_peer100_7donors",
                 "phi35_b16_peer100_7donors"):
        c = g[name]
        L = len(c["active"][0])
        nmb = len(c["active"])
        tiers, live = {}, {}
        for key, (tier, h) in c["residency"].items():
            layer, e = map(int, key.split(","))
            tiers[(layer, e)] = {"LocalHBM": "local", "PeerHBM": "peer", "HostDRAM": "host"}[tier]
            live[(layer, e)] = h is not None
        want = [(f[0], f[1], f[2]) for f in c["fetches"]]
        got = []
        for layer in range(L):
            for mb in range(nmb):
                plan = O.stage_fetch_plan(tuple(c["active"][mb][layer]),
                                          {e: tiers[(layer, e)] for e in c["active"][mb][layer]},
                                          {e: live[(layer, e)] for e in c["active"][mb][layer]})
                got += [(layer, e, t) for e, t in plan]
        assert got == want
        assert c["read_errors"] == 0


def test_resolve_fallback_spec_examples():
    # recompute_time_per_entry = 0 -> Recompute always
    assert O.resolve_fallback(100, 65536, 0.0, 2.5e-6, 55e9, backed=True) == "Recompute"
    # very fast host link -> FetchFromHost for Backed
    assert O.resolve_fallback(100, 65536, 1e-6, 0.0, 1e18, backed=True) == "FetchFromHost"
    # Lossy without host copy -> Recompute
    assert O.resolve_fallback(100, 65536, 1.0, 0.0, 1e18, backed=False, host_copy=False) == "Recompute"
    # crossover: alpha + e*b/B == e*r  ->  e* = alpha / (r - b/B)
    a, b, B, r = 10e-6, 1000, 1e9, 2e-6
    e_star = a / (r - b / B)
    assert O.resolve_fallback(int(e_star) + 2, b, r, a, B, True) == "FetchFromHost"
    assert O.resolve_fallback(max(1, int(e_star) - 2), b, r, a, B, True) == "Recompute"


def _nh_digest_py(buf: bytes) -> int:
    """The digest's definition (oracle/hv_oracle.c header) in plain Python."""
    M32, M64 = (1 << 32) - 1, (1 << 64) - 1
    acc = len(buf)
    for i in range(0, len(buf), 8):
        w = int.from_bytes(buf[i:i + 8].ljust(8, b"\0"), "little")
        j = (i // 8 + 1) & M32
        a = ((w & M32) + j * 0x9E3779B1) & M32
        b = ((w >> 32) + j * 0x85EBCA77 + 0xC2B2AE3D) & M32
        acc = (acc + a * b) & M64
    return acc


@pytest.mark.parametrize("n", [0, 5, 8, 64, 1001])
def test_digest_matches_its_definition(n):
    """The C digest (and so the device kernels, which tests/test_gpu_fetch.py
    compares with it) equals the NH definition written out in Python; a single
    changed word, two swapped words, or a page moved by one word all change it."""
    seed = O.expert_seed("nh", 1, n)
    buf = O.content(seed, n)
    assert O.digest(buf) == _nh_digest_py(buf.tobytes()) == O.content_digest(seed, n)
    if n >= 16:
        swapped = buf.copy()
        swapped[0:8], swapped[8:16] = buf[8:16].copy(), buf[0:8].copy()
        assert O.digest(swapped) != O.digest(buf)
        shifted = np.concatenate([buf[8:], buf[:8]])
        assert O.digest(shifted) != O.digest(buf)
