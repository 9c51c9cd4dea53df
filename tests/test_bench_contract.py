"""The bench.py output contract, checked on the committed bench lines
(profiles/r1_bench_*.json, written by bench.py on a B200) and on the
north_star_targets helper.  CPU only: guards the JSON shape the driver and
the judge read against regressions in bench.py."""
import json
import os
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
PROF = os.path.join(REPO, "profiles")


def _line(name):
    """The newest recorded line of this kind (r2_* supersedes r1_*)."""
    for cand in (name.replace("r1_", "r2_", 1), name):
        p = os.path.join(PROF, cand)
        if os.path.exists(p):
            return json.loads(open(p).read().strip().splitlines()[-1])
    pytest.skip(f"{name} not recorded")


def test_n1_line_has_the_contract_keys():
    d = _line("r1_bench_n1.json")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches", "roofline", "cpu_baseline", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["warmup"] >= 3 and d["higher_is_better"] is True
    assert d["scaling"] == "weak" and d["vs_baseline"] is None and d["data"] == "synthetic"
    assert "workload" in d["config"] and "model" not in d["config"]
    e = d["e2e"]
    assert {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"} <= set(e)
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0 and e["verify_mismatched_words"] == 0
    assert e.get("read_errors", 0) == 0
    r = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(r)
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    c = d["cpu_baseline"]
    assert {"value", "unit", "cores", "kind", "sample"} <= set(c) and c["kind"] in ("port", "reference")
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert d["gpu_launches"] > 0
    be = d["north_star_targets"]["bit_exact"]
    assert be.get("fetch_read_errors", be.get("fetch_verify_mismatched_words")) == 0


def test_reference_line():
    d = _line("r1_bench_reference_n1.json")
    assert d["impl"] == "reference"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["cpu_baseline"]["value"] == d["value"] == d["e2e"]["value"]
    assert d["cpu_baseline"]["cores"] >= 1


@pytest.mark.parametrize("name,world", [("r1_bench_2ranks_1gpu_gloo.json", 2), ("r1_bench_4ranks_1gpu_gloo.json", 4)])
def test_multi_rank_lines(name, world):
    d = _line(name)
    assert d["n_gpus"] == world and len(d["per_rank_GBps"]) == world
    assert d["roofline"]["bound"] == "nvlink"
    assert d["cpu_baseline"].get("skipped")            # timed at N=1 only
    t = d["north_star_targets"]
    assert "stand_in" in t                              # one-GPU stand-ins are labelled as such
    assert t["bit_exact"]["decode_outputs_equal_all_local_under_churn"] is True


def test_targets_helper_on_a_synthetic_line():
    sys.path.insert(0, REPO)
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(REPO, "bench.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    line = {"roofline": {"frac": 0.9}, "single_expert_latency_us": {"peer_vs_host_speedup": 12.0},
            "kv_config1_layer_gather": {"peer_vs_host_speedup": 40.0},
            "decode": {"best": {"mode": "fused_cuda_graph", "speedup_vs_host_offload_per_gpu": 9.0}},
            "e2e": {"verify_mismatched_words": 0}, "churn_config5": {"all_outputs_bit_identical": True}}
    t = b.north_star_targets(line, 8)
    assert t["peer_fetch_frac_of_nvlink"]["value"] == 0.9
    assert t["fetch_latency_host_over_peer"]["value"] == 12.0
    assert t["moe_decode_vs_host_offload"]["mode"] == "fused_cuda_graph"
    assert b.north_star_targets(line, 1)["peer_fetch_frac_of_nvlink"]["value"] is None


def test_workload_routing_matches_the_product():
    """The product-free workload (benchlib/workload.py) routes exactly like
    the product's topk_routing, so both bench arms fetch the same experts."""
    sys.path.insert(0, REPO)
    from benchlib.common import model, routing, shape
    from paper_2602_00328_b200.moe import QWEN15_MOE_A27B, topk_routing
    assert model() == QWEN15_MOE_A27B
    a, b = routing(shape(), 3), topk_routing(QWEN15_MOE_A27B, 32, 3, 2)
    assert all((x == y).all() for ra, rb in zip(a, b) for x, y in zip(ra, rb))


def test_reference_arm_never_loads_the_product():
    """--impl reference maps only the oracle's library (the arm
    must not import paper_2602_00328_b200) and runs every layer."""
    import subprocess
    code = (
        "import sys, runpy\n"
        "sys.argv = ['bench.py', '--impl', 'reference', '--steps', '1', '--warmup', '3']\n"
        "try:\n    runpy.run_path('bench.py', run_name='__main__')\nexcept SystemExit:\n    pass\n"
        "maps = open('/proc/self/maps').read()\n"
        "print('PRODUCT', [k for k in sys.modules if k.startswith('paper_2602')], 'libharvest_b200' in maps)\n")
    env = dict(os.environ, HV_BENCH_QWEN_LAYERS="1")
    r = subprocess.run([sys.executable, "-c", code], cwd=REPO, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = r.stdout.strip().splitlines()
    assert lines[-1] == "PRODUCT [] False"
    d = json.loads(lines[-2])
    assert d["impl"] == "reference" and d["value"] > 0 and "every layer (1)" in d["cpu_baseline"]["sample"]
