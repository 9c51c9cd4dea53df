"""A real vLLM engine (0.22, V1, in-process scheduler and worker) serving with
the Harvest PEER medium as its KV offloading connector (tools/
vllm_engine_probe.py --quick, in a subprocess so the engine's process-wide
state and memory stay out of the other tests): prompts prefilled once store
their KV blocks to the peer pool; after the GPU prefix cache is reset the
same prompts find their prefixes only there, the handler loads them back, and
the greedy outputs are identical to the first pass -- and again after every
donor slab has been revoked (the lookups miss and the engine recomputes)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_vllm_engine_serves_through_the_peer_medium():
    pytest.importorskip("vllm")
    r = subprocess.run([sys.executable, os.path.join(REPO, "tools", "vllm_engine_probe.py"), "--quick"],
                       capture_output=True, text=True, timeout=900, cwd=REPO)
    assert r.returncode == 0, r.stderr[-3000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    assert "offload_error" not in res, res.get("offload_error")
    h = res["offload"]["handler"]
    assert h["store_jobs"] > 0 and h["store_blocks"] > 0
    assert h["load_jobs"] > 0 and h["load_blocks"] > 0 and h["failed_loads"] == 0
    assert res["offload_after_reset_equals_first"]
    # every donor slab revoked mid-serving: lookups miss, vLLM recomputes, same outputs
    assert h["revoked_slabs"] > 0 and h["slabs_live_after_revocation"] == 0
    assert h["loads_after_revocation"] == 0 and h["stores_after_revocation"] > 0   # misses, recomputed, re-stored
    assert res["offload_after_revocation_equals_first"]
