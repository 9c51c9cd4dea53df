"""The vLLM adapter binds to vLLM's own OffloadingHandler contract when vLLM is
installed (vllm/v1/kv_offload/worker/worker.py:26-75)."""
import inspect

import pytest


def test_adapter_implements_vllm_contract():
    from paper_2602_00328_b200 import vllm_adapter as v
    for name in ("transfer_async", "get_finished", "wait", "shutdown"):
        assert callable(getattr(v.HarvestPeerHandler, name))
    sig = inspect.signature(v.HarvestPeerHandler.transfer_async)
    assert list(sig.parameters) == ["self", "job_id", "spec"]
    if not v.HAVE_VLLM:
        pytest.skip("vLLM not installed")
    from vllm.v1.kv_offload.worker.worker import OffloadingHandler
    assert issubclass(v.HarvestPeerHandler, OffloadingHandler)
    assert v.PeerBlocks.medium() == "PEER" and v.GPUBlocks.medium() == "GPU"
