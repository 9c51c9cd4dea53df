"""A real vLLM engine (0.22, V1, in-process) serving with the Harvest PEER
medium as its KV offloading connector: a tiny random-weight Llama
(load_format="dummy", no tokenizer, no network), prefix caching on.

  1. generate greedily from a long prompt with offloading to peer HBM;
  2. reset the GPU prefix cache, so the next request finds its prefix only in
     the offload medium, and generate again: the PEER handler loads the
     blocks back (K1 over the block table);
  3. the same two requests on an engine without a connector.

Every output token sequence must be equal.  Prints JSON: outputs equal,
handler load / store job counts, bytes moved.

    python tools/vllm_engine_probe.py
"""
import json
import os
import sys
import tempfile

os.environ.setdefault("VLLM_ENABLE_V1_MULTIPROCESSING", "0")   # scheduler and worker in this process

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def tiny_llama(path):
    cfg = {"architectures": ["LlamaForCausalLM"], "model_type": "llama", "hidden_size": 512,
           "intermediate_size": 1024, "num_hidden_layers": 2, "num_attention_heads": 8, "num_key_value_heads": 4,
           "vocab_size": 2048, "max_position_embeddings": 4096, "rms_norm_eps": 1e-5, "rope_theta": 10000.0,
           "torch_dtype": "bfloat16", "tie_word_embeddings": False, "bos_token_id": 1, "eos_token_id": 2}
    os.makedirs(path, exist_ok=True)
    with open(os.path.join(path, "config.json"), "w") as f:
        json.dump(cfg, f)
    return path


def run(model, offload, prompts):
    from vllm import LLM, SamplingParams
    kw = dict(model=model, load_format="dummy", skip_tokenizer_init=True, enforce_eager=True, seed=0,
              gpu_memory_utilization=0.25, max_model_len=2048, enable_prefix_caching=True, dtype="bfloat16")
    if offload:
        from vllm.config import KVTransferConfig
        kw["kv_transfer_config"] = KVTransferConfig(
            kv_connector="OffloadingConnector", kv_role="kv_both",
            kv_connector_extra_config={"spec_name": "HarvestOffloadingSpec",
                                       "spec_module_path": "paper_2602_00328_b200.vllm_adapter",
                                       "peer_bytes_to_use": 256 << 20})
    llm = LLM(**kw)
    sp = SamplingParams(temperature=0.0, max_tokens=16, detokenize=False)
    outs = []
    first = llm.generate([{"prompt_token_ids": p} for p in prompts], sp, use_tqdm=False)
    outs.append([list(o.outputs[0].token_ids) for o in first])
    llm.reset_prefix_cache()
    second = llm.generate([{"prompt_token_ids": p} for p in prompts], sp, use_tqdm=False)
    outs.append([list(o.outputs[0].token_ids) for o in second])
    stats = None
    if offload:
        # every donor slab revoked (a co-tenant reclaims the HBM): the next
        # lookups are misses and vLLM recomputes -- outputs must not change
        from paper_2602_00328_b200 import vllm_adapter as VA
        from paper_2602_00328_b200.runtime import RevokeReason
        pool = VA._WORKER_POOL[0]
        rt = pool.rt
        before = VA.handler_stats()
        for h in list(pool.slabs.values()):
            if h is not None and rt.is_live(h):
                rt.revoke(h, RevokeReason.EXTERNAL_RECLAIM)
        import torch
        torch.cuda.synchronize()
        rt.sim.run()   # drain: the revocations finish once the reads already enqueued complete
        live_after_revoke = sum(1 for h in pool.slabs.values() if rt.is_live(h))
        llm.reset_prefix_cache()
        third = llm.generate([{"prompt_token_ids": p} for p in prompts], sp, use_tqdm=False)
        outs.append([list(o.outputs[0].token_ids) for o in third])
        stats = VA.handler_stats()
        stats["revoked_slabs"] = len(before) and sum(1 for _ in pool.slabs)
        stats["slabs_live_after_revocation"] = live_after_revoke
        stats["loads_after_revocation"] = stats["load_jobs"] - before["load_jobs"]
        stats["stores_after_revocation"] = stats["store_jobs"] - before["store_jobs"]
    del llm
    return outs, stats


def main():
    import random
    rng = random.Random(0)
    prompts = [[rng.randrange(3, 2048) for _ in range(n)] for n in (900, 517, 1200)]
    model = tiny_llama(os.path.join(tempfile.mkdtemp(), "tiny-llama"))
    res = {"model": "tiny Llama (2 layers, hidden 512, 4 KV heads x 64), dummy weights, bf16",
           "prompts_tokens": [len(p) for p in prompts], "max_tokens": 16, "greedy": True}
    quick = "--quick" in sys.argv   # the offloading engine alone (tests/test_gpu_vllm_engine.py)
    outs_ref = None
    if not quick:
        # the engine without a connector first: a connector's worker registers a
        # process-wide KV transfer group that a later engine would inherit
        outs_ref, _ = run(model, False, prompts)
        res["reference_first"] = outs_ref[0]
        res["reference_after_reset"] = outs_ref[1]
    try:
        outs_off, stats = run(model, True, prompts)
        res["offload"] = {"first": outs_off[0], "after_reset": outs_off[1], "after_revocation": outs_off[2],
                          "handler": stats}
        res["offload_after_reset_equals_first"] = outs_off[1] == outs_off[0]
        res["offload_after_revocation_equals_first"] = outs_off[2] == outs_off[0]
        if outs_ref is not None:
            res["equal_first"] = outs_off[0] == outs_ref[0]
            res["equal_after_reset"] = outs_off[1] == outs_ref[0]
    except Exception:   # noqa: BLE001 -- reported
        import traceback
        res["offload_error"] = traceback.format_exc()[-3000:]
    print(json.dumps(res))


if __name__ == "__main__":
    main()
