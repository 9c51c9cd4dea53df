"""KV reload through a real vLLM 0.22 engine (the paper's reload experiment,
PAPER.md:323, in a serving engine): a Llama-3-8B-shaped
model (32 layers, 8 KV heads x 128, dummy weights), 4 prompts of 4,096
tokens.  Pass 1 prefills them (and, with a connector, stores their KV);
reset_prefix_cache() drops the GPU copies; pass 2 asks for the same prompts
with max_tokens=1, so its time is the time to get the prefix back:

  recompute   no connector: prefill again
  cpu         vLLM's own CPUOffloadingSpec: reload from pinned host DRAM
  peer        HarvestOffloadingSpec: reload from the peer pool (on one GPU
              the "peer" is this GPU's HBM: a stand-in, not NVLink)

Each engine runs in its own process (a connector's worker registers
process-wide state).  Prints JSON: pass-1 and pass-2 wall ms (median of
3 repetitions of pass 2 after resets), handler stats, output equality.

    python tools/vllm_reload_probe.py            # all three
    python tools/vllm_reload_probe.py --serving  # prefix reuse under GPU KV pressure (serving_child)
    python tools/vllm_reload_probe.py --one MODE # child
"""
import json
import os
import subprocess
import sys
import tempfile
import time

os.environ.setdefault("VLLM_ENABLE_V1_MULTIPROCESSING", "0")
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
PROMPTS, CTX = 4, 4096


def llama8b(path):
    cfg = {"architectures": ["LlamaForCausalLM"], "model_type": "llama", "hidden_size": 4096,
           "intermediate_size": 14336, "num_hidden_layers": 32, "num_attention_heads": 32,
           "num_key_value_heads": 8, "vocab_size": 32768, "max_position_embeddings": 8192, "rms_norm_eps": 1e-5,
           "rope_theta": 500000.0, "torch_dtype": "bfloat16", "tie_word_embeddings": False, "bos_token_id": 1,
           "eos_token_id": 2}
    os.makedirs(path, exist_ok=True)
    with open(os.path.join(path, "config.json"), "w") as f:
        json.dump(cfg, f)
    return path


def serving_child(mode, model, n_prefixes=16, rounds=3, gpu_blocks=1100):
    """Prefix reuse under GPU KV pressure: the GPU holds ~4 of the 16
    prefixes; each round asks for all 16 again (max_tokens=1), so rounds 2..
    find their prefixes only in the offload medium (or recompute them)."""
    import random

    import torch
    from vllm import LLM, SamplingParams
    kw = dict(model=model, load_format="dummy", skip_tokenizer_init=True, enforce_eager=True, seed=0,
              gpu_memory_utilization=0.5, max_model_len=CTX + 64, enable_prefix_caching=True, dtype="bfloat16",
              num_gpu_blocks_override=gpu_blocks, max_num_seqs=4)
    kv_bytes = n_prefixes * CTX * 32 * 8 * 128 * 2 * 2
    if mode != "recompute":
        from vllm.config import KVTransferConfig
        extra = ({"spec_name": "CPUOffloadingSpec", "cpu_bytes_to_use": 2 * kv_bytes} if mode == "cpu" else
                 {"spec_name": "HarvestOffloadingSpec", "spec_module_path": "paper_2602_00328_b200.vllm_adapter",
                  "peer_bytes_to_use": 2 * kv_bytes})
        kw["kv_transfer_config"] = KVTransferConfig(kv_connector="OffloadingConnector", kv_role="kv_both",
                                                    kv_connector_extra_config=extra)
    llm = LLM(**kw)
    rng = random.Random(2)
    prompts = [{"prompt_token_ids": [rng.randrange(3, 32768) for _ in range(CTX)]} for _ in range(n_prefixes)]
    sp = SamplingParams(temperature=0.0, max_tokens=1, detokenize=False)
    times, toks = [], []
    for _ in range(rounds):
        torch.cuda.synchronize()
        a = time.perf_counter()
        outs = llm.generate(prompts, sp, use_tqdm=False)
        torch.cuda.synchronize()
        times.append((time.perf_counter() - a) * 1e3)
        toks.append([o.outputs[0].token_ids[0] for o in outs])
    stats = None
    if mode == "peer":
        from paper_2602_00328_b200 import vllm_adapter as VA
        stats = VA.handler_stats()
    return {"mode": mode, "round_ms": times, "prefix_tokens_per_s_later_rounds":
            n_prefixes * CTX * (rounds - 1) / (sum(times[1:]) * 1e-3), "first_token": toks,
            "handler": stats, "gpu_blocks": gpu_blocks, "prefixes": n_prefixes}


def child(mode, model):
    import random

    import torch
    from vllm import LLM, SamplingParams
    kw = dict(model=model, load_format="dummy", skip_tokenizer_init=True, enforce_eager=True, seed=0,
              gpu_memory_utilization=0.5, max_model_len=CTX + 64, enable_prefix_caching=True, dtype="bfloat16")
    kv_bytes = PROMPTS * CTX * 32 * 8 * 128 * 2 * 2          # K and V of every layer
    if mode != "recompute":
        from vllm.config import KVTransferConfig
        extra = ({"spec_name": "CPUOffloadingSpec", "cpu_bytes_to_use": 2 * kv_bytes} if mode == "cpu" else
                 {"spec_name": "HarvestOffloadingSpec", "spec_module_path": "paper_2602_00328_b200.vllm_adapter",
                  "peer_bytes_to_use": 2 * kv_bytes})
        kw["kv_transfer_config"] = KVTransferConfig(kv_connector="OffloadingConnector", kv_role="kv_both",
                                                    kv_connector_extra_config=extra)
    llm = LLM(**kw)
    rng = random.Random(1)
    prompts = [{"prompt_token_ids": [rng.randrange(3, 32768) for _ in range(CTX)]} for _ in range(PROMPTS)]
    sp1 = SamplingParams(temperature=0.0, max_tokens=8, detokenize=False)
    sp = SamplingParams(temperature=0.0, max_tokens=1, detokenize=False)
    t0 = time.perf_counter()
    first = llm.generate(prompts, sp1, use_tqdm=False)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    # the stores of pass 1 finish asynchronously: give them a moment
    llm.generate([{"prompt_token_ids": [5, 6, 7]}], SamplingParams(max_tokens=1, detokenize=False), use_tqdm=False)
    times, outs = [], None
    for _ in range(3):
        llm.reset_prefix_cache()
        torch.cuda.synchronize()
        a = time.perf_counter()
        outs = llm.generate(prompts, sp, use_tqdm=False)
        torch.cuda.synchronize()
        times.append((time.perf_counter() - a) * 1e3)
    stats = None
    if mode == "peer":
        from paper_2602_00328_b200 import vllm_adapter as VA
        stats = VA.handler_stats()
    times.sort()
    return {"mode": mode, "pass1_ms": (t1 - t0) * 1e3, "pass2_ms": times, "pass2_ms_median": times[1],
            "first_token": [o.outputs[0].token_ids[0] for o in outs],
            "pass1_first_token": [o.outputs[0].token_ids[0] for o in first], "handler": stats,
            "kv_bytes": kv_bytes}


def main():
    serving = "--serving" in sys.argv
    if "--one" in sys.argv:
        mode, model = sys.argv[sys.argv.index("--one") + 1], sys.argv[sys.argv.index("--one") + 2]
        print(json.dumps(serving_child(mode, model) if serving else child(mode, model)))
        return
    model = llama8b(os.path.join(tempfile.mkdtemp(), "llama3-8b-shape"))
    out = {"model": "Llama-3-8B shape (32 layers, 8 KV heads x 128, bf16), dummy weights",
           "prompts": PROMPTS, "context_tokens": CTX, "experiment": "serving" if serving else "reload"}
    for mode in ("recompute", "cpu", "peer"):
        r = subprocess.run([sys.executable, os.path.abspath(__file__), "--one", mode, model]
                           + (["--serving"] if serving else []), capture_output=True,
                           text=True, timeout=1200, cwd=REPO)
        try:
            out[mode] = json.loads(r.stdout.strip().splitlines()[-1])
        except Exception:   # noqa: BLE001 -- reported
            out[mode] = {"error": r.stderr[-2000:]}
    if serving:
        base = out.get("recompute", {}).get("prefix_tokens_per_s_later_rounds")
        for mode in ("cpu", "peer"):
            m = out.get(mode, {})
            if base and m.get("prefix_tokens_per_s_later_rounds"):
                m["speedup_vs_recompute"] = m["prefix_tokens_per_s_later_rounds"] / base
                m["first_tokens_equal_recompute"] = m["first_token"] == out["recompute"]["first_token"]
        print(json.dumps(out, indent=1))
        return
    rec = out.get("recompute", {}).get("pass2_ms_median")
    for mode in ("cpu", "peer"):
        m = out.get(mode, {})
        if rec and m.get("pass2_ms_median"):
            m["pass2_speedup_vs_recompute"] = rec / m["pass2_ms_median"]
            m["first_token_equals_recompute"] = m["first_token"] == out["recompute"]["first_token"]
    if out.get("cpu", {}).get("pass2_ms_median") and out.get("peer", {}).get("pass2_ms_median"):
        out["peer_vs_cpu_reload_speedup"] = out["cpu"]["pass2_ms_median"] / out["peer"]["pass2_ms_median"]
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
