"""tools/timeline_probe.py's interval analysis (CPU): fetch-class and
compute-class intervals merged per class and intersected, on a synthetic
CUPTI/Kineto chrome trace."""
import gzip
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(os.path.dirname(HERE), "tools"))


def test_overlap_fractions(tmp_path):
    import timeline_probe as T
    ev = [
        {"ph": "X", "cat": "kernel", "name": "desc_op_kernel<CopyOpT<0, 8>>", "ts": 0, "dur": 10, "args": {"stream": 7}},
        {"ph": "X", "cat": "kernel", "name": "nvjet_gemm", "ts": 5, "dur": 10, "args": {"stream": 9}},
        {"ph": "X", "cat": "gpu_memcpy", "name": "Memcpy HtoD (Pinned -> Device)", "ts": 20, "dur": 4,
         "args": {"stream": 7}},
        {"ph": "X", "cat": "gpu_memcpy", "name": "Memcpy DtoH (Device -> Pageable)", "ts": 30, "dur": 1,
         "args": {"stream": 7}},
        {"ph": "X", "cat": "kernel", "name": "silu", "ts": 22, "dur": 1, "args": {"stream": 9}},
        {"ph": "X", "cat": "kernel", "name": "paged_decode_mma", "ts": 40, "dur": 10, "args": {"stream": 9}},
        {"ph": "X", "cat": "kernel", "name": "paged_decode_mma", "ts": 45, "dur": 10, "args": {"stream": 9}},
        {"ph": "X", "cat": "cpu_op", "name": "aten::mm", "ts": 0, "dur": 100},
    ]
    p = tmp_path / "t.json.gz"
    with gzip.open(p, "wt") as f:
        json.dump({"traceEvents": ev}, f)
    r = T.analyse(str(p))
    assert (r["fetch_events"], r["compute_events"]) == (2, 5)
    assert r["fetch_busy_us"] == 14 and r["overlap_us"] == 6
    assert r["compute_busy_us"] == 11 + 1 + 15           # gemm 5-15, silu, DtoH, two overlapping K5 40-55
    assert abs(r["fetch_hidden_frac"] - 6 / 14) < 1e-12
    assert r["span_us"] == 55
    assert abs(r["compute_concurrency"] - (10 + 1 + 1 + 20) / 27) < 1e-12
