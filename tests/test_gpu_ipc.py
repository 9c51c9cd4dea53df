"""Cross-process peer pool (cudaIpc, the one-process-per-GPU path bench.py
uses at N>1), exercised with two processes on one GPU: the donor process
creates and fills an IPC pool and exports its handle; the reader process
imports it and fetches through K2; bytes must match the oracle."""
import os
import subprocess
import sys
import textwrap

import pytest

pytestmark = pytest.mark.gpu
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

DONOR = textwrap.dedent("""
    import sys, time, os
    sys.path.insert(0, {repo!r})
    import torch
    from paper_2602_00328_b200.pool import PeerPool
    from paper_2602_00328_b200 import fetch as F
    S, n = 1 << 20, 8
    p = PeerPool(0, S * n, readers=[0], mode="ipc")
    F.fill_content(F.ptrs_tensor([p.address(i * S) for i in range(n)], "cuda:0"),
                   F.ptrs_tensor([S] * n, "cuda:0"), list(range(100, 100 + n)))
    torch.cuda.synchronize()
    open({hpath!r} + ".tmp", "wb").write(p.export_ipc())
    os.replace({hpath!r} + ".tmp", {hpath!r})
    while not os.path.exists({done!r}):
        time.sleep(0.05)
    p.close()
""")

READER = textwrap.dedent("""
    import sys, time, os
    sys.path.insert(0, {repo!r})
    import numpy as np, torch
    from paper_2602_00328_b200.pool import PeerPool
    from paper_2602_00328_b200 import fetch as F
    from oracle import harvest_oracle as O
    S, n = 1 << 20, 8
    while not os.path.exists({hpath!r}):
        time.sleep(0.05)
    p = PeerPool.import_ipc(open({hpath!r}, "rb").read(), 0, S * n, 0)
    dst = torch.empty(S * n, dtype=torch.uint8, device="cuda:0")
    order = list(range(n))[::-1]
    F.batch_copy(F.ptrs_tensor([p.address(e * S) for e in order], "cuda:0"),
                 F.ptrs_tensor([dst.data_ptr() + i * S for i in range(n)], "cuda:0"), F.ptrs_tensor([S] * n, "cuda:0"))
    torch.cuda.synchronize()
    got = dst.cpu().numpy()
    for i, e in enumerate(order):
        assert np.array_equal(got[i * S:(i + 1) * S], O.content(100 + e, S)), e
    p.close()
    open({done!r}, "w").write("ok")
    print("reader ok")
""")


def test_ipc_pool_two_processes(tmp_path):
    hpath, done = str(tmp_path / "handle"), str(tmp_path / "done")
    env = dict(os.environ, PYTHONPATH=REPO)
    d = subprocess.Popen([sys.executable, "-c", DONOR.format(repo=REPO, hpath=hpath, done=done)], env=env)
    try:
        r = subprocess.run([sys.executable, "-c", READER.format(repo=REPO, hpath=hpath, done=done)], env=env,
                           capture_output=True, text=True, timeout=240)
        assert r.returncode == 0, r.stderr[-2000:]
        assert "reader ok" in r.stdout
    finally:
        open(done, "w").write("x")
        d.wait(timeout=60)
    assert d.returncode == 0
