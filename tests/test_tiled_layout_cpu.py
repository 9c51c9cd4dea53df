"""The HV_FFN_TILED expert layout on the host side (CPU, no GPU): the tile
permutation (fetch.tile_expert_matrix) and its inverse, the byte position of
an element against the layout the header states, and ExpertStore's argument
checks.  The GPU tests check that K4 over tiled bytes equals K4 over
row-major bytes bit for bit."""
import pytest
import torch


def test_tile_roundtrip_and_element_position():
    from paper_2602_00328_b200 import fetch as F
    R, K = 384, 192
    w = torch.arange(R * K, dtype=torch.int32).to(torch.int16).view(R, K)
    t = F.tile_expert_matrix(w)
    assert t.shape == w.shape and t.dtype == w.dtype
    assert torch.equal(F.tile_expert_matrix(t, inverse=True), w)
    flat = t.reshape(-1)
    for rb, kt, r, c, e in [(0, 0, 0, 0, 0), (1, 2, 3, 2, 5), (2, 1, 127, 7, 7), (0, 2, 9, 4, 1)]:
        # tile (rb, kt) is 128 x 64 elements; row r's 16-byte chunk c sits at chunk c ^ (r & 7)
        idx = (rb * (K // 64) + kt) * 128 * 64 + r * 64 + (c ^ (r & 7)) * 8 + e
        assert flat[idx] == w[rb * 128 + r, kt * 64 + c * 8 + e]


def test_tile_rejects_shapes_the_kernel_cannot_read():
    from paper_2602_00328_b200 import fetch as F
    with pytest.raises(ValueError):
        F.tile_expert_matrix(torch.zeros(192, 64, dtype=torch.int16))    # rows not a multiple of 128
    with pytest.raises(ValueError):
        F.tile_expert_matrix(torch.zeros(128, 96, dtype=torch.int16))    # columns not a multiple of 64
    with pytest.raises(ValueError):
        F.tile_expert_matrix(torch.zeros(128, 64, dtype=torch.float32))  # not 16-bit


def test_expert_store_layout_arguments():
    from paper_2602_00328_b200.moe import ExpertStore, MoEProfile
    ok = MoEProfile("t", 1, 2, 1, 3 * 256 * 128 * 2, hidden=256, intermediate=128)
    odd = MoEProfile("t", 1, 2, 1, 3 * 256 * 192 * 2, hidden=256, intermediate=192)
    assert ExpertStore(ok, 0).layout == "row"
    with pytest.raises(ValueError):
        ExpertStore(ok, 0).fill_host(layout="columns")
    with pytest.raises(ValueError):
        ExpertStore(ok, 0).fill_host(layout="tiled")                 # tiles are a layout of bf16 weights
    with pytest.raises(ValueError):
        ExpertStore(odd, 0).fill_host(weights=True, layout="tiled")  # 192 rows: not 128-row tiles
