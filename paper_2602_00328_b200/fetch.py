"""Device-side fetch primitives (K1 KV-page gather, K2 batched fetch, K3 copy-in).

Thin typed wrappers over the C ABI; device buffers are torch tensors (torch
is plumbing for device memory and streams here, the copies are the library's
own sm_100a kernels).  Reference call sites these replace:

* ``kv_gather``       one app_transfer per KV block reload (SPEC.md:408-416,
                      runtime.py:320-364) -> one launch per step x layer
* ``batch_copy``      one app_transfer per activated expert of a stage
                      (moe.py:298-313) -> one launch per stage; also the
                      host->peer placement copy-in of rebalance (moe.py:191-195)
* ``swap_blocks_batch``  vLLM's offload data plane signature
                      (vllm/_custom_ops.py:2681-2703), host int64 arrays
* ``ce_batch_copy``   copy-engine baselines (cudaMemcpyPeerAsync per object,
                      or per contiguous run), the paper's own data path
"""
from __future__ import annotations

import numpy as np
import torch

from . import _native as N


def _engine(engine) -> int:
    if isinstance(engine, int):
        return engine
    return N.ENGINES[engine]


def _dev_u64(t: torch.Tensor, name: str) -> int:
    if t is None:
        return 0
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if t.dtype not in (torch.int64, torch.uint64):
        raise ValueError(f"{name} must be int64")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t.data_ptr()


def kv_gather(src_page_ptrs: torch.Tensor, page_bytes: int, dst: torch.Tensor | None = None,
              dst_page_ptrs: torch.Tensor | None = None, engine="auto", max_ctas: int = 0,
              stream=None) -> None:
    """Copy page i from src_page_ptrs[i] to dst (contiguous, page i at offset
    i*page_bytes) or to dst_page_ptrs[i]."""
    n = src_page_ptrs.numel()
    if dst is None and dst_page_ptrs is None:
        raise ValueError("need dst or dst_page_ptrs")
    if dst is not None and dst.numel() * dst.element_size() < n * page_bytes:
        raise ValueError("dst too small")
    N.call("hv_kv_gather", _dev_u64(src_page_ptrs, "src_page_ptrs"),
           _dev_u64(dst_page_ptrs, "dst_page_ptrs") if dst_page_ptrs is not None else 0,
           dst.data_ptr() if dst is not None else 0, n, page_bytes, _engine(engine), max_ctas,
           N.stream_handle(stream))


def kv_gather_table(slot_bases: torch.Tensor, locs: torch.Tensor, page_bytes: int,
                    dst: torch.Tensor | None = None, dst_page_ptrs: torch.Tensor | None = None,
                    engine="auto", max_ctas: int = 0, stream=None) -> None:
    """K1 with device-side table resolution: page i comes from
    slot_bases[locs[i] >> 32] + (locs[i] & 0xffffffff) * page_bytes."""
    n = locs.numel()
    N.call("hv_kv_gather_table", _dev_u64(slot_bases, "slot_bases"), _dev_u64(locs, "locs"),
           dst.data_ptr() if dst is not None else 0,
           _dev_u64(dst_page_ptrs, "dst_page_ptrs") if dst_page_ptrs is not None else 0,
           n, page_bytes, _engine(engine), max_ctas, N.stream_handle(stream))


def kv_gather_blocks(src_base: torch.Tensor, src_stride: torch.Tensor, dst_base: torch.Tensor,
                     dst_stride: torch.Tensor, n_layers: int, page_bytes: int, engine="auto", max_ctas: int = 0,
                     stream=None) -> None:
    """K1 over a block table with per-layer strides: page (l, b) goes from
    src_base[b] + l*src_stride[b] to dst_base[b] + l*dst_stride[b]."""
    n = src_base.numel()
    if not (src_stride.numel() == dst_base.numel() == dst_stride.numel() == n):
        raise ValueError("block arrays must have equal length")
    N.call("hv_kv_gather_blocks", _dev_u64(src_base, "src_base"), _dev_u64(src_stride, "src_stride"),
           _dev_u64(dst_base, "dst_base"), _dev_u64(dst_stride, "dst_stride"), n, n_layers, page_bytes,
           _engine(engine), max_ctas, N.stream_handle(stream))


def batch_copy(src_ptrs: torch.Tensor, dst_ptrs: torch.Tensor, sizes: torch.Tensor,
               engine="auto", max_ctas: int = 0, stream=None) -> None:
    n = src_ptrs.numel()
    if dst_ptrs.numel() != n or sizes.numel() != n:
        raise ValueError("src_ptrs, dst_ptrs and sizes must have equal length")
    N.call("hv_batch_copy", _dev_u64(src_ptrs, "src_ptrs"), _dev_u64(dst_ptrs, "dst_ptrs"),
           _dev_u64(sizes, "sizes"), n, _engine(engine), max_ctas, N.stream_handle(stream))


def _host_u64(a) -> np.ndarray:
    if isinstance(a, torch.Tensor):
        if a.is_cuda:
            raise ValueError("host arrays expected")
        a = a.numpy()
    return np.ascontiguousarray(a, dtype=np.uint64)


def swap_blocks_batch(src_ptrs, dst_ptrs, sizes, engine="auto", max_ctas: int = 0, stream=None) -> None:
    """vLLM swap_blocks_batch contract: CPU int64 arrays of raw pointers/sizes."""
    s, d, z = _host_u64(src_ptrs), _host_u64(dst_ptrs), _host_u64(sizes)
    if not (len(s) == len(d) == len(z)):
        raise ValueError("length mismatch")
    N.call("hv_swap_blocks_batch", s.ctypes.data, d.ctypes.data, z.ctypes.data, len(s),
           _engine(engine), max_ctas, N.stream_handle(stream))


def ce_batch_copy(src_ptrs, dst_ptrs, sizes, batched: bool = True, stream=None) -> None:
    """Copy-engine baseline: one cudaMemcpyAsync per object, or with
    ``batched`` one per run of objects whose source and destination are both
    contiguous with the previous object's."""
    s, d, z = _host_u64(src_ptrs), _host_u64(dst_ptrs), _host_u64(sizes)
    if not (len(s) == len(d) == len(z)):
        raise ValueError("length mismatch")
    N.call("hv_ce_batch_copy", s.ctypes.data, d.ctypes.data, z.ctypes.data, len(s), int(batched),
           N.stream_handle(stream))


def seeds_tensor(seeds, device) -> torch.Tensor:
    arr = np.asarray([int(x) & ((1 << 64) - 1) for x in seeds], dtype=np.uint64).view(np.int64)
    return torch.from_numpy(arr.copy()).to(device)


def fill_content(dst_ptrs: torch.Tensor, sizes: torch.Tensor, seeds, stream=None) -> None:
    """Write the synthetic content of each object (splitmix64 keyed by its seed)."""
    sd = seeds if isinstance(seeds, torch.Tensor) else seeds_tensor(seeds, dst_ptrs.device)
    N.call("hv_fill_content", _dev_u64(dst_ptrs, "dst_ptrs"), _dev_u64(sizes, "sizes"),
           _dev_u64(sd, "seeds"), dst_ptrs.numel(), N.stream_handle(stream))


def fill_weights_bf16(dst_ptrs: torch.Tensor, sizes: torch.Tensor, seeds, stream=None) -> None:
    """Same keyed stream, each 16-bit lane mapped to a small finite bf16 weight."""
    sd = seeds if isinstance(seeds, torch.Tensor) else seeds_tensor(seeds, dst_ptrs.device)
    N.call("hv_fill_weights_bf16", _dev_u64(dst_ptrs, "dst_ptrs"), _dev_u64(sizes, "sizes"),
           _dev_u64(sd, "seeds"), dst_ptrs.numel(), N.stream_handle(stream))


def digest(src_ptrs: torch.Tensor, sizes: torch.Tensor, stream=None) -> torch.Tensor:
    out = torch.empty(src_ptrs.numel(), dtype=torch.int64, device=src_ptrs.device)
    N.call("hv_digest", _dev_u64(src_ptrs, "src_ptrs"), _dev_u64(sizes, "sizes"), src_ptrs.numel(),
           out.data_ptr(), N.stream_handle(stream))
    return out


def verify_content(src_ptrs: torch.Tensor, sizes: torch.Tensor, seeds, stream=None,
                   weights: bool = False) -> torch.Tensor:
    """Per-object count of 8-byte words that differ from the generator
    (``weights=True``: the bf16-weights variant)."""
    sd = seeds if isinstance(seeds, torch.Tensor) else seeds_tensor(seeds, src_ptrs.device)
    out = torch.empty(src_ptrs.numel(), dtype=torch.int64, device=src_ptrs.device)
    N.call("hv_verify_weights_bf16" if weights else "hv_verify_content", _dev_u64(src_ptrs, "src_ptrs"), _dev_u64(sizes, "sizes"),
           _dev_u64(sd, "seeds"), src_ptrs.numel(), out.data_ptr(), N.stream_handle(stream))
    return out


def ptrs_tensor(ptrs, device) -> torch.Tensor:
    arr = np.asarray(ptrs, dtype=np.uint64).view(np.int64)
    return torch.from_numpy(arr.copy()).to(device)


def layer_runs(src_b, src_s, dst_b, dst_s, page: int, n_layers: int, min_run_bytes: int = 1 << 20):
    """Coalesce a block-table move (page (l, b) from src_b[b] + l*src_s[b] to
    dst_b[b] + l*dst_s[b]) into contiguous runs: consecutive blocks whose
    pages follow each other in both the source and the destination, with the
    same layer strides, form one run per layer.  Returns host arrays
    (src, dst, bytes) of the per-layer runs, or None when the runs are too
    short to be worth it (average under ``min_run_bytes``).  Evicted blocks
    of a sequence usually hold consecutive host slots, so a whole layer of a
    reload is one run -- which the engine per source then hands to the copy
    engine (hv_swap_blocks_batch AUTO)."""
    sb, ss = np.asarray(src_b, dtype=np.uint64), np.asarray(src_s, dtype=np.uint64)
    db, ds = np.asarray(dst_b, dtype=np.uint64), np.asarray(dst_s, dtype=np.uint64)
    n = len(sb)
    if n == 0:
        return None
    pg = np.uint64(page)
    cont = np.ones(n, dtype=bool)
    cont[0] = False
    if n > 1:
        cont[1:] = (sb[1:] == sb[:-1] + pg) & (db[1:] == db[:-1] + pg) & (ss[1:] == ss[:-1]) & (ds[1:] == ds[:-1])
    starts = np.nonzero(~cont)[0]
    lengths = np.diff(np.append(starts, n))
    if lengths.mean() * page < min_run_bytes:
        return None
    lay = np.arange(n_layers, dtype=np.uint64)[:, None]
    src = (sb[starts][None, :] + lay * ss[starts][None, :]).reshape(-1)
    dst = (db[starts][None, :] + lay * ds[starts][None, :]).reshape(-1)
    nbytes = np.broadcast_to(lengths.astype(np.uint64) * pg, (n_layers, len(starts))).reshape(-1)
    return np.ascontiguousarray(src), np.ascontiguousarray(dst), np.ascontiguousarray(nbytes)


def tile_expert_matrix(w: torch.Tensor, inverse: bool = False) -> torch.Tensor:
    """The HV_FFN_TILED storage of one bf16 matrix [R][K] (R % 128 == 0,
    K % 64 == 0): [R/128][K/64] tiles of 128 rows x 64 columns, 16 KiB each,
    row r of a tile holding its 16-byte chunk c at chunk (c ^ (r & 7)) -- the
    128B-swizzled K-major layout the tcgen05 K4 reads, so each tile is one
    bulk copy.  Returns a new [R][K]-sized tensor of the same dtype holding
    the tiled bytes; ``inverse=True`` turns tiled bytes back into the
    row-major matrix.  Pure permutation: any device, no arithmetic."""
    R, K = w.shape
    if R % 128 or K % 64 or w.element_size() != 2:
        raise ValueError("tiled expert matrices are 16-bit [R][K] with R % 128 == 0 and K % 64 == 0")
    r = torch.arange(128, device=w.device)
    c = torch.arange(8, device=w.device)
    sw = c[None, :] ^ (r[:, None] & 7)          # [128, 8]: the XOR is its own inverse
    if not inverse:
        t = w.reshape(R // 128, 128, K // 64, 8, 8).permute(0, 2, 1, 3, 4)    # [rb, kt, r, c, 8 elems]
        return t[:, :, r[:, None], sw].contiguous().view(R, K)
    t = w.reshape(R // 128, K // 64, 128, 8, 8)[:, :, r[:, None], sw]        # [rb, kt, r, c, 8]
    return t.permute(0, 2, 1, 3, 4).contiguous().view(R, K)
