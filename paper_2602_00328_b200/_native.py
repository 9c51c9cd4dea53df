"""ctypes binding of libharvest_b200.so (include/harvest_b200.h).

This is the only way the package reaches the GPU.  There is no CPU or eager
fallback: if the library is missing, importing the package raises.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

from ._build import LIB_PATH

HV_OK = 0
HV_E_INVALID = -1
HV_E_NOCAPACITY = -2
HV_E_DOUBLEFREE = -3
HV_E_UNSUPPORTED = -4
HV_E_NOMEM = -5

ENGINE_AUTO = 0
ENGINE_LDG = 1
ENGINE_TMA = 2
ENGINE_LDG256 = 3
ENGINE_LDG16 = 4
ENGINE_CE = 5                    # host-array entry points: every object through the copy engine (cudaMemcpyAsync per contiguous run)
ENGINE_FLAG_INTERLEAVE = 0x100   # HV_ENGINE_FLAG_INTERLEAVE: round-robin chunks over equal-size objects
ENGINES = {"auto": ENGINE_AUTO, "ldg": ENGINE_LDG, "tma": ENGINE_TMA, "ldg256": ENGINE_LDG256,
           "ldg16": ENGINE_LDG16}
ENGINES.update({f"{k}+il": v | ENGINE_FLAG_INTERLEAVE for k, v in list(ENGINES.items())})
ENGINES["ce"] = ENGINE_CE

POOL_VMM = 0
POOL_IPC = 1
POOL_EAGER = 2
POOL_REMOTE = 4
ATTN_OVERLAP_PREVIOUS = 1        # HV_ATTN_OVERLAP_PREVIOUS: programmatic dependent launch of K5
FFN_WAIT_PREVIOUS = 4            # HV_FFN_WAIT_PREVIOUS: K4 as a programmatic dependent of a kernel that wrote its inputs
MOE_OVERLAP_PREVIOUS = 1         # HV_MOE_OVERLAP_PREVIOUS: route / combine as programmatic dependents
FFN_TILED = 2                    # HV_FFN_TILED: K4 over experts stored as swizzled 128 x 64 tiles (bulk-copy stream)
ATTN_BALANCED = 2                # HV_ATTN_BALANCED: K5 as balanced (stream-K) ranges over `splits` CTAs
FFN_OVERLAP_PREVIOUS = 1         # HV_FFN_OVERLAP_PREVIOUS: K4 down behind gate/up
GRAPH_NODE_PRIORITY = 1          # HV_GRAPH_NODE_PRIORITY


class HarvestNativeError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        msg = _lib.hv_error_string(status).decode() if _lib is not None else "library not loaded"
        super().__init__(f"{where}: status {status} ({msg})")


class NoCapacity(HarvestNativeError):
    pass


class NativeDoubleFree(HarvestNativeError):
    pass


u64 = C.c_uint64
u32 = C.c_uint32
i32 = C.c_int
vp = C.c_void_p
P64 = C.POINTER(C.c_uint64)

# name -> argtypes (restype is always int status unless listed in _RESTYPES)
_SIGS = {
    "hv_abi_version": [],
    "hv_error_string": [i32],
    "hv_device_count": [C.POINTER(i32)],
    "hv_sm_count": [i32, C.POINTER(i32)],
    "hv_can_access_peer": [i32, i32, C.POINTER(i32)],
    "hv_enable_peer_access": [i32, i32],
    "hv_device_synchronize": [i32],
    "hv_mem_get_info": [i32, P64, P64],
    "hv_seg_create": [u64, C.POINTER(vp)],
    "hv_seg_destroy": [vp],
    "hv_seg_alloc": [vp, u64, P64],
    "hv_seg_probe": [vp, u64, P64, P64],
    "hv_seg_free": [vp, u64, u64],
    "hv_seg_allocated_bytes": [vp, P64],
    "hv_seg_free_bytes": [vp, P64],
    "hv_seg_num_free": [vp, P64],
    "hv_seg_free_list": [vp, P64, P64],
    "hv_seg_check": [vp],
    "hv_placer_create": [i32, C.c_double, C.c_double, C.c_double, C.c_int64, C.POINTER(vp)],
    "hv_placer_destroy": [vp],
    "hv_placer_add_donor": [vp, i32, vp, u64, u32],
    "hv_placer_set_ceiling": [vp, i32, u64],
    "hv_placer_ceiling": [vp, i32, P64],
    "hv_placer_select": [vp, u64, u32, C.c_double, C.POINTER(i32), i32, C.POINTER(i32)],
    "hv_placer_alloc": [vp, u64, u32, C.c_double, C.POINTER(i32), i32, C.POINTER(i32), P64],
    "hv_placer_spend": [vp, u32, u64, C.c_double],
    "hv_placer_tokens": [vp, u32, C.c_double, C.POINTER(C.c_double)],
    "hv_placer_note_revocation": [vp, i32, C.c_double],
    "hv_placer_churn": [vp, i32, C.c_double, C.POINTER(C.c_int64)],
    "hv_pool_create": [i32, u64, u64, C.POINTER(i32), i32, C.c_uint, C.POINTER(vp)],
    "hv_pool_destroy": [vp],
    "hv_pool_info": [vp, P64, P64, P64, C.POINTER(i32)],
    "hv_pool_commit": [vp, u64, u64],
    "hv_pool_decommit": [vp, u64, u64],
    "hv_pool_committed_bytes": [vp, P64],
    "hv_pool_export_ipc": [vp, vp],
    "hv_pool_import_ipc": [vp, i32, u64, i32, C.POINTER(vp)],
    "hv_chunk_granularity": [i32, P64],
    "hv_chunk_create_shareable": [i32, u64, P64, C.POINTER(i32)],
    "hv_chunk_release": [u64],
    "hv_pool_map_fd": [vp, u64, i32],
    "hv_pool_unmap_chunk": [vp, u64],
    "hv_host_alloc": [u64, C.POINTER(vp), P64],
    "hv_host_alloc_flags": [u64, C.c_uint, C.POINTER(vp), P64],
    "hv_host_free": [vp],
    "hv_host_register": [vp, u64, P64],
    "hv_host_unregister": [vp],
    "hv_dev_alloc": [i32, u64, P64],
    "hv_dev_free": [i32, u64],
    "hv_memcpy_h2d": [u64, vp, u64, vp],
    "hv_memcpy_d2h": [vp, u64, u64, vp],
    "hv_memset_d8": [u64, i32, u64, vp],
    "hv_stream_create": [i32, i32, C.POINTER(vp)],
    "hv_stream_destroy": [vp],
    "hv_stream_priority_range": [i32, C.POINTER(i32), C.POINTER(i32)],
    "hv_graph_instantiate": [vp, C.c_uint, C.POINTER(vp)],
    "hv_graph_launch": [vp, vp],
    "hv_graph_exec_destroy": [vp],
    "hv_stream_synchronize": [vp],
    "hv_event_create": [i32, C.c_uint, C.POINTER(vp)],
    "hv_event_destroy": [vp],
    "hv_event_record": [vp, vp],
    "hv_event_query": [vp, C.POINTER(i32)],
    "hv_event_synchronize": [vp],
    "hv_event_elapsed_ms": [vp, vp, C.POINTER(C.c_float)],
    "hv_stream_wait_event": [vp, vp],
    "hv_kv_gather": [u64, u64, u64, u32, u64, i32, i32, vp],
    "hv_kv_gather_table": [u64, u64, u64, u64, u32, u64, i32, i32, vp],
    "hv_kv_gather_blocks": [u64, u64, u64, u64, u32, u32, u64, i32, i32, vp],
    "hv_kv_gather_blocks_h": [vp, vp, vp, vp, u32, u32, u64, i32, i32, vp],
    "hv_batch_copy": [u64, u64, u64, u32, i32, i32, vp],
    "hv_swap_blocks_batch": [vp, vp, vp, u32, i32, i32, vp],
    "hv_ce_batch_copy": [vp, vp, vp, u32, i32, vp],
    "hv_fill_content": [u64, u64, u64, u32, vp],
    "hv_fill_weights_bf16": [u64, u64, u64, u32, vp],
    "hv_digest": [u64, u64, u32, u64, vp],
    "hv_verify_content": [u64, u64, u64, u32, u64, vp],
    "hv_check_digests": [u64, u64, u64, u32, u64, u64, u64, vp],
    "hv_check_digests_batch": [vp, vp, vp, u32, u64, u64, u64, vp],
    "hv_swap_blocks_batch_checked": [vp, vp, vp, vp, u32, i32, i32, u64, u64, u64, vp],
    "hv_verify_weights_bf16": [u64, u64, u64, u32, u64, vp],
    "hv_launch_count": [P64],
    "hv_expert_ffn_gate_up": [u64, u64, u64, u64, u64, u64, u32, u32, u32, vp],
    "hv_expert_ffn_down": [u64, u64, u64, u64, u64, u32, u32, u32, vp],
    "hv_expert_ffn_max_tokens": [C.POINTER(i32)],
    "hv_expert_ffn_down_ex": [u64, u64, u64, u64, u64, u32, u32, u32, C.c_uint, vp],
    "hv_expert_ffn_gate_up_ex": [u64, u64, u64, u64, u64, u64, u32, u32, u32, C.c_uint, vp],
    "hv_moe_route": [u64, u64, u32, u32, u32, u32, u64, u64, u64, u64, u64, u64, u64, u64, C.c_uint, vp],
    "hv_moe_combine": [u64, u64, u64, u64, u32, u32, u32, C.c_float, C.c_uint, vp],
    "hv_moe_stage_plan": [u64, u64, u64, u64, u64, u32, u64, u64, u64, vp],
    "hv_paged_decode_attention": [u64, u64, u64, u64, u64, u64, u32, u32, u32, u32, u32, u32, C.c_float, vp],
    "hv_paged_decode_attention_ex": [u64, u64, u64, u64, u64, u64, u32, u32, u32, u32, u32, u32, C.c_float,
                                     C.c_uint, vp],
}
_RESTYPES = {"hv_error_string": C.c_char_p}

_lib = None
_lock = threading.Lock()


def exported_symbols() -> list[str]:
    return list(_SIGS)


def load(path: str | None = None):
    """Load the native library (idempotent).  Raises if it is missing."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = path or os.environ.get("HARVEST_B200_LIB", LIB_PATH)
        if not os.path.exists(path):
            raise ImportError(
                f"{path} is missing: build it with `python paper_2602_00328_b200/_build.py` "
                "(the peer-fetch path has no CPU fallback)")
        lib = C.CDLL(path)
        for name, args in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = _RESTYPES.get(name, C.c_int)
        _lib = lib
        return lib


def lib():
    return _lib if _lib is not None else load()


def check(status: int, where: str = "harvest_b200") -> None:
    if status == HV_OK:
        return
    if status == HV_E_NOCAPACITY:
        raise NoCapacity(status, where)
    if status == HV_E_DOUBLEFREE:
        raise NativeDoubleFree(status, where)
    raise HarvestNativeError(status, where)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args), name)


def device_count() -> int:
    n = C.c_int(0)
    call("hv_device_count", C.byref(n))
    return n.value


def c_int_out(name: str) -> int:
    """Call an entry point of the form int f(int* out) and return *out."""
    v = C.c_int(0)
    call(name, C.byref(v))
    return v.value


def launch_count() -> int:
    v = C.c_uint64(0)
    call("hv_launch_count", C.byref(v))
    return v.value


def stream_handle(stream) -> int:
    """Accept a torch.cuda.Stream, a raw int handle or None (legacy default)."""
    if stream is None:
        return 0
    if isinstance(stream, int):
        return stream
    return int(stream.cuda_stream)
