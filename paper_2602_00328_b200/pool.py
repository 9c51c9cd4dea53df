"""Donor memory pools and the pinned host tier (the three tiers of memalloc.Tier,
memalloc.py:14-17, made real).

* ``PeerPool`` — a donor GPU's harvestable range.  The reference models it as a
  DeviceSpec with ``usable = capacity - reserved - headroom`` (memalloc.py:43-45)
  and never allocates anything; here it is a VA range on the donor whose
  physical chunks are created/mapped only while live segments overlap them
  (``commit``/``decommit``), or a cudaIpc-exportable slab for multi-process use.
* ``HostTier`` — pinned, portable, mapped host DRAM holding the authoritative
  copy of every Backed object (runtime.py:47-49, moe.py:124-129).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N


class PeerPool:
    def __init__(self, donor: int, nbytes: int, readers=(), chunk_bytes: int = 0,
                 mode: str = "vmm", eager: bool = False, _handle=None):
        self.donor = donor
        self.mode = mode
        self._p = C.c_void_p()
        if _handle is not None:
            self._p = _handle
        else:
            rd = (C.c_int * max(1, len(readers)))(*readers)
            flags = N.POOL_IPC if mode == "ipc" else N.POOL_VMM
            if eager:
                flags |= N.POOL_EAGER
            N.call("hv_pool_create", donor, nbytes, chunk_bytes, rd, len(readers), flags, C.byref(self._p))
        va, nb, ch, dn = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_int()
        N.call("hv_pool_info", self._p, C.byref(va), C.byref(nb), C.byref(ch), C.byref(dn))
        self.va, self.nbytes, self.chunk_bytes = va.value, nb.value, ch.value

    def commit(self, offset: int, nbytes: int) -> None:
        N.call("hv_pool_commit", self._p, offset, nbytes)

    def decommit(self, offset: int, nbytes: int) -> None:
        N.call("hv_pool_decommit", self._p, offset, nbytes)

    @property
    def committed_bytes(self) -> int:
        v = C.c_uint64()
        N.call("hv_pool_committed_bytes", self._p, C.byref(v))
        return v.value

    def address(self, offset: int) -> int:
        return self.va + offset

    def export_ipc(self) -> bytes:
        buf = (C.c_char * 64)()
        N.call("hv_pool_export_ipc", self._p, buf)
        return bytes(buf)

    @classmethod
    def import_ipc(cls, handle: bytes, donor: int, nbytes: int, reader: int) -> "PeerPool":
        if len(handle) != 64:
            raise ValueError("cudaIpcMemHandle_t is 64 bytes")
        p = C.c_void_p()
        buf = (C.c_char * 64).from_buffer_copy(handle)
        N.call("hv_pool_import_ipc", buf, donor, nbytes, reader, C.byref(p))
        return cls(donor, nbytes, mode="ipc", _handle=p)

    def view(self, offset: int, nbytes: int) -> "PoolView":
        """A window of a pre-backed (IPC) pool, e.g. one reader's section of a
        donor slab shared by several compute processes."""
        if offset + nbytes > self.nbytes:
            raise ValueError("view outside the pool")
        return PoolView(self, offset, nbytes)

    def close(self) -> None:
        if self._p:
            N.call("hv_pool_destroy", self._p)
            self._p = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class PoolView:
    """Section [offset, offset+nbytes) of an IPC pool; commit/decommit are
    no-ops because IPC slabs are backed for their whole lifetime."""

    def __init__(self, pool: PeerPool, offset: int, nbytes: int):
        self.pool, self.offset = pool, offset
        self.donor, self.mode = pool.donor, "ipc-view"
        self.va, self.nbytes, self.chunk_bytes = pool.va + offset, nbytes, nbytes

    def commit(self, offset: int, nbytes: int) -> None:
        pass

    def decommit(self, offset: int, nbytes: int) -> None:
        pass

    @property
    def committed_bytes(self) -> int:
        return self.nbytes

    def address(self, offset: int) -> int:
        return self.va + offset

    def close(self) -> None:
        pass


class HostTier:
    """Pinned + mapped host memory; ``d_alias`` is its device-visible address."""

    def __init__(self, nbytes: int, write_combined: bool = False):
        self.nbytes = nbytes
        self.write_combined = write_combined
        self.h_ptr = C.c_void_p()
        alias = C.c_uint64()
        N.call("hv_host_alloc_flags", nbytes, 1 if write_combined else 0, C.byref(self.h_ptr), C.byref(alias))
        self.d_alias = alias.value

    def view(self) -> np.ndarray:
        buf = (C.c_uint8 * self.nbytes).from_address(self.h_ptr.value)
        return np.frombuffer(buf, dtype=np.uint8)

    def host_address(self, offset: int = 0) -> int:
        return self.h_ptr.value + offset

    def device_address(self, offset: int = 0) -> int:
        return self.d_alias + offset

    def close(self) -> None:
        if self.h_ptr:
            N.call("hv_host_free", self.h_ptr)
            self.h_ptr = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
