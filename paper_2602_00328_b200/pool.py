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


# ---------------------------------------------------------------------------
# cross-process donation: one process per GPU (torchrun), VMM chunks handed
# from the donor's process to its readers as POSIX file descriptors

import json as _json
import os as _os
import socket as _socket
import struct as _struct
import threading as _threading

_HDR = _struct.Struct("!I")


def _send_msg(sock, obj, fds=()):
    data = _json.dumps(obj).encode()
    payload = _HDR.pack(len(data)) + data
    if fds:
        _socket.send_fds(sock, [payload], list(fds))
    else:
        sock.sendall(payload)


def _recv_exact(sock, n, fds_out=None):
    buf = b""
    while len(buf) < n:
        if fds_out is not None and not buf:
            chunk, fds, _flags, _addr = _socket.recv_fds(sock, n - len(buf), 4)
            fds_out.extend(fds)
        else:
            chunk = sock.recv(n - len(buf))
        if not chunk:
            raise ConnectionError("peer closed the donation socket")
        buf += chunk
    return buf


def _recv_msg(sock, want_fds=False):
    fds = [] if want_fds else None
    (n,) = _HDR.unpack(_recv_exact(sock, _HDR.size, fds))
    obj = _json.loads(_recv_exact(sock, n).decode())
    return (obj, fds) if want_fds else obj


class DonorServer:
    """The donor side of cross-process harvesting (one per donor GPU process).

    Readers connect over a Unix socket and ask for chunk ``i`` of their
    section; the server creates it on this GPU (hv_chunk_create_shareable,
    cuMemCreate with a POSIX-FD handle), sends the FD (SCM_RIGHTS) and keeps
    its own handle until the reader releases the chunk -- or disconnects, in
    which case every chunk of that reader is released.  ``budget`` caps the
    bytes any one reader may hold (its section of the donor's harvestable
    range); ``donated_bytes`` is the HBM this GPU currently lends out."""

    def __init__(self, device: int, path: str, chunk_bytes: int, budget: int):
        g = C.c_uint64()
        N.call("hv_chunk_granularity", device, C.byref(g))
        if chunk_bytes % g.value:
            raise ValueError(f"chunk_bytes must be a multiple of the granularity {g.value}")
        self.device, self.path, self.chunk, self.budget = device, path, chunk_bytes, budget
        self._lock = _threading.Lock()
        self._held: dict[tuple[int, int], int] = {}   # (connection id, chunk index) -> driver handle
        self.donated_bytes = 0
        self.peak_donated_bytes = 0
        self.requests = 0
        self.releases = 0           # chunks given back (reader free / revoke / disconnect)
        try:
            _os.unlink(path)
        except FileNotFoundError:
            pass
        self._srv = _socket.socket(_socket.AF_UNIX, _socket.SOCK_STREAM)
        self._srv.bind(path)
        self._srv.listen(64)
        self._stop = False
        self._threads = []
        t = _threading.Thread(target=self._accept, daemon=True)
        t.start()
        self._threads.append(t)

    def _accept(self):
        cid = 0
        while not self._stop:
            try:
                conn, _ = self._srv.accept()
            except OSError:
                return
            cid += 1
            t = _threading.Thread(target=self._serve, args=(conn, cid), daemon=True)
            t.start()
            self._threads.append(t)

    def _release(self, key):
        h = self._held.pop(key, None)
        if h is not None:
            N.call("hv_chunk_release", h)
            self.donated_bytes -= self.chunk
            self.releases += 1

    def _serve(self, conn, cid):
        try:
            while True:
                msg = _recv_msg(conn)
                op, idx = msg.get("op"), int(msg.get("chunk", -1))
                if op == "create":
                    with self._lock:
                        mine = sum(1 for (c, _i) in self._held if c == cid)
                        if (mine + 1) * self.chunk > self.budget or (cid, idx) in self._held:
                            _send_msg(conn, {"ok": False, "error": "over budget or already held"})
                            continue
                        h, fd = C.c_uint64(), C.c_int(-1)
                        try:
                            N.call("hv_chunk_create_shareable", self.device, self.chunk, C.byref(h), C.byref(fd))
                        except N.HarvestNativeError as e:     # the donor has no free HBM left
                            _send_msg(conn, {"ok": False, "error": str(e)})
                            continue
                        self._held[(cid, idx)] = h.value
                        self.donated_bytes += self.chunk
                        self.peak_donated_bytes = max(self.peak_donated_bytes, self.donated_bytes)
                        self.requests += 1
                    try:
                        _send_msg(conn, {"ok": True, "bytes": self.chunk}, fds=[fd.value])
                    finally:
                        _os.close(fd.value)
                elif op == "release":
                    with self._lock:
                        self._release((cid, idx))
                    _send_msg(conn, {"ok": True})
                elif op == "bye":          # the reader unmapped everything: release, then acknowledge
                    with self._lock:
                        for key in [k for k in self._held if k[0] == cid]:
                            self._release(key)
                    _send_msg(conn, {"ok": True})
                    break
        except (ConnectionError, OSError, ValueError):
            pass
        finally:
            with self._lock:
                for key in [k for k in self._held if k[0] == cid]:
                    self._release(key)
            conn.close()

    def close(self):
        """Stop serving; chunks still lent (a reader that never said goodbye)
        are released here, so the donor always gets its HBM back."""
        self._stop = True
        try:
            self._srv.close()
        finally:
            try:
                _os.unlink(self.path)
            except FileNotFoundError:
                pass
            with self._lock:
                for key in list(self._held):
                    self._release(key)


class RemotePool:
    """The reader side: a VA range reserved in this process (HV_POOL_REMOTE)
    whose chunks are donor-created VMM allocations received as FDs.  Same
    interface as PeerPool (commit/decommit with per-chunk reference counts,
    committed_bytes, address, close), so the runtime's harvest_alloc commits
    and its final free decommits exactly as on a single process -- and a
    decommitted chunk is released by the donor, returning the HBM."""

    def __init__(self, path: str, donor: int, nbytes: int, chunk_bytes: int, reader: int,
                 connect_timeout: float = 60.0):
        import time as _time
        self.donor, self.mode, self.path = donor, "remote", path
        self._sock = _socket.socket(_socket.AF_UNIX, _socket.SOCK_STREAM)
        deadline = _time.monotonic() + connect_timeout
        while True:
            try:
                self._sock.connect(path)
                break
            except (FileNotFoundError, ConnectionRefusedError):
                if _time.monotonic() > deadline:
                    raise
                _time.sleep(0.05)
        self._p = C.c_void_p()
        rd = (C.c_int * 1)(reader)
        N.call("hv_pool_create", donor, nbytes, chunk_bytes, rd, 1, N.POOL_REMOTE, C.byref(self._p))
        va, nb, ch, dn = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_int()
        N.call("hv_pool_info", self._p, C.byref(va), C.byref(nb), C.byref(ch), C.byref(dn))
        self.va, self.nbytes, self.chunk_bytes = va.value, nb.value, ch.value
        if self.chunk_bytes != chunk_bytes:
            raise ValueError("chunk_bytes must be a multiple of the VMM granularity")
        self._refs = np.zeros(-(-self.nbytes // self.chunk_bytes), dtype=np.int64)
        self._lock = _threading.Lock()

    def _map(self, ci: int) -> None:
        try:
            _send_msg(self._sock, {"op": "create", "chunk": int(ci)})
            reply, fds = _recv_msg(self._sock, want_fds=True)
        except (OSError, ConnectionError, ValueError) as e:
            # the donor process is gone: to the runtime this is NoCapacity
            raise N.HarvestNativeError(N.HV_E_NOCAPACITY, f"donor unreachable: {e!r}") from e
        try:
            if not reply.get("ok"):
                raise N.HarvestNativeError(N.HV_E_NOCAPACITY, f"donor refused chunk {ci}: {reply.get('error')}")
            N.call("hv_pool_map_fd", self._p, int(ci), fds[0])
        finally:
            for fd in fds:
                _os.close(fd)

    def _unmap(self, ci: int) -> None:
        N.call("hv_pool_unmap_chunk", self._p, int(ci))
        try:
            _send_msg(self._sock, {"op": "release", "chunk": int(ci)})
            _recv_msg(self._sock)
        except (OSError, ConnectionError, ValueError):
            pass   # donor gone: its handle died with it; ours is released above

    def commit(self, offset: int, nbytes: int) -> None:
        if nbytes == 0:
            return
        if offset < 0 or offset + nbytes > self.nbytes:
            raise ValueError("commit outside the pool")
        c0, c1 = offset // self.chunk_bytes, (offset + nbytes - 1) // self.chunk_bytes
        with self._lock:
            done = []
            try:
                for ci in range(c0, c1 + 1):
                    if self._refs[ci] == 0:
                        self._map(ci)
                    self._refs[ci] += 1
                    done.append(ci)
            except Exception:
                for ci in done:             # roll back what this call took
                    self._refs[ci] -= 1
                    if self._refs[ci] == 0:
                        self._unmap(ci)
                raise

    def decommit(self, offset: int, nbytes: int) -> None:
        if nbytes == 0:
            return
        c0, c1 = offset // self.chunk_bytes, (offset + nbytes - 1) // self.chunk_bytes
        with self._lock:
            if (self._refs[c0:c1 + 1] <= 0).any():
                raise ValueError("decommit of an uncommitted range")
            for ci in range(c0, c1 + 1):
                self._refs[ci] -= 1
                if self._refs[ci] == 0:
                    self._unmap(ci)

    @property
    def committed_bytes(self) -> int:
        v = C.c_uint64()
        N.call("hv_pool_committed_bytes", self._p, C.byref(v))
        return v.value

    def address(self, offset: int) -> int:
        return self.va + offset

    def close(self) -> None:
        if self._p:
            N.call("hv_pool_destroy", self._p)      # unmaps whatever is still mapped
            self._p = C.c_void_p()
            try:
                _send_msg(self._sock, {"op": "bye"})
                self._sock.settimeout(30.0)
                _recv_msg(self._sock)           # the donor has released this reader's chunks
            except (OSError, ConnectionError, ValueError):
                pass
            self._sock.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _socket_path(tag: str, rank: int) -> str:
    job = _os.environ.get("MASTER_PORT") or _os.environ.get("TORCHELASTIC_RUN_ID") or str(_os.getppid())
    return f"/tmp/hv-{job}-{tag}-{rank}.sock"


class NodePools:
    """Donor pools of one rank of a one-process-per-GPU node
    (cluster.DonorLayout gives the roles and sections).

    ``mode="remote"`` (default): every donor rank runs a DonorServer; each
    reader opens a RemotePool per donor -- its section, committed chunk by
    chunk as its runtime allocates, released (HBM back to the donor GPU) when
    its runtime frees or revokes.  ``mode="ipc"``: round 1's one cudaMalloc
    slab per donor exported with cudaIpc, backed for the whole run.  If the
    remote setup fails on any rank, every rank falls back to "ipc" (the
    decision is collective, so no rank is left waiting).

    ``views`` maps the reader's peer index (1..n, the reference's device
    ids) to a pool object with the PeerPool interface."""

    def __init__(self, group, layout, rank: int, device_of, mode: str = "remote", tag: str = "main",
                 chunk_bytes: int = 32 << 20):
        self.group, self.layout, self.rank = group, layout, rank
        self.dev = device_of(rank)
        self.views: dict = {}
        self._own = None          # this rank's IPC slab or DonorServer
        self._readers = []        # pools this rank opened
        self.error = None         # set when this rank has no usable pools
        self.fallback_reason = None   # why the remote mode was abandoned (informational)
        self.mode = mode
        if mode == "remote":
            # two phases (servers listen, then readers connect), each closed by
            # a collective status check that doubles as the barrier between
            # them: a failure anywhere sends every rank to the fallback at the
            # same point, so no rank waits in a different collective
            failed = False
            for phase in (self._start_server, self._connect):
                try:
                    phase(device_of, tag, chunk_bytes)
                except Exception as e:   # noqa: BLE001 - reported, then the collective fallback
                    self.fallback_reason = self.fallback_reason or repr(e)[:300]
                if group.any(self.fallback_reason is not None):
                    failed = True
                    break
            if failed:
                self._close_all()
                self.mode = "ipc"
        if self.mode == "ipc":
            self._open_ipc()

    def _start_server(self, device_of, tag, chunk_bytes):
        lay, r = self.layout, self.rank
        self.section_bytes = -(-lay.per_reader // chunk_bytes) * chunk_bytes
        if r in lay.donors and lay.readers_of(r):
            self._own = DonorServer(self.dev, _socket_path(tag, r), chunk_bytes, budget=self.section_bytes)

    def _connect(self, device_of, tag, chunk_bytes):
        lay, r = self.layout, self.rank
        if r in lay.compute:
            for d in lay.donors_of(r):
                p = RemotePool(_socket_path(tag, d), device_of(d), self.section_bytes, chunk_bytes, self.dev,
                               connect_timeout=30.0)
                self._readers.append(p)
                self.views[lay.peer_index(r, d)] = p

    def _open_ipc(self):
        lay, r = self.layout, self.rank
        mine = None
        if r in lay.donors and lay.readers_of(r):
            try:
                self._own = PeerPool(self.dev, lay.slab_bytes(r), readers=[self.dev], mode="ipc")
                mine = self._own.export_ipc()
            except Exception as e:   # noqa: BLE001
                self.error = repr(e)[:300]
        handles = self.group.all_gather(mine)
        self.ipc_handles = handles
        if r in lay.compute:
            try:
                for d in lay.donors_of(r):
                    if handles[d] is None:
                        raise RuntimeError(f"donor rank {d} failed to create its pool")
                    p = PeerPool.import_ipc(handles[d], d, lay.slab_bytes(d), self.dev)
                    self._readers.append(p)
                    self.views[lay.peer_index(r, d)] = p.view(*lay.section(d, r))
            except Exception as e:   # noqa: BLE001 - no views: the caller reports it; close() stays collective
                self.error = repr(e)[:300]
                self.views = {}

    def donor_stats(self) -> dict:
        """This rank's lending (remote mode): chunks created and given back."""
        if isinstance(self._own, DonorServer):
            o = self._own
            return {"chunk_bytes": o.chunk, "created": o.requests, "returned": o.releases,
                    "peak_donated_bytes": o.peak_donated_bytes, "donated_bytes_now": o.donated_bytes}
        return {}

    def donated_bytes(self) -> int:
        """HBM this rank currently lends out (remote mode; the slab size in ipc mode)."""
        if isinstance(self._own, DonorServer):
            return self._own.donated_bytes
        return self._own.nbytes if self._own is not None else 0

    def _close_all(self):
        for p in self._readers:
            try:
                p.close()
            except Exception:   # noqa: BLE001
                pass
        self._readers, self.views = [], {}
        if self._own is not None:
            self._own.close()
            self._own = None

    def close(self) -> None:
        """Close the readers' pools, wait for every rank, then the donors'."""
        for p in self._readers:
            p.close()
        self._readers, self.views = [], {}
        self.group.barrier()
        self.final_stats = self.donor_stats()     # every reader gone: what was lent and given back
        if self._own is not None:
            self._own.close()
            self._own = None
