"""NVLink byte counters of one GPU from NVML, read around a timed region.

The hardware evidence that a peer fetch crossed NVLink: the reading GPU's
receive counter grows by (at least) the fetched bytes and each donor's
transmit counter by its share.  NVML exposes per-link data-throughput
counters (NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX/_TX, KiB) and, on newer
drivers, byte counters (NVML_FI_DEV_NVLINK_COUNT_RCV_BYTES/_XMIT_BYTES);
the first family that reads successfully on any link is used, summed over
links.  Without NVML or NVLink the snapshot carries the reason, never a guess.
"""
from __future__ import annotations

MAX_LINKS = 18


class NvlinkCounters:
    def __init__(self, device: int = 0):
        self.device = device
        self.error = None
        self.family = None
        try:
            import pynvml as nv
            nv.nvmlInit()
            self._nv = nv
            self._h = nv.nvmlDeviceGetHandleByIndex(device)
            fams = []
            if hasattr(nv, "NVML_FI_DEV_NVLINK_COUNT_RCV_BYTES") and hasattr(nv, "NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES"):
                fams.append(("count_bytes", nv.NVML_FI_DEV_NVLINK_COUNT_RCV_BYTES,
                             nv.NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES, 1))
            fams.append(("throughput_data_kib", nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX,
                         nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX, 1024))
            for fam in fams:
                vals = self._read(fam)
                if vals is not None:
                    self.family = fam
                    self.links = vals[2]
                    break
            if self.family is None:
                self.error = (f"NVLink byte counters not readable on this GPU (NVML return {self._last_ret} on "
                              f"{nv.nvmlDeviceGetFieldValues.__name__}; 3 = NOT_SUPPORTED)")
        except Exception as e:  # NVML missing or unsupported
            self.error = repr(e)[:200]

    def _read(self, fam):
        nv = self._nv
        _name, rx_id, tx_id, scale = fam
        rx = tx = 0
        links = 0
        self._last_ret = None
        for link in range(MAX_LINKS):
            try:
                r = nv.nvmlDeviceGetFieldValues(self._h, [(rx_id, link), (tx_id, link)])
            except Exception:
                continue
            if r[0].nvmlReturn != 0 or r[1].nvmlReturn != 0:
                self._last_ret = r[0].nvmlReturn or r[1].nvmlReturn
                continue
            rx += _value(r[0]) * scale
            tx += _value(r[1]) * scale
            links += 1
        return (rx, tx, links) if links else None

    def snapshot(self) -> dict:
        if self.family is None:
            return {"error": self.error}
        v = self._read(self.family)
        if v is None:
            return {"error": "counter read failed"}
        return {"rx_bytes": v[0], "tx_bytes": v[1], "links": v[2], "field": self.family[0]}


_ATTR = {0: "dVal", 1: "uiVal", 2: "ulVal", 3: "ullVal", 4: "sllVal", 5: "siVal"}   # nvmlValueType_t


def _value(fv) -> int:
    return int(getattr(fv.value, _ATTR.get(fv.valueType, "ullVal")))


def delta(a: dict, b: dict, seconds: float | None = None) -> dict:
    """Counter growth between two snapshots (and GB/s when a duration is given)."""
    if "error" in a or "error" in b:
        return {"error": a.get("error") or b.get("error")}
    d = {"rx_bytes": b["rx_bytes"] - a["rx_bytes"], "tx_bytes": b["tx_bytes"] - a["tx_bytes"],
         "links": b["links"], "field": b["field"]}
    if seconds:
        d["rx_GBps"] = d["rx_bytes"] / seconds / 1e9
        d["tx_GBps"] = d["tx_bytes"] / seconds / 1e9
    return d
