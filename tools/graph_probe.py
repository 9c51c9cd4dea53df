"""Which pieces of a decode step capture into a CUDA graph?  Prints one JSON
object: piece -> "ok" or the capture error (diagnostic tool, one GPU)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_00328_b200 import _native as N  # noqa: E402
from paper_2602_00328_b200 import fetch as F  # noqa: E402


def try_capture(fn, mode="global"):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    try:
        with torch.cuda.graph(g, capture_error_mode=mode):
            fn()
        g.replay()
        torch.cuda.synchronize()
        return "ok"
    except Exception as e:  # noqa: BLE001
        torch.cuda.synchronize()
        return repr(e)[:200]


def main():
    torch.cuda.set_device(0)
    out = {}
    n, S = 8, 1 << 20
    src = torch.empty(n * S, dtype=torch.uint8, device="cuda")
    dst = torch.empty(n * S, dtype=torch.uint8, device="cuda")
    sp = F.ptrs_tensor([src.data_ptr() + i * S for i in range(n)], "cuda")
    dp = F.ptrs_tensor([dst.data_ptr() + i * S for i in range(n)], "cuda")
    sz = F.ptrs_tensor([S] * n, "cuda")
    h = N.lib()
    import ctypes as C
    s = C.c_void_p()
    N.call("hv_stream_create", 0, 0, C.byref(s))
    ext = torch.cuda.ExternalStream(s.value, device="cuda:0")

    def on_torch_stream():
        F.batch_copy(sp, dp, sz, stream=torch.cuda.current_stream())

    def on_ext_stream():
        cur = torch.cuda.current_stream()
        ext.wait_stream(cur)
        F.batch_copy(sp, dp, sz, stream=s.value)
        cur.wait_stream(ext)

    for mode in ("global", "thread_local", "relaxed"):
        out[f"batch_copy_torch_stream_{mode}"] = try_capture(on_torch_stream, mode)
        out[f"batch_copy_ext_stream_{mode}"] = try_capture(on_ext_stream, mode)
    # isolate the ABI calls the launch path makes
    ev = torch.cuda.Event()
    ev.record()
    torch.cuda.synchronize()
    pieces = {
        "torch_only": lambda: dst.add_(1),
        "hv_memset_d8(bind+memset)": lambda: N.call("hv_memset_d8", dst.data_ptr(), 0, 4096,
                                                    torch.cuda.current_stream().cuda_stream),
        "hv_device_count": lambda: N.device_count(),
        "hv_sm_count": lambda: N.call("hv_sm_count", 0, C.byref(C.c_int())),
    }
    import glob
    rt_paths = glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib",
                                      "libcudart.so*"))
    if rt_paths:  # the runtime query bind_stream_device must avoid under capture
        rt = C.CDLL(rt_paths[0])
        rt.cudaStreamGetDevice.argtypes = [C.c_void_p, C.POINTER(C.c_int)]
        pieces["shared cudart cudaStreamGetDevice"] = lambda: rt.cudaStreamGetDevice(
            torch.cuda.current_stream().cuda_stream, C.byref(C.c_int()))
    for name, fn in pieces.items():
        out[name] = try_capture(fn, "relaxed")
    print(json.dumps(out, indent=1))
    _ = h


if __name__ == "__main__":
    main()
