"""Write-only HBM bandwidth by store flavour (B200), vs copy: is the bwd sweep's
18.7 GB of gradient writes near a write-side bound?"""
import ctypes, json, os, sys
import torch
L = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libwbw.so"))
L.probe.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
nb = 18 << 30
buf = torch.empty(nb, dtype=torch.uint8, device="cuda")
src = torch.empty(nb // 2, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream().cuda_stream
names = {0: "STG.128", 1: "STG.128.cs", 2: "STG.256", 3: "STG.128.cs per-CTA ranges", 4: "TMA bulk store 4KB", 5: "cudaMemsetAsync"}
for which in (0, 1, 2, 3, 4, 5):
    for grid, block in ((148 * 8, 256), (148, 256), (148 * 2, 256)):
        if which == 5 and grid != 148 * 8:
            continue
        f = lambda: L.probe(which, buf.data_ptr(), nb, grid, block, st)
        for _ in range(2):
            assert f() == 0
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(10):
            f()
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / 10
        print(json.dumps({"store": names[which], "grid": grid, "block": block, "write_GBps": round(nb / ms / 1e6, 1)}), flush=True)
a, b = buf[: nb // 2], src
for _ in range(2):
    a.copy_(b)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10):
    a.copy_(b)
e.record()
torch.cuda.synchronize()
print(json.dumps({"copy_GBps(read+write)": round(2 * (nb // 2) / (s.elapsed_time(e) / 10) / 1e6, 1)}))
s.record()
for _ in range(10):
    buf.sum(dtype=torch.int64) if False else torch.ops.aten.amax(buf.view(torch.int64), 0)
e.record()
torch.cuda.synchronize()
print(json.dumps({"read_only_GBps(amax)": round(nb / (s.elapsed_time(e) / 10) / 1e6, 1)}))
