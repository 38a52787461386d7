"""Read+write copy ceiling for SM kernels vs cudaMemcpyAsync (tools only).
Buffer = the single config's logits (61440 x 152064 bf16, 18.7 GB) copied
into a second buffer; GB/s counts read + write bytes."""
import ctypes, json, os, subprocess
import torch
HERE = os.path.dirname(os.path.abspath(__file__))
so = os.path.join(HERE, "libcopyceil.so")
if not os.path.exists(so):
    subprocess.check_call(["nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "--shared", "-Xcompiler",
                           "-fPIC", "-o", so, os.path.join(HERE, "copy_ceiling.cu")])
L = ctypes.CDLL(so)
L.probe.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                    ctypes.c_int, ctypes.c_void_p]
nb = 61440 * 152064 * 2
a = torch.empty(nb, dtype=torch.uint8, device="cuda")
a.fill_(3)
b = torch.empty_like(a)
st = torch.cuda.current_stream().cuda_stream
SM = torch.cuda.get_device_properties(0).multi_processor_count
names = {0: "LDG/STG U1", 1: "LDG/STG U4", 2: "LDG/STG U8", 3: "LDG.nc/STG.cs U4", 4: "LDG.nc/STG.cs U8",
         5: "TMA bulk ring 4x4KB", 6: "TMA bulk ring 6x4KB", 7: "cudaMemcpyAsync D2D"}


def timeit(f, k=8):
    for _ in range(2):
        assert f() == 0
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(k):
        f()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / k


cases = [(7, 1, 1, 0)]
import sys
only_spin = '--spin' in sys.argv
for w in (0, 1, 2, 3, 4):
    for g in (SM * 4, SM * 8, SM * 16):
        cases.append((w, g, 256, 0))
for w in (5, 6):
    for g, blk in ((SM, 256), (SM * 2, 256)) if w == 5 else ((SM, 256),):
        for contig in (1, 0):
            cases.append((w, g, blk, contig))
for w, g, blk, arg in ([] if only_spin else cases):
    ms = timeit(lambda: L.probe(w, a.data_ptr(), b.data_ptr(), nb, g, blk, arg, st))
    ok = bool(torch.equal(a[:1 << 20], b[:1 << 20])) and bool(torch.equal(a[-(1 << 20):], b[-(1 << 20):]))
    b.zero_()
    print(json.dumps({"copy": names[w], "grid": g, "block": blk, "contiguous": arg, "ms": round(ms, 3),
                      "GBps": round(2 * nb / ms / 1e6, 1), "ok": ok}), flush=True)
# is cudaMemcpyAsync D2D on the SMs?  time it while a spin kernel holds every SM
s2 = torch.cuda.Stream()
torch.cuda.synchronize()
L.probe(8, None, None, 0, SM * 8, 1024, 60000, s2.cuda_stream)     # ~30 ms of spinning on all SMs
ms = timeit(lambda: L.probe(7, a.data_ptr(), b.data_ptr(), nb, 1, 1, 0, st), k=3)
torch.cuda.synchronize()
print(json.dumps({"copy": "cudaMemcpyAsync D2D while a spin kernel occupies every SM", "ms": round(ms, 3),
                  "GBps": round(2 * nb / ms / 1e6, 1)}), flush=True)
