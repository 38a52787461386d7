"""Probe: does compressible device memory (cuMemCreate, CU_MEM_ALLOCATION_COMP_GENERIC)
cut the DRAM traffic of the gradient buffer (20% of its rows are zero-filled)?"""
import sys, time, json
sys.path.insert(0, '.')
import torch
from cuda.bindings import driver as D

torch.cuda.init()
dev = torch.device("cuda", 0)
torch.zeros(1, device=dev)


def chk(r):
    err = r[0] if isinstance(r, tuple) else r
    if err != D.CUresult.CUDA_SUCCESS:
        raise RuntimeError(str(err))
    return r[1] if isinstance(r, tuple) and len(r) > 1 else None


cu_dev = chk(D.cuDeviceGet(0))
sup = chk(D.cuDeviceGetAttribute(D.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_GENERIC_COMPRESSION_SUPPORTED, cu_dev))
print("generic compression supported:", sup, flush=True)


class Arr:
    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"data": (ptr, False), "shape": shape, "typestr": typestr, "version": 3}


def comp_alloc(nbytes, comp=True):
    prop = D.CUmemAllocationProp()
    prop.type = D.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
    prop.location.type = D.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
    prop.location.id = 0
    if comp:
        prop.allocFlags.compressionType = int(D.CUmemAllocationCompType.CU_MEM_ALLOCATION_COMP_GENERIC)
    gran = chk(D.cuMemGetAllocationGranularity(prop, D.CUmemAllocationGranularity_flags.CU_MEM_ALLOC_GRANULARITY_RECOMMENDED))
    size = (nbytes + gran - 1) // gran * gran
    h = chk(D.cuMemCreate(size, prop, 0))
    got = chk(D.cuMemGetAllocationPropertiesFromHandle(h))
    ptr = chk(D.cuMemAddressReserve(size, 0, 0, 0))
    chk(D.cuMemMap(ptr, size, 0, h, 0))
    acc = D.CUmemAccessDesc()
    acc.location.type = D.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
    acc.location.id = 0
    acc.flags = D.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
    chk(D.cuMemSetAccess(ptr, size, [acc], 1))
    return int(ptr), size, got.allocFlags.compressionType


def timeit(f, n=20):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        f()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / n


nb = 8 << 30
ptr, size, ct = comp_alloc(nb, True)
print("compressible alloc type:", ct, flush=True)
comp = torch.as_tensor(Arr(ptr, (nb // 2,), "<i2"), device=dev).view(torch.bfloat16)
norm = torch.empty(nb // 2, dtype=torch.bfloat16, device=dev)
src = torch.randn(nb // 2, device=dev, dtype=torch.bfloat16)
for name, t in (("normal", norm), ("compressible", comp)):
    tz = timeit(lambda: t.zero_())
    tr = timeit(lambda: t.copy_(src))
    t.zero_()
    tsum = timeit(lambda: t.sum(), 10)
    print(json.dumps({"buf": name, "zero_fill_GBps": nb / tz / 1e6, "copy_random_GBps": 2 * nb / tr / 1e6,
                      "read_zeros_GBps": nb / tsum / 1e6}), flush=True)

# the real pass: gradient buffer in compressible memory
from paper_2509_23866_b200 import dart, synth
layout, V, dtype, _ = synth.config_layout("single", seed=0)
batch = synth.make_batch("single", seed=0, device=dev, layout=layout, V=V, dtype=dtype)
dl = dart.DartLoss(layout, dart.whole_shard(layout), V, dart.Config(), dev)
inp = (batch.logits, batch.target, batch.logp_old, batch.logp_rollout, batch.logp_ref)
T, ldg = dl.dlogits_store.shape
del comp, norm, src
torch.cuda.empty_cache()
ptr2, size2, _ = comp_alloc(T * ldg * 2, True)
cbuf = torch.as_tensor(Arr(ptr2, (T * ldg,), "<i2"), device=dev).view(torch.bfloat16).view(T, ldg)
ref_store = dl.dlogits_store
for name, store in (("normal", ref_store), ("compressible", cbuf), ("normal", ref_store), ("compressible", cbuf)):
    dl.dlogits_store = store
    dl.dlogits = store[:, :V]
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(20)]
    for e in evs:
        for x in e:
            x.record()
    for _ in range(3):
        dl.run(*inp)
    torch.cuda.synchronize()
    for i in range(20):
        dart.set_timing_events(*evs[i])
        dl.run(*inp)
    torch.cuda.synchronize()
    dart.set_timing_events()
    f = sorted(e[0].elapsed_time(e[1]) for e in evs)[10]
    b = sorted(e[2].elapsed_time(e[3]) for e in evs)[10]
    print(json.dumps({"dlogits": name, "fwd_ms": f, "bwd_ms": b}), flush=True)
eq = torch.equal(cbuf[:, :V], ref_store[:, :V])
print("same gradient bits:", eq)
