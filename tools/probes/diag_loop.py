"""Diagnostics: sweep kernel times in different loop patterns (fwd only,
bwd only, full pass, full pass with idle gaps) to separate kernel efficiency
from sustained-load effects (power cap / clocks)."""
import sys, time, json, statistics
sys.path.insert(0, '.')
import torch
from paper_2509_23866_b200 import dart, synth
import bench

dev = torch.device("cuda", 0)
layout, V, dtype, _ = synth.config_layout("single", seed=0)
batch = synth.make_batch("single", seed=0, device=dev, layout=layout, V=V, dtype=dtype)
cfg = dart.Config()
dl = dart.DartLoss(layout, dart.whole_shard(layout), V, cfg, dev, logits_dtype=dtype)
inp = (batch.logits, batch.target, batch.logp_old, batch.logp_rollout, batch.logp_ref)
for _ in range(3):
    dl.run(*inp)
torch.cuda.synchronize()
fb = 18687098880; bb = 33634123776; peak = 6456.5e9

def timed(mode, n=40, gap=0.0):
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(n)]
    for e in evs:
        for x in e: x.record()
    torch.cuda.synchronize()
    clk = bench.ClockSampler(0); clk.start(); time.sleep(0.1)
    for i in range(n):
        dart.set_timing_events(*evs[i])
        if mode in ("fwd", "full"):
            dl.forward(*inp)
        if mode == "full":
            dl.select()
        if mode in ("bwd", "full"):
            dl.backward()
        if gap:
            torch.cuda.synchronize(); time.sleep(gap)
    torch.cuda.synchronize()
    dart.set_timing_events()
    c = clk.stop()
    f = [e[0].elapsed_time(e[1]) for e in evs] if mode != "bwd" else [0]
    b = [e[2].elapsed_time(e[3]) for e in evs] if mode != "fwd" else [0]
    fm, bm = statistics.median(f), statistics.median(b)
    print(json.dumps({"mode": mode, "gap": gap, "fwd_ms": round(fm, 4), "fwd_frac": round(fb / (fm * 1e-3) / peak, 4) if fm else None,
                      "bwd_ms": round(bm, 4), "bwd_frac": round(bb / (bm * 1e-3) / peak, 4) if bm else None, "clocks": c}), flush=True)

timed("fwd")
timed("bwd")
timed("full")
timed("full", n=15, gap=0.05)
timed("fwd", n=15, gap=0.05)
timed("bwd", n=15, gap=0.05)
