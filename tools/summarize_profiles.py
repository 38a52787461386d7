"""Copy the ncu evidence of a gpurun (gpurun_out/) into profiles/<tag>_* and
MERGE per-launch DRAM traffic into profiles/ncu_traffic.json (bench.py's
`roofline.traffic`); print a markdown table of the launch-list shares.

    python tools/summarize_profiles.py r02

Inputs (written on the box by tools/gpu_bench_prof.sh): gpurun_out/launches.csv
(ncu gpu__time_duration launch list of bench.py) and gpurun_out/prof_<k>.ncu-rep
(`ncu --set full` of one launch) for k in fwd, bwd, fused, lmfwd, lmdz (those present)."""
import collections
import csv
import json
import os
import subprocess
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
G, P = "gpurun_out", "profiles"
os.makedirs(P, exist_ok=True)
tpath = f"{P}/ncu_traffic.json"
traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
KEYS = {"fwd": "fwd_sweep", "bwd": "bwd_sweep", "fused": "fused_sweep",
        "lmfwd": "lmhead_fwd", "lmdz": "lmhead_dz"}    # the last two: tools/gpu_prof_lmhead.sh
rows_md = []
for k, key in KEYS.items():
    rep = f"{G}/prof_{k}.ncu-rep"
    if not os.path.exists(rep):
        continue
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    open(f"{P}/{tag}_{key}_raw.csv", "w").write(raw)
    det = subprocess.run(["ncu", "-i", rep, "--page", "details"], capture_output=True, text=True).stdout
    open(f"{P}/{tag}_{key}_details.txt", "w").write(det)
    r = list(csv.reader(raw.splitlines()))
    h, u, v = r[0], r[1], r[2]

    def g(n):
        i = h.index(n)
        x = float(v[i].replace(",", ""))
        m = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-6, "us": 1e-3, "ms": 1,
             "s": 1e3}.get(u[i], 1)
        return x * m
    rd, wr, t = g("dram__bytes_read.sum"), g("dram__bytes_write.sum"), g("gpu__time_duration.sum")
    traffic[key] = {"dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr,
                    "ncu_duration_ms": t, "ncu_GBps": (rd + wr) / (t * 1e-3) / 1e9,
                    "source": f"profiles/{tag}_{key}_raw.csv (ncu --set full, 1 launch, single config)"}
    rows_md.append((key, rd, wr, t))
json.dump(traffic, open(tpath, "w"), indent=1)
if os.path.exists(f"{G}/launches.csv"):
    rows = list(csv.reader(open(f"{G}/launches.csv")))
    open(f"{P}/{tag}_launches.csv", "w").write(open(f"{G}/launches.csv").read())
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hh, data = rows[hi], rows[hi + 1:]
    ki, vi = hh.index("Kernel Name"), hh.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in data:
        name = r[ki].split("(")[0].split("<")[0].replace("void ", "").replace("dart::", "")
        agg[name].append(float(r[vi].replace(",", "")))
    tot = sum(sum(x) for x in agg.values())
    out = ["| kernel | launches | avg (us) | share |", "|---|---|---|---|"]
    for n, x in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"| {n} | {len(x)} | {sum(x)/len(x)/1e3:.1f} | {100*sum(x)/tot:.1f}% |")
    open(f"{P}/{tag}_launch_shares.md", "w").write("\n".join(out) + "\n")
    print("\n".join(out))
for k, rd, wr, t in rows_md:
    print(f"{k}: {t:.3f} ms, read {rd/1e9:.3f} GB, write {wr/1e9:.3f} GB, {(rd+wr)/(t*1e-3)/1e9:.0f} GB/s")
