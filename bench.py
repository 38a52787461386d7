#!/usr/bin/env python
"""DART loss-pass benchmark (BASELINE.json metric):
"loss fwd+bwd logit-tokens/s at V=152064 bf16, % of HBM peak, 1/2/4/8 GPU".

One step = one whole pass over one batch: fwd sweep (all rows) -> C1
all-gather of step entropies (N > 1) -> select -> bwd sweep (kept rows read +
written, masked rows written as zeros) -> C2 stats all-reduce (N > 1).

Usage:  python bench.py [--gpus N] [--steps K] [--warmup W] [--config single]
        python bench.py --impl reference ...   (the float64 CPU oracle arm)
For N > 1 either launch with torchrun (one rank per GPU, NCCL; the driver's
way) or run `python bench.py --gpus N`, which starts the N ranks itself the
same way.  Weak scaling: every rank owns its own batch of the config (its own
rewards, drawn with seed + 1000 r; global G = 8 N for `single`).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM = 6650.0  # GB/s, /opt/skills/guides/B200_PROFILING.md fallback


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def hbm_peak():
    try:
        with open(PEAKS_PATH) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown," \
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown," \
             "clocks_event_reasons.sw_power_cap,power.draw,clocks.mem"

    def __init__(self, index):
        self.index = index
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                       "--format=csv,noheader,nounits", "-lms", "50"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        time.sleep(0.06)
        self.p.terminate()
        try:
            out, _ = self.p.communicate(timeout=5)
        except Exception:
            self.p.kill()
            out, _ = self.p.communicate()
        rows = []
        for line in out.strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                rows.append(parts)
            except Exception:
                pass
        if not rows:
            return None
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i].lower() == "active"})
        pw, mem = [], []
        for r in rows:
            try:
                pw.append(float(r[7]))
            except (ValueError, IndexError):
                pass
            try:
                mem.append(float(r[8]))
            except (ValueError, IndexError):
                pass
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows), "power_w": statistics.median(pw) if pw else None,
                "mem_mhz": statistics.median(mem) if mem else None}


# ------------------------------------------------------------------ setup
def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        dev = local % max(torch.cuda.device_count(), 1)
        torch.cuda.set_device(dev)
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:   # test path: several ranks may share one GPU; collectives staged via host
            dist.init_process_group("gloo")
    else:
        if torch.cuda.is_available():
            torch.cuda.set_device(0)
    return world, rank, local


def rank_seed(seed, r):
    """Seed of rank r's own batch (rank 0 keeps the N = 1 seed)."""
    return seed + 1000 * r


def weak_layouts(config, seed, world):
    """Weak scaling: every rank owns its own batch of `config` (its own
    rewards and, for ragged configs, its own lengths), drawn with
    rank_seed(seed, r).  Returns (per-rank layouts, global layout = their
    concatenation with group ids offset, shards = the per-rank blocks, V,
    dtype).  All ranks compute the same global layout."""
    from paper_2509_23866_b200 import dart, synth
    lays = []
    V = dtype = None
    for r in range(world):
        L, V, dtype, _ = synth.config_layout(config, seed=rank_seed(seed, r))
        lays.append(L)
    tg, tr, tso, sto, fk, shards = [], [], [0], [0], [], []
    g0 = n0 = s0 = t0 = 0
    for L in lays:
        tg.append(L.traj_group + g0)
        tr.append(L.traj_reward)
        tso.extend((L.traj_step_off[1:] + s0).tolist())
        sto.extend((L.step_tok_off[1:] + t0).tolist())
        fk.append(L.step_fork)
        shards.append(dart.Shard(n0, n0 + L.N_traj, s0, s0 + L.S, t0, t0 + L.T))
        g0, n0, s0, t0 = g0 + L.G, n0 + L.N_traj, s0 + L.S, t0 + L.T
    glayout = synth.Layout(G=g0, traj_group=np.concatenate(tg).astype(np.int32),
                           traj_reward=np.concatenate(tr).astype(np.float32),
                           traj_step_off=np.asarray(tso, dtype=np.int64),
                           step_tok_off=np.asarray(sto, dtype=np.int64), step_fork=np.concatenate(fk))
    return lays, glayout, shards, V, dtype


def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def self_launch(args, argv):
    """`python bench.py --gpus N` without torchrun: launch N ranks the way the
    driver does (torch.distributed.run, one process per GPU, 127.0.0.1) and
    pass rank 0's JSON line through.  Returns the launcher's exit code."""
    if args.backend == "nccl" and not args.dry_run:
        n = torch.cuda.device_count()
        if n < args.gpus:
            log(f"--gpus {args.gpus} needs {args.gpus} visible GPUs for one NCCL rank per GPU, found {n}")
            return 2
        from paper_2509_23866_b200 import build as B      # build once, before the ranks start
        B.build()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + list(argv)
    log("launching: " + " ".join(cmd))
    return subprocess.call(cmd)


def run_dry(args):
    """--dry-run (CPU, any backend): the N-rank plumbing without kernels --
    launch, weak-scaling layouts and shards, C1 (all-gather of per-rank
    step values padded to S_pad) and C2 (all-reduce) over the process group,
    max-over-ranks timing -- so the launcher and the collectives' shapes
    can be tested on a host without a GPU.  Prints a JSON line with
    "dry_run": true and no throughput."""
    import torch.distributed as tdist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        tdist.init_process_group("gloo")
    lays, glayout, shards, V, _ = weak_layouts(args.config, args.seed, world)
    me = shards[rank]
    S_pad = max(s.S_loc for s in shards)
    local = torch.full((S_pad,), -1.0, dtype=torch.float32)
    local[:me.S_loc] = torch.arange(me.step_begin, me.step_end, dtype=torch.float32)
    t0 = time.perf_counter()
    if world > 1:
        gathered = torch.empty(world * S_pad, dtype=torch.float32)
        tdist.all_gather_into_tensor(gathered, local)
        stats = torch.tensor([float(me.T_loc), float(me.S_loc)], dtype=torch.float64)
        tdist.all_reduce(stats)
    else:
        gathered, stats = local, torch.tensor([float(me.T_loc), float(me.S_loc)], dtype=torch.float64)
    ms = torch.tensor([(time.perf_counter() - t0) * 1e3], dtype=torch.float64)
    if world > 1:
        tdist.all_reduce(ms, op=tdist.ReduceOp.MAX)
    # C1 delivered every rank's steps, in global step order, at rank r's padded slot
    g = gathered.view(world, S_pad)
    order_ok = all(bool(torch.equal(g[r, :s.S_loc], torch.arange(s.step_begin, s.step_end, dtype=torch.float32)))
                   for r, s in enumerate(shards))
    if rank == 0:
        print(json.dumps({
            "dry_run": True, "metric": METRIC, "value": None, "unit": "logit-tokens/s", "n_gpus": world,
            "steps": 0, "warmup": 0, "ms_per_step": None, "collectives_ms_max_over_ranks": float(ms),
            "backend": tdist.get_backend() if world > 1 else None,
            "config": {"workload": args.config, "global_tokens": glayout.T, "groups": glayout.G,
                       "steps_total": glayout.S, "tokens_per_rank": [s.T_loc for s in shards],
                       "rewards_distinct_per_rank": world == 1 or any(
                           not np.array_equal(lays[0].traj_reward, L.traj_reward) for L in lays[1:]),
                       "parallelism": f"dp{world} (trajectory-sharded)"},
            "c1_layout_ok": order_ok, "c2_sum_tokens": float(stats[0]), "c2_sum_steps": float(stats[1])}),
            flush=True)
    if world > 1:
        tdist.barrier()
        tdist.destroy_process_group()


METRIC = "loss fwd+bwd logit-tokens/s at V=152064 bf16, % of HBM peak, 1/2/4/8 GPU"


CONFIG_DESC = {
    "single": "single GPU: 8 tasks x 8 rollouts x 15 steps x 64 tokens (T=61440), V=152064 bf16",
    "single_ragged": "8 tasks x 8 rollouts, ragged 1-15 steps x 64 tokens, V=152064 bf16",
    "mid": "2 tasks x 4 rollouts, ragged, V=152064 bf16 (parity size)",
}


# ------------------------------------------------------------------ streamed arm
def run_streamed(args):
    """Configs whose logits exceed HBM (long-horizon 249 GB, scale sweep):
    forward over chunks -> select -> backward over chunks, logits/dlogits in a
    pool of P buffers (chunk c -> slot c mod P in both sweeps; the synthetic
    slot contents are generated once, so both sweeps read identical bytes).
    N > 1 (torchrun): the config's batch is the GLOBAL batch (strong scaling),
    sharded into token-balanced ranges of whole trajectories; each rank
    streams its own shard, C1 all-gathers every rank's per-chunk step
    entropies, one selection, C2 all-reduces the statistics."""
    from paper_2509_23866_b200 import build as B
    if int(os.environ.get("RANK", "0")) == 0:
        B.build()
    world, rank, local = dist_setup(args)
    import torch.distributed as tdist
    if world > 1:
        tdist.barrier()
    from paper_2509_23866_b200 import dart, synth
    from paper_2509_23866_b200 import dist as D
    from paper_2509_23866_b200.stream import StreamedPass
    dev = torch.device("cuda", torch.cuda.current_device())
    layout, V, dtype, _ = synth.config_layout(args.config, seed=args.seed)
    cfg = dart.Config(entropy_q=args.q, beta_kl=args.beta, zero_fill_masked=0 if args.compact else 1,
                      select_rule=dart.SEL_OFF if args.q <= 0 else dart.SEL_FLOOR)
    group = tdist.group.WORLD if world > 1 else None
    shards = D.shard_layout(layout, world)
    me = shards[rank]
    sp = StreamedPass(layout, V, cfg, dev, max_rows=args.stream_rows, pool=args.pool, logits_dtype=dtype,
                      group=group, world_shards=shards)
    P = sp.P
    # synthetic rows for the P pool slots (P x rows tokens, the config's value
    # recipe); chunk c row r reads slot (c mod P) row r in both sweeps
    rows = sp.rows
    nstep = -(-P * rows // 64)
    sub = synth.Layout(G=1, traj_group=np.zeros(1, np.int32), traj_reward=np.ones(1, np.float32),
                       traj_step_off=np.array([0, nstep], np.int64),
                       step_tok_off=np.minimum(np.arange(nstep + 1, dtype=np.int64) * 64, P * rows),
                       step_fork=np.random.default_rng(args.seed).random(nstep) < 0.3)
    t0 = time.time()
    sb = synth.make_batch(args.config, seed=args.seed * 1000 + rank, device=dev, layout=sub, V=V, dtype=dtype)
    for k in range(P):
        sp.pool_logits[k].copy_(sb.logits[k * rows:(k + 1) * rows])
    T = layout.T
    idx = torch.empty(me.T_loc, dtype=torch.int64, device=dev)
    for i, c in enumerate(sp.chunks):
        base = (i % P) * rows
        idx[c.tok_begin - me.tok_begin:c.tok_end - me.tok_begin] = torch.arange(base, base + c.T_loc, device=dev)
    target, lo, lr, lref = (x[idx].contiguous() for x in (sb.target, sb.logp_old, sb.logp_rollout, sb.logp_ref))
    del sb
    torch.cuda.synchronize()
    log(f"[rank {rank}] streamed {args.config}: T={T} (local {me.T_loc}) in {len(sp.chunks)} chunks of "
        f"<= {sp.rows} rows, pool {P}; setup {time.time() - t0:.1f}s")
    for _ in range(args.warmup):
        sp.run(target, lo, lr, lref)
    torch.cuda.synchronize()
    sp.status.zero_()
    sp.launches = 0
    if world > 1:
        tdist.barrier()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.15)
    s0 = torch.cuda.Event(enable_timing=True)
    s1 = torch.cuda.Event(enable_timing=True)
    s0.record(stream)
    for _ in range(args.steps):
        sp.run(target, lo, lr, lref)
    s1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        tdist.barrier()
    clocks = clk.stop()
    sp.check_status()
    ms_loc = s0.elapsed_time(s1) / args.steps
    ms = ms_loc
    if world > 1:
        t = torch.tensor([ms_loc, -ms_loc], dtype=torch.float64, device=dev)
        D.all_reduce(t, op=tdist.ReduceOp.MAX)
        ms, ms_min = float(t[0].item()), -float(t[1].item())
    keep = sp.keep.cpu().numpy()[:layout.S].astype(bool)
    n = np.diff(layout.step_tok_off)
    kept_loc = int(n[me.step_begin:me.step_end][keep[me.step_begin:me.step_end]].sum())
    kept = int(n[keep].sum())
    es = 2
    byts = me.T_loc * (es * V + 24) + kept_loc * 2 * es * V + (0 if args.compact else (me.T_loc - kept_loc) * es * V)
    peak, src = hbm_peak()
    gbs = byts / (ms * 1e-3) / 1e9
    if rank == 0:
        line = {"metric": METRIC,
                "value": T / (ms * 1e-3), "unit": "logit-tokens/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
                "scaling": "strong" if world > 1 else "weak",
                "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded; pooled chunk logits)",
                "config": {"workload": args.config, "global_tokens": T, "tokens_per_gpu": me.T_loc, "V": V,
                           "groups": layout.G, "steps_total": layout.S, "chunks": len(sp.chunks),
                           "chunk_rows": sp.rows, "pool": P, "kept_token_frac": kept / T, "streamed": True,
                           "l2": "inputs larger than L2 (pooled chunks of %.1f GB)" % (sp.rows * V * es / 1e9),
                           "parallelism": f"dp{world} (trajectory-sharded, global batch split across ranks)"},
                "roofline": {"bound": "hbm", "kernel": "whole step (fwd+select+bwd sweeps), rank 0",
                             "achieved": gbs, "peak": peak, "peak_source": src, "unit": "GB/s", "frac": gbs / peak,
                             "traffic": None},
                "gpu_launches": sp.launches, "clocks": clocks, "e2e": None, "cpu_baseline": None}
        if world > 1:
            line["rank_time_ms"] = {"max": ms, "min": ms_min}
        print(json.dumps(line), flush=True)
    if world > 1:
        tdist.barrier()
        tdist.destroy_process_group()


# ------------------------------------------------------------------ our arm
def run_dart(args):
    from paper_2509_23866_b200 import build as B
    if int(os.environ.get("RANK", "0")) == 0:
        B.build()
    world, rank, local = dist_setup(args)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    from paper_2509_23866_b200 import dart, synth
    dev = torch.device("cuda", torch.cuda.current_device())
    lays, glayout, shards, V, dtype = weak_layouts(args.config, args.seed, world)
    layout_r = lays[rank]
    me = shards[rank]
    cfg = dart.Config(entropy_q=args.q, beta_kl=args.beta, zero_fill_masked=0 if args.compact else 1,
                      select_rule=dart.SEL_OFF if args.q <= 0 else dart.SEL_FLOOR,
                      kl_mode=dart.KL_EXACT if args.kl == "exact" else dart.KL_K3)
    t0 = time.time()
    batch = synth.make_batch(args.config, seed=args.seed * 1000 + rank, device=dev, layout=layout_r, V=V,
                             dtype=dtype, with_ref=args.kl == "exact")
    torch.cuda.synchronize()
    log(f"[rank {rank}] generated {layout_r.T} x {V} {dtype} logits in {time.time() - t0:.1f}s")
    group = None
    if world > 1:
        import torch.distributed as dist
        group = dist.group.WORLD
    dl = dart.DartLoss(glayout, me, V, cfg, dev, logits_dtype=dtype, grad_dtype=torch.bfloat16,
                       group=group, world_shards=shards)
    inputs = (batch.logits, batch.target, batch.logp_old, batch.logp_rollout, batch.logp_ref)
    if args.kl == "exact":
        inputs = inputs + (batch.ref_logits,)

    stream = torch.cuda.current_stream()

    if args.fused:
        # the mask comes from an earlier (untimed)
        # old-policy pass; the timed step is the single-read fused update
        dl.run(*inputs)
        torch.cuda.synchronize()
        keep0, norm0 = dl.keep.clone(), dl.norm.clone()

        def step():
            dl.fused(*inputs, keep=keep0, norm=norm0)
    else:
        def step():
            dl.run(*inputs)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    dl.status.zero_()
    dl.launches = 0
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()

    fwd_ms, bwd_ms = [], []
    ev_pairs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.15)
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    start.record(stream)
    for k in range(args.steps):
        step()
    end.record(stream)
    torch.cuda.synchronize()
    clocks = clk.stop()
    dart.set_timing_events()
    elapsed_ms = start.elapsed_time(end)
    launches = dl.launches
    dl.check_status()

    # per-kernel timing pass (same work; the library records the events on its
    # stream immediately around the two sweep kernels)
    for k in range(args.steps):
        for x in ev_pairs[k]:
            x.record(stream)          # creates the event handles
    torch.cuda.synchronize()
    for k in range(args.steps):
        dart.set_timing_events(*ev_pairs[k])
        step()
    torch.cuda.synchronize()
    dart.set_timing_events()
    for k in range(args.steps):
        e = ev_pairs[k]
        fwd_ms.append(e[0].elapsed_time(e[1]))
        bwd_ms.append(e[2].elapsed_time(e[3]))

    # the same pass replayed from a CUDA graph (one host launch per step): context
    graph = None
    if args.graph and world == 1 and not args.fused:
        g = dl.capture(*inputs)
        for _ in range(args.warmup):
            g.replay()
        torch.cuda.synchronize()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(args.steps):
            g.replay()
        g1.record(stream)
        torch.cuda.synchronize()
        gms = g0.elapsed_time(g1) / args.steps
        graph = {"ms_per_step": gms, "value": layout_r.T / (gms * 1e-3), "what": "DartLoss.capture() replayed"}
        del g

    # per-phase pass (SURVEY §8(d) timing protocol: K0-K2, C1, K3, K4+K5(+K6), C2),
    # events on the launching stream between the public API's phase calls
    phases = None
    if not args.fused:
        names = ["fwd (K0-K2)", "C1 all-gather", "select (K3)", "bwd (K6, K4/K5)", "C2 all-reduce"]
        pev = [[torch.cuda.Event(enable_timing=True) for _ in range(6)] for _ in range(args.steps)]
        acc = {n: [] for n in names}
        for k in range(args.steps):
            ev = pev[k]
            ev[0].record(stream)
            dl.forward(*inputs)
            ev[1].record(stream)
            dl.gather()
            ev[2].record(stream)
            dl.select()
            ev[3].record(stream)
            dl.backward()
            ev[4].record(stream)
            dl.reduce_stats()
            ev[5].record(stream)
        torch.cuda.synchronize()
        for k in range(args.steps):
            for i, n in enumerate(names):
                acc[n].append(pev[k][i].elapsed_time(pev[k][i + 1]))
        phases = {n: round(statistics.median(v), 4) for n, v in acc.items()}

    # context, not the roofline denominator: a plain device copy (torch
    # copy_, the kernel MEASURED_PEAKS.json's hbm_gbs is taken with) timed the
    # same way as the step -- back to back, as long as the timed loop, under
    # the same power-cap conditions -- over buffers of the step's size
    copy_ref = None
    if not args.fused and dl.dlogits is not None and rank == 0 and world == 1 and batch.logits.is_contiguous() \
            and dl.dlogits_store.numel() >= batch.logits.numel() and dl.dlogits_store.dtype == batch.logits.dtype:
        src = batch.logits.view(-1)
        dst = dl.dlogits_store.view(-1)[:src.numel()]
        n_copy = max(3, int(round(elapsed_ms / max(1e-3, 2.0 * src.numel() * src.element_size() / 6.0e9))))
        for _ in range(3):
            dst.copy_(src)
        torch.cuda.synchronize()
        clk2 = ClockSampler(local)
        clk2.start()
        time.sleep(0.15)
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0.record(stream)
        for _ in range(n_copy):
            dst.copy_(src)
        c1.record(stream)
        torch.cuda.synchronize()
        cclk = clk2.stop()
        cms = c0.elapsed_time(c1) / n_copy
        copy_ref = {"what": "torch copy_ of the logits buffer into dlogits, back to back for the timed loop's duration",
                    "bytes": 2 * src.numel() * src.element_size(), "launches": n_copy, "avg_ms": cms,
                    "GBps": 2 * src.numel() * src.element_size() / (cms * 1e-3) / 1e9, "clocks": cclk}

    ms = elapsed_ms / args.steps
    rank_ms = None
    if world > 1:
        import torch.distributed as dist
        from paper_2509_23866_b200 import dist as D
        t = torch.tensor([ms, -ms], dtype=torch.float64, device=dev)
        D.all_reduce(t, op=dist.ReduceOp.MAX)
        tm = torch.tensor([ms], dtype=torch.float64, device=dev)
        D.all_reduce(tm)
        rank_ms = {"max": float(t[0].item()), "min": -float(t[1].item()), "mean": float(tm.item()) / world,
                   "what": "per-rank device time of the timed loop / steps (SURVEY §8(d): max/mean rank time)"}
        ms = rank_ms["max"]
    T_tot = glayout.T
    value = T_tot / (ms * 1e-3)

    # algorithmic bytes: fwd 2V per row (+ 24 B of per-token
    # I/O); bwd 4V per kept row (2V read + 2V write), 2V per masked row
    # (write only; 0 with --compact)
    keep = dl.keep.cpu().numpy()
    n = np.diff(glayout.step_tok_off)
    kept_tok_loc = int(n[me.step_begin:me.step_end][keep[me.step_begin:me.step_end].astype(bool)].sum())
    masked_tok_loc = me.T_loc - kept_tok_loc
    es = 2
    fwd_bytes = me.T_loc * (es * V + 24)
    bwd_bytes = kept_tok_loc * (2 * es * V) + (0 if args.compact else masked_tok_loc * es * V)
    if args.kl == "exact":   # both sweeps also stream the reference logits
        fwd_bytes = me.T_loc * (2 * es * V + 24)
        bwd_bytes = kept_tok_loc * (3 * es * V) + (0 if args.compact else masked_tok_loc * es * V)
    if args.fused:   # one kernel: kept rows read once + written once, masked rows written
        fwd_bytes = 0
        bwd_bytes = kept_tok_loc * (2 * es * V + 24) + (0 if args.compact else masked_tok_loc * es * V)
    fwd_avg, bwd_avg = statistics.mean(fwd_ms), statistics.mean(bwd_ms)
    if args.fused:
        fwd_avg = 1e-9
    peak, peak_src = hbm_peak()
    fwd_gbs = fwd_bytes / (fwd_avg * 1e-3) / 1e9
    bwd_gbs = bwd_bytes / (bwd_avg * 1e-3) / 1e9
    dom = ("bwd_sweep", bwd_gbs, bwd_bytes, bwd_avg) if bwd_avg >= fwd_avg else ("fwd_sweep", fwd_gbs, fwd_bytes, fwd_avg)
    if args.fused:
        dom = ("fused_sweep",) + dom[1:]
    step_bytes = fwd_bytes + bwd_bytes
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            with open(tpath) as f:
                tj = json.load(f)
            key = dom[0]
            if args.kl == "exact" and not args.fused:      # the exact-KL sweeps have their own captures
                key = {"fwd_sweep": "fwd_kl", "bwd_sweep": "bwd_kl"}.get(key, key)
            traffic = tj.get(key, {}).get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    # ---- e2e through the public API with host buffers (pinned), rank-local
    e2e = None
    if not args.no_e2e:
        ok, why = e2e_host_memory_ok(inputs, world)
        e2e = run_e2e(args, dl, batch, stream, world, inputs) if ok else {"skipped": why}

    # ---- CPU oracle baseline (rank 0, N == 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(args, batch, cfg)

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": value, "unit": "logit-tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded; DESIGN.md §5 recipe)",
            "config": {"workload": args.config + (" (fused update, mask known in advance: NEXT #1)" if args.fused else "")
                       + (" (exact full-vocabulary KL from reference logits: NEXT #4)" if args.kl == "exact" else ""),
                       "desc": CONFIG_DESC.get(args.config, args.config),
                       "global_tokens": T_tot, "tokens_per_gpu": me.T_loc, "V": V,
                       "groups": glayout.G, "steps_total": glayout.S, "entropy_q": args.q, "beta_kl": args.beta,
                       "is_cap": cfg.is_cap, "dlogits": "compact" if args.compact else "dense (masked rows zero)",
                       "kept_token_frac": kept_tok_loc / max(me.T_loc, 1),
                       "l2": "inputs larger than L2 (%.1f GB logits + %.1f GB dlogits per GPU >> 126 MB)" % (
                           me.T_loc * V * es / 1e9, me.T_loc * V * es / 1e9),
                       "parallelism": f"dp{world} (trajectory-sharded)"},
            "roofline": {"bound": "hbm", "kernel": dom[0], "achieved": dom[1], "peak": peak,
                         "peak_source": peak_src, "unit": "GB/s", "frac": dom[1] / peak,
                         "traffic": traffic,
                         "traffic_source": ("prior ncu --set full capture of this kernel at this config "
                                            "(profiles/ncu_traffic.json, not measured in this run)") if traffic else None,
                         "algorithmic_bytes_per_launch": dom[2],
                         "avg_launch_ms": dom[3]},
            "kernels": {"fwd_sweep": {"avg_ms": fwd_avg, "median_ms": statistics.median(fwd_ms) if not args.fused else None,
                                      "best_ms": min(fwd_ms) if not args.fused else None,
                                      "GBps": fwd_gbs, "frac": fwd_gbs / peak, "bytes": fwd_bytes},
                        "bwd_sweep": {"avg_ms": bwd_avg, "median_ms": statistics.median(bwd_ms), "best_ms": min(bwd_ms),
                                      "GBps": bwd_gbs, "frac": bwd_gbs / peak, "bytes": bwd_bytes},
                        "step_GBps": step_bytes / (ms * 1e-3) / 1e9,
                        "step_frac": step_bytes / (ms * 1e-3) / 1e9 / peak,
                        "step_frac_of_8TBps_spec": step_bytes / (ms * 1e-3) / 1e9 / 8000.0,
                        "phases_median_ms": phases},
            "gpu_launches": launches,
            "clocks": clocks,
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        if rank_ms is not None:
            line["rank_ms"] = rank_ms
        if copy_ref is not None:
            copy_ref["step_frac_vs_copy"] = line["kernels"]["step_GBps"] / copy_ref["GBps"]
            line["copy_sustained"] = copy_ref
        if graph is not None:
            line["cuda_graph"] = graph
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


def tensor_peak():
    try:
        with open(PEAKS_PATH) as f:
            j = json.load(f)
        return float(j["bf16_tflops_sustained"]), float(j["bf16_tflops"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 2250.0, 2250.0, "fallback (B200_PROFILING.md nominal dense bf16)"


def run_lmhead(args):
    """the old-log-prob pass with the LM head fused in.
    One step = dart_lmhead_fwd (z = h W^T on tcgen05 + log-softmax / entropy /
    target log-prob in the epilogue, per-step entropies) + select, over the
    config's tokens; the [T, V] logits never exist.  Timed beside it: the
    unfused pipeline (cuBLAS bf16 GEMM writing the logits, then the same
    forward + select over them)."""
    from paper_2509_23866_b200 import build as B
    if int(os.environ.get("RANK", "0")) == 0:
        B.build()
    world, rank, local = dist_setup(args)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    from paper_2509_23866_b200 import dart, synth
    dev = torch.device("cuda", torch.cuda.current_device())
    lays, glayout, shards, V, _ = weak_layouts(args.config, args.seed, world)
    layout_r = lays[rank]
    me = shards[rank]
    d = args.hidden
    cfg = dart.Config(entropy_q=args.q, beta_kl=args.beta)
    t0 = time.time()
    lb = synth.make_lmhead(None, d, seed=args.seed * 1000 + rank, device=dev, layout=layout_r, V=V)
    torch.cuda.synchronize()
    log(f"[rank {rank}] generated hidden {layout_r.T} x {d} and W {V} x {d} in {time.time() - t0:.1f}s")
    group = dist.group.WORLD if world > 1 else None
    dl = dart.DartLoss(glayout, me, V, cfg, dev, group=group, world_shards=shards, with_grad=False)
    b = lb.batch
    inputs = (lb.hidden, lb.weight, b.target, b.logp_old, b.logp_rollout, b.logp_ref)
    stream = torch.cuda.current_stream()

    def step():
        dl.forward_lmhead(*inputs)
        dl.gather()
        dl.select()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    dl.status.zero_()
    dl.launches = 0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.15)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record(stream)
    for _ in range(args.steps):
        step()
    end.record(stream)
    torch.cuda.synchronize()
    clocks = clk.stop()
    elapsed_ms = start.elapsed_time(end)
    launches = dl.launches
    dl.check_status()
    # kernel timing pass: events recorded by the library around the tcgen05 kernel
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    for e in ev:
        for x in e:
            x.record(stream)
    torch.cuda.synchronize()
    for k in range(args.steps):
        dart.set_timing_events(*ev[k])
        step()
    torch.cuda.synchronize()
    dart.set_timing_events()
    gemm_ms = statistics.mean(e[0].elapsed_time(e[1]) for e in ev)
    ms = elapsed_ms / args.steps
    if world > 1:
        from paper_2509_23866_b200 import dist as D
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        D.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = glayout.T / (ms * 1e-3)
    flops = 2.0 * me.T_loc * d * V
    peak_s, peak_b, peak_src = tensor_peak()
    achieved = flops / (gemm_ms * 1e-3) / 1e12
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            traffic = json.load(f).get("lmhead_fwd", {}).get("dram_bytes_per_launch")
    except Exception:
        traffic = None

    # ---- the unfused pipeline, timed beside it (cuBLAS GEMM -> bf16 logits -> same fwd + select)
    unfused = None
    if not args.no_unfused and rank == 0:
        try:
            logits = torch.empty((me.T_loc, V), dtype=torch.bfloat16, device=dev)
            # this rank's own batch as a one-rank problem: the same rows and work
            dl2 = dart.DartLoss(layout_r, dart.whole_shard(layout_r), V, cfg, dev, with_grad=False)
            k = max(3, min(args.steps, 10))

            def ustep():
                torch.matmul(lb.hidden, lb.weight.T, out=logits)
                dl2.forward(logits, b.target, b.logp_old, b.logp_rollout, b.logp_ref)
                dl2.select()
            for _ in range(2):
                ustep()
            torch.cuda.synchronize()
            s1, s2, s3 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            g_ms = []
            s1.record(stream)
            for _ in range(k):
                ustep()
            s2.record(stream)
            torch.cuda.synchronize()
            for _ in range(k):
                a, c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                torch.matmul(lb.hidden, lb.weight.T, out=logits)
                c.record(stream)
                c.synchronize()
                g_ms.append(a.elapsed_time(c))
            u_ms = s1.elapsed_time(s2) / k
            cub = statistics.mean(g_ms)
            unfused = {"ms_per_step": u_ms, "tokens_per_s": me.T_loc / (u_ms * 1e-3), "cublas_gemm_ms": cub,
                       "cublas_tflops": flops / (cub * 1e-3) / 1e12,
                       "logits_bytes": me.T_loc * V * 2, "steps": k}
            del logits, dl2
            torch.cuda.empty_cache()
        except torch.OutOfMemoryError:
            unfused = {"skipped": "out of memory for the [T, V] bf16 logits"}

    # ---- e2e: hidden states + per-token inputs from pinned host memory each step, step entropies back
    e2e = None
    if not args.no_e2e:
        host = [t.cpu().pin_memory() for t in (lb.hidden, b.target, b.logp_old, b.logp_rollout, b.logp_ref)]
        dbuf = [torch.empty_like(t, device=dev) for t in host]
        out_h = torch.empty(me.S_loc, dtype=torch.float32).pin_memory()
        h2d = sum(t.numel() * t.element_size() for t in host)

        def one():
            for x, hh in zip(dbuf, host):
                x.copy_(hh, non_blocking=True)
            dl.forward_lmhead(dbuf[0], lb.weight, *dbuf[1:])
            dl.gather()
            dl.select()
            out_h.copy_(dl.step_H[:me.S_loc], non_blocking=True)
        one()
        torch.cuda.synchronize()
        n = max(1, min(args.steps, args.e2e_steps))
        a, c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(n):
            one()
        c.record(stream)
        torch.cuda.synchronize()
        ems = a.elapsed_time(c) / n
        if world > 1:
            from paper_2509_23866_b200 import dist as D
            t = torch.tensor([ems], dtype=torch.float64, device=dev)
            D.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        e2e = {"value": glayout.T / (ems * 1e-3), "unit": "tokens/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": out_h.numel() * 4, "steps": n, "ms_per_step": ems,
               "note": "weight stays resident (model parameter); hidden states and per-token inputs copied"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = lmhead_cpu_baseline(args, lb, cfg)

    if rank == 0:
        line = {
            "metric": "LM-head-fused old-log-prob pass tokens/s (h W^T + log-softmax + entropy + select), "
                      "V=152064, d=%d" % d,
            "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "bf16", "data": "synthetic (seeded; synth.make_lmhead recipe, DESIGN.md §9)",
            "config": {"workload": args.config + " (LM-head-fused forward: NEXT #3)",
                       "desc": CONFIG_DESC.get(args.config, args.config), "global_tokens": glayout.T,
                       "tokens_per_gpu": me.T_loc, "V": V, "d": d,
                       "l2": "inputs larger than L2 (W %.2f GB + hidden %.2f GB >> 126 MB)" % (
                           V * d * 2 / 1e9, me.T_loc * d * 2 / 1e9),
                       "parallelism": f"dp{world} (trajectory-sharded)"},
            "roofline": {"bound": "tensor", "kernel": "lmhead_fwd_kernel", "achieved": achieved, "peak": peak_s,
                         "peak_source": peak_src + " bf16_tflops_sustained (kernel inside a long step loop)",
                         "unit": "TFLOP/s", "frac": achieved / peak_s, "frac_of_burst_peak": achieved / peak_b,
                         "traffic": traffic, "traffic_unit": "DRAM bytes per launch (ncu); the tensor-bound kernel's operand re-reads hit L2 95%",
                         "traffic_source": "prior ncu capture (profiles/ncu_traffic.json)" if traffic else None,
                         "algorithmic_flops_per_launch": flops, "avg_launch_ms": gemm_ms},
            "unfused_cublas_pipeline": unfused,
            "gpu_launches": launches,
            "clocks": clocks,
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_lmhead_update(args):
    """SURVEY §8(f) NEXT #3, training half: the update pass through the LM
    head with the mask from the (untimed) old-log-prob pass.  One step =
    LmHeadUpdate.run: dart_lmhead_fwd at theta (tcgen05 z + softmax epilogue)
    -> dart_lmhead_bwd (kept rows gathered, z recomputed on tcgen05, bf16 dz
    from the TMEM epilogue) -> dh = dz W, dW = dz^T h_kept (cuBLAS, kept rows
    only).  Timed beside it, in the same process:
      * the cuBLAS pipeline with the [T, V] logits materialised: torch.matmul
        bf16 logits -> dart_loss_fused (dz) -> cuBLAS dh, dW over all rows;
      * the whole LM-head training step at theta = theta_old (one update per
        batch): ours = forward_lmhead + select + backward_lmhead +
        the two GEMMs on ONE DartLoss; materialised = cuBLAS logits +
        DartLoss.run (fwd + select + bwd sweeps) + cuBLAS dh, dW."""
    from paper_2509_23866_b200 import build as B
    B.build()
    world, rank, local = dist_setup(args)
    if world > 1:
        raise SystemExit("--lmhead --update is single-GPU")
    from paper_2509_23866_b200 import dart, lmhead, synth
    dev = torch.device("cuda", torch.cuda.current_device())
    layout, V, _, _ = synth.config_layout(args.config, seed=args.seed)
    d = args.hidden
    cfg = dart.Config(entropy_q=args.q, beta_kl=args.beta)
    lb = synth.make_lmhead(None, d, seed=args.seed * 1000, device=dev, layout=layout, V=V)
    b = lb.batch
    T = layout.T
    old = dart.DartLoss(layout, dart.whole_shard(layout), V, cfg, dev, with_grad=False)
    old.forward_lmhead(lb.hidden, lb.weight, b.target, b.logp_old, b.logp_rollout, b.logp_ref)
    old.select()
    torch.cuda.synchronize()
    keep, norm = old.keep.clone(), old.norm.clone()
    up = lmhead.LmHeadUpdate(layout, V, d, cfg, dev, chunk_rows=args.chunk_rows or None)
    dh = torch.empty((T, d), dtype=torch.float32, device=dev)
    dW = torch.empty((V, d), dtype=torch.float32, device=dev)
    args_in = (lb.hidden, lb.weight, b.target, b.logp_old, b.logp_rollout, b.logp_ref, keep, norm)
    stream = torch.cuda.current_stream()

    def step():
        up.run(*args_in, dh=dh, dW=dW)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    up.status.zero_()
    up.launches = 0
    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.15)
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record(stream)
    for _ in range(args.steps):
        step()
    s1.record(stream)
    torch.cuda.synchronize()
    clocks = clk.stop()
    up.check_status()
    ms = s0.elapsed_time(s1) / args.steps
    launches = up.launches // args.steps
    K = up.last_n_kept
    # per-kernel pass: events around the tcgen05 forward (dart_lmhead_fwd) and dz (dart_lmhead_bwd) kernels
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    for e in ev:
        for x in e:
            x.record(stream)
    torch.cuda.synchronize()
    for k in range(args.steps):
        dart.set_timing_events(*ev[k])
        step()
    torch.cuda.synchronize()
    dart.set_timing_events()
    fwd_ms = statistics.mean(e[0].elapsed_time(e[1]) for e in ev)
    dz_ms = statistics.mean(e[2].elapsed_time(e[3]) for e in ev)
    peak_s, peak_b, peak_src = tensor_peak()
    f_fwd, f_dz = 2.0 * T * d * V, 2.0 * K * d * V
    flops = f_fwd + 3 * f_dz          # forward + dz recompute + dh + dW
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            traffic = json.load(f).get("lmhead_dz", {}).get("dram_bytes_per_launch")
    except Exception:
        traffic = None

    # ---- theta = theta_old: the whole LM-head training step on one DartLoss (old pass = update forward)
    full = dart.DartLoss(layout, dart.whole_shard(layout), V, cfg, dev, with_grad=False)

    def whole_step():
        full.forward_lmhead(lb.hidden, lb.weight, b.target, b.logp_old, b.logp_rollout, b.logp_ref)
        full.select()
        full.backward_lmhead(up.dz, up.h_kept, up.kept_rows, up.n_kept)
        dh.zero_()
        lmhead.backward_grads(up.dz, up.h_kept, up.kept_rows, up.n_kept, lb.weight, dh, dW)
    for _ in range(2):
        whole_step()
    torch.cuda.synchronize()
    kk = max(3, min(args.steps, 5))
    a, c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(kk):
        whole_step()
    c.record(stream)
    torch.cuda.synchronize()
    whole_ms = a.elapsed_time(c) / kk
    full.check_status()
    del full
    torch.cuda.empty_cache()

    unfused = None
    if not args.no_unfused:
        try:
            logits = torch.empty((T, V), dtype=torch.bfloat16, device=dev)
            dl2 = dart.DartLoss(layout, dart.whole_shard(layout), V, cfg, dev)
            dh2 = torch.empty((T, d), dtype=torch.bfloat16, device=dev)
            dW2 = torch.empty((V, d), dtype=torch.bfloat16, device=dev)

            def ustep():
                torch.matmul(lb.hidden, lb.weight.T, out=logits)
                g = dl2.fused(logits, b.target, b.logp_old, b.logp_rollout, b.logp_ref, keep=keep, norm=norm)
                torch.matmul(g, lb.weight, out=dh2)
                torch.matmul(g.T, lb.hidden, out=dW2)

            def uwhole():
                torch.matmul(lb.hidden, lb.weight.T, out=logits)
                g = dl2.run(logits, b.target, b.logp_old, b.logp_rollout, b.logp_ref)
                torch.matmul(g, lb.weight, out=dh2)
                torch.matmul(g.T, lb.hidden, out=dW2)
            res = {}
            for name, fn in (("update", ustep), ("whole", uwhole)):
                for _ in range(2):
                    fn()
                torch.cuda.synchronize()
                a, c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                for _ in range(kk):
                    fn()
                c.record(stream)
                torch.cuda.synchronize()
                res[name] = a.elapsed_time(c) / kk
            unfused = {"ms_per_step": res["update"], "tokens_per_s": T / (res["update"] * 1e-3),
                       "whole_step_ms": res["whole"], "hbm_bytes_materialised": 2 * T * V * 2, "steps": kk,
                       "what": "update: torch.matmul (cuBLAS) bf16 logits [T, V] -> dart_loss_fused -> cuBLAS dh, dW; "
                               "whole: cuBLAS logits -> DartLoss.run (fwd + select + bwd) -> cuBLAS dh, dW"}
            del logits, dl2, dh2, dW2
            torch.cuda.empty_cache()
        except torch.OutOfMemoryError:
            unfused = {"skipped": "out of memory for the [T, V] logits + gradient"}

    line = {
        "metric": "LM-head update pass tokens/s (forward at theta, dz from the z-GEMM epilogue, dh = dz W, "
                  "dW = dz^T h), V=152064, d=%d" % d,
        "value": T / (ms * 1e-3), "unit": "tokens/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded; synth.make_lmhead recipe, DESIGN.md §9)",
        "config": {"workload": args.config + " (LM-head update pass: NEXT #3 training half)",
                   "tokens": T, "kept_rows": K, "V": V, "d": d, "chunks": len(up.chunks),
                   "kept_token_frac": float(up.stats_dict()["n_kept_tok"]) / T,
                   "l2": "inputs larger than L2 (W %.2f GB, hidden %.2f GB, dz %.2f GB)" % (
                       V * d * 2 / 1e9, T * d * 2 / 1e9, K * V * 2 / 1e9),
                   "parallelism": "dp1"},
        "roofline": {"bound": "tensor", "kernel": "lmhead_kernel<DZ> (z recompute + dz epilogue, kept rows)",
                     "achieved": f_dz / (dz_ms * 1e-3) / 1e12, "peak": peak_s,
                     "peak_source": peak_src + " bf16_tflops_sustained (kernel inside a long step loop)",
                     "unit": "TFLOP/s", "frac": f_dz / (dz_ms * 1e-3) / 1e12 / peak_s, "traffic": traffic,
                     "traffic_source": "prior ncu capture (profiles/ncu_traffic.json)" if traffic else None,
                     "algorithmic_flops_per_launch": f_dz, "avg_launch_ms": dz_ms},
        "kernels": {"lmhead_fwd_ms": fwd_ms, "lmhead_fwd_tflops": f_fwd / (fwd_ms * 1e-3) / 1e12,
                    "lmhead_dz_ms": dz_ms, "step_tflops": flops / (ms * 1e-3) / 1e12,
                    "cublas_dh_dW_ms": ms - fwd_ms - dz_ms},
        "theta_old_whole_step": {"ms": whole_ms, "what": "forward_lmhead + select + backward_lmhead + dh, dW "
                                                         "(one object: the old pass's forward is the update's)"},
        "unfused_cublas_pipeline": unfused,
        "gpu_launches": launches,
        "clocks": clocks,
        "e2e": None,
        "cpu_baseline": None,
    }
    print(json.dumps(line), flush=True)


def lmhead_cpu_baseline(args, lb, cfg, rows=64):
    """The oracle (float64 NumPy, BLAS limited to one thread) on the first
    `rows` tokens: LM-head logits + log-softmax / entropy per token."""
    from oracle import dart_oracle as O
    try:
        from threadpoolctl import threadpool_limits
    except Exception:
        threadpool_limits = None
    h = lb.hidden[:rows].float().cpu().numpy()
    W = lb.weight.float().cpu().numpy()
    y = lb.batch.target[:rows].cpu().numpy()
    invT = cfg.as_f32()["inv_temperature"]

    def work():
        z = O.lmhead_logits(h, W)
        for t in range(rows):
            O.token_row(z[t], int(y[t]), invT)
    t0 = time.time()
    if threadpool_limits is not None:
        with threadpool_limits(limits=1):
            work()
    else:
        work()
    dt = time.time() - t0
    return {"value": rows / dt, "unit": "tokens/s", "cores": 1, "cpu_model": cpu_model(), "kind": "oracle",
            "sample": f"{rows} tokens: float64 h W^T (d={h.shape[1]}, V={W.shape[0]}) + per-token log-softmax / "
                      f"entropy, NumPy with BLAS limited to 1 thread", "seconds": dt}


def e2e_host_memory_ok(inputs, world):
    """The e2e leg pins every rank's step inputs in host memory (18.7 GB per
    rank at the single config).  Run it only if all ranks of this host fit in
    70% of the available host memory -- the same decision on every rank (a
    MIN all-reduce), so no rank waits in a collective another one skipped."""
    need = sum(t.numel() * t.element_size() for t in inputs)
    local = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:
        avail = None
    ok = avail is None or need * local <= 0.7 * avail
    if world > 1:
        import torch.distributed as dist
        from paper_2509_23866_b200 import dist as D
        t = torch.tensor([1 if ok else 0], dtype=torch.int32, device=inputs[0].device)
        D.all_reduce(t, op=dist.ReduceOp.MIN)
        ok = bool(t.item())
    why = None if ok else (f"host memory: {local} ranks x {need / 1e9:.1f} GB pinned inputs > 70% of "
                           f"{(avail or 0) / 1e9:.0f} GB available")
    return ok, why


def run_e2e(args, dl, batch, stream, world, inputs):
    """Same pass through the public API with the step's inputs copied from
    pinned host memory each step and the loss read back to the host."""
    from paper_2509_23866_b200 import dart  # noqa: F401
    host = []
    for t in inputs:           # straight into pinned memory (no pageable staging copy)
        h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        h.copy_(t)
        host.append(h)
    dev_bufs = [torch.empty_like(t, device=batch.logits.device) for t in host]
    loss_h = torch.empty(len(dl.stats), dtype=torch.float64).pin_memory()
    h2d = sum(t.numel() * t.element_size() for t in host)
    d2h = loss_h.numel() * loss_h.element_size()
    steps = max(1, min(args.steps, args.e2e_steps))

    def one():
        for d, h in zip(dev_bufs, host):
            d.copy_(h, non_blocking=True)
        dl.run(*dev_bufs)
        loss_h.copy_(dl.stats, non_blocking=True)

    one()
    torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    s.record(stream)
    for _ in range(steps):
        one()
    e.record(stream)
    torch.cuda.synchronize()
    _ = float(loss_h[0])
    ms = s.elapsed_time(e) / steps
    if world > 1:
        import torch.distributed as dist
        from paper_2509_23866_b200 import dist as D
        t = torch.tensor([ms], dtype=torch.float64, device=batch.logits.device)
        D.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = dl.layout.T / (ms * 1e-3)
    del host, dev_bufs
    return {"value": value, "unit": "logit-tokens/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "steps": steps, "ms_per_step": ms,
            "d2h_what": "the step's loss + statistics (dart_stats, 11 float64); dlogits stay in HBM for the "
                        "model's backward (a trainer never copies them to the host)"}


# ------------------------------------------------------------------ oracle arms
def oracle_sample(batch, n_traj=None, max_tokens=1024, group=0):
    """A bounded sample of the workload: task group `group`'s first
    trajectories, truncated to whole steps totalling <= max_tokens tokens."""
    from paper_2509_23866_b200 import synth
    L = batch.layout
    steps, toks = 0, 0
    tso, sto = L.traj_step_off, L.step_tok_off
    lens = []
    i0 = int(np.searchsorted(L.traj_group, group, side="left"))
    i = i0
    while i < L.N_traj and L.traj_group[i] == L.traj_group[i0]:
        li = 0
        for s in range(tso[i], tso[i + 1]):
            ns = int(sto[s + 1] - sto[s])
            if toks + ns > max_tokens:
                break
            li += 1
            toks += ns
        if li == 0:
            break
        lens.append(li)
        i += 1
    # rebuild a 1-group layout with these trajectory lengths (rows taken in order)
    rows = []
    tso2, sto2 = [0], [0]
    for j, li in enumerate(lens):
        for s in range(tso[i0 + j], tso[i0 + j] + li):
            rows.extend(range(int(sto[s]), int(sto[s + 1])))
            sto2.append(sto2[-1] + int(sto[s + 1] - sto[s]))
        tso2.append(tso2[-1] + li)
    lay = synth.Layout(G=1, traj_group=np.zeros(len(lens), np.int32), traj_reward=L.traj_reward[i0:i0 + len(lens)],
                       traj_step_off=np.asarray(tso2, np.int64), step_tok_off=np.asarray(sto2, np.int64),
                       step_fork=np.zeros(len(sto2) - 1, bool))
    rows_t = torch.as_tensor(rows, device=batch.logits.device)
    d = dict(G=1, traj_group=lay.traj_group, traj_reward=lay.traj_reward.astype(np.float64),
             traj_step_off=lay.traj_step_off, step_tok_off=lay.step_tok_off,
             target=batch.target[rows_t].cpu().numpy().astype(np.int64),
             logp_old=batch.logp_old[rows_t].cpu().numpy().astype(np.float64),
             logp_rollout=batch.logp_rollout[rows_t].cpu().numpy().astype(np.float64),
             logp_ref=batch.logp_ref[rows_t].cpu().numpy().astype(np.float64),
             logits=batch.logits[rows_t].float().cpu().numpy())
    if batch.ref_logits is not None:        # exact-KL workload: the reference policy's logits too
        d["ref_logits"] = batch.ref_logits[rows_t].float().cpu().numpy()
    return d, len(rows), len(lens), len(sto2) - 1


# ---- the oracle on the host cores: the unmodified oracle, one independent
# bounded sample per worker process (fork: the samples are inherited, never
# pickled), wall time over all of them.  SURVEY §8(d): "parallelised over
# token rows with multiprocessing across all host cores".
_ORACLE_JOBS = None


def _oracle_job(i):
    from oracle import dart_oracle as O
    d, cfg = _ORACLE_JOBS[i]
    O.loss_pass(d, cfg)
    return i


def oracle_procs(sample_bytes):
    """Worker count: the host's usable cores, bounded by ~3x the sample's
    bytes of free memory per worker (the oracle holds float64 rows)."""
    try:
        cores = len(os.sched_getaffinity(0))
    except Exception:
        cores = os.cpu_count() or 1
    try:
        import psutil
        avail = psutil.virtual_memory().available
        cores = min(cores, max(1, int(0.6 * avail // max(1, 3 * sample_bytes))))
    except Exception:
        pass
    return max(1, min(cores, 64))


class OraclePool:
    def __init__(self, samples, cfg, procs):
        global _ORACLE_JOBS
        import multiprocessing as mp
        self.n = len(samples)
        _ORACLE_JOBS = [(d, cfg) for d in samples]
        for v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
            os.environ[v] = "1"
        self.procs = procs
        self.pool = mp.get_context("fork").Pool(procs) if procs > 1 else None

    def run(self):
        """One pass over every sample; returns wall seconds."""
        t0 = time.perf_counter()
        if self.pool is None:
            for i in range(self.n):
                _oracle_job(i)
        else:
            self.pool.map(_oracle_job, range(self.n), chunksize=1)
        return time.perf_counter() - t0

    def close(self):
        if self.pool is not None:
            self.pool.close()
            self.pool.join()


def oracle_samples(batch, per_sample_tokens, n):
    """n samples (task groups 0, 1, ... cycled), whole steps, <= per_sample_tokens each."""
    G = int(batch.layout.G)
    out, ntok = [], 0
    for i in range(n):
        d, nt, _, _ = oracle_sample(batch, max_tokens=per_sample_tokens, group=i % G)
        out.append(d)
        ntok += nt
    return out, ntok


def cpu_model():
    """The host CPU's model name (lscpu / /proc/cpuinfo), for the cpu_baseline record."""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    try:
        import subprocess
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def cpu_baseline(args, batch, cfg):
    per = args.cpu_tokens
    procs = oracle_procs(per * batch.V * 4) if args.cpu_procs <= 0 else args.cpu_procs
    samples, ntok = oracle_samples(batch, per, procs)
    pool = OraclePool(samples, cfg.as_f32(), procs)
    # bounded CPU work of about args.cpu_seconds: the concurrent samples are
    # re-run until that much wall time has passed (at most 8 rounds)
    dt, rounds = 0.0, 0
    try:
        while rounds < 8 and (rounds == 0 or dt < args.cpu_seconds):
            dt += pool.run()
            rounds += 1
    finally:
        pool.close()
    return {"value": ntok * rounds / dt, "unit": "logit-tokens/s", "cores": procs, "cpu_model": cpu_model(),
            "host_cores": os.cpu_count(), "kind": "oracle",
            "sample": f"{procs} independent samples run concurrently, one per process, each <= {per} tokens "
                      f"of whole steps of one task group (groups cycled; {ntok} tokens per round, V={batch.V}), "
                      f"{rounds} rounds; full fwd+select+bwd incl. dlogits, float64 NumPy, one thread per process",
            "seconds": dt, "rounds": rounds}


def run_reference(args):
    """--impl reference: the float64 CPU oracle on the same config, each step a
    bounded sample of the workload."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import dart_oracle as O
    from paper_2509_23866_b200 import dart, synth
    layout_r, V, dtype, _ = synth.config_layout(args.config, seed=args.seed)
    # generate only the sample's rows on the CPU (identical recipe)
    exact = args.kl == "exact"
    batch = synth.make_batch(args.config, seed=args.seed * 1000, device="cpu", layout=_first_traj_layout(layout_r),
                             V=V, dtype=dtype, with_ref=exact)
    cfg = dart.Config(entropy_q=args.q, beta_kl=args.beta, kl_mode=dart.KL_EXACT if exact else dart.KL_K3)
    d, ntok1, ntraj, nstep = oracle_sample(batch, max_tokens=args.cpu_tokens)
    procs = oracle_procs(ntok1 * V * 4) if args.cpu_procs <= 0 else args.cpu_procs
    pool = OraclePool([d] * procs, cfg.as_f32(), procs)      # the same sample on every core
    ntok = ntok1 * procs
    try:
        for _ in range(args.warmup):
            pool.run()
        dt = sum(pool.run() for _ in range(args.steps)) / args.steps
    finally:
        pool.close()
    value = ntok / dt
    line = {"impl": "reference", "metric": METRIC,
            "value": value, "unit": "logit-tokens/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded; DESIGN.md §5 recipe)",
            "config": {"workload": args.config + (" (fused update, mask known in advance: NEXT #1)" if args.fused else "")
                       + (" (exact full-vocabulary KL from reference logits: NEXT #4)" if args.kl == "exact" else ""),
                       "desc": CONFIG_DESC.get(args.config, args.config),
                       "sample_tokens": ntok},
            "cpu_baseline": {"value": value, "unit": "logit-tokens/s", "cores": procs, "cpu_model": cpu_model(),
                             "host_cores": os.cpu_count(), "kind": "oracle",
                             "sample": f"per step: {procs} concurrent runs (one process per core) of one sample of "
                                       f"{ntok1} tokens of {args.config} ({ntraj} trajectories of task 0, whole "
                                       f"steps), float64 NumPy oracle, one thread per process"},
            "e2e": {"value": value, "unit": "logit-tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _first_traj_layout(L):
    """The first task group of layout L (the oracle sample is drawn from it)."""
    from paper_2509_23866_b200 import synth
    nt = int(np.sum(L.traj_group == L.traj_group[0]))
    tso = L.traj_step_off[:nt + 1]
    S = int(tso[-1])
    sto = L.step_tok_off[:S + 1]
    return synth.Layout(G=1, traj_group=L.traj_group[:nt], traj_reward=L.traj_reward[:nt], traj_step_off=tso,
                        step_tok_off=sto, step_fork=L.step_fork[:S])


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="dart", choices=["dart", "reference"])
    ap.add_argument("--config", default="single")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--q", type=float, default=0.2)
    ap.add_argument("--beta", type=float, default=0.1)
    ap.add_argument("--compact", action="store_true", help="do not zero-fill masked rows")
    ap.add_argument("--kl", default="k3", choices=["k3", "exact"],
                    help="KL estimator: per-token k3 (default) or exact full-vocabulary KL (NEXT #4)")
    ap.add_argument("--fused", action="store_true",
                    help="time the single-read fused update with the mask known in advance (NEXT #1)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--graph", action="store_true", help="also time the pass replayed from a CUDA graph")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-tokens", type=int, default=1024, help="oracle sample tokens per worker process")
    ap.add_argument("--cpu-seconds", type=float, default=10.0, help="cpu_baseline: minimum oracle wall time")
    ap.add_argument("--cpu-procs", type=int, default=0, help="oracle worker processes (0: host cores, memory-bounded)")
    ap.add_argument("--stream-rows", type=int, default=0,
                    help="chunk-stream the batch with chunks of at most this many rows (configs > HBM)")
    ap.add_argument("--pool", type=int, default=3, help="logits/dlogits pool buffers when streaming")
    ap.add_argument("--lmhead", action="store_true",
                    help="time the LM-head-fused old-log-prob pass (NEXT #3) instead of the loss pass")
    ap.add_argument("--hidden", type=int, default=3584, help="hidden size d for --lmhead (Qwen2.5-7B: 3584)")
    ap.add_argument("--no-unfused", action="store_true", help="--lmhead: skip the cuBLAS + logits comparison")
    ap.add_argument("--update", action="store_true", help="--lmhead: time the update pass (dh, dW) instead")
    ap.add_argument("--chunk-rows", type=int, default=0, help="--lmhead --update: rows per chunk (0: whole batch)")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: test path (ranks may share a GPU; collectives staged via host)")
    ap.add_argument("--dry-run", action="store_true",
                    help="N-rank plumbing only (launcher, shards, C1/C2 over gloo), no kernels: CPU tests")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        log("warning: --warmup < 3 violates the timing rules; using 3")
        args.warmup = 3
    argv = sys.argv[1:] if argv is None else list(argv)
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is None and args.gpus > 1:
        # not under torchrun: start one rank per GPU ourselves (the driver's launch)
        raise SystemExit(self_launch(args, argv))
    if env_world is not None and int(env_world) != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} does not match WORLD_SIZE={env_world} (one rank per GPU)")
    if args.dry_run:
        run_dry(args)
    elif args.impl == "reference":
        run_reference(args)
    elif args.lmhead and args.update:
        run_lmhead_update(args)
    elif args.lmhead:
        run_lmhead(args)
    elif args.stream_rows > 0:
        run_streamed(args)
    else:
        run_dart(args)


if __name__ == "__main__":
    main()
