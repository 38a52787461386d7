"""bench.py's N-rank launch on the host (CPU, gloo): `--gpus N` without
torchrun starts N ranks itself, the weak-scaling layouts give every rank its
own rewards, C1 delivers every rank's step values at its padded slot, and
rank 0 prints exactly one JSON line with n_gpus = N."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _run(*extra, env=None):
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *extra],
                          capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)


def _json_lines(out):
    return [json.loads(l) for l in out.splitlines() if l.startswith("{")]


@pytest.mark.parametrize("n,config", [(2, "single"), (3, "adaptive")])
def test_gpus_n_spawns_n_ranks(n, config):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = _run("--gpus", str(n), "--backend", "gloo", "--dry-run", "--config", config, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1, r.stdout            # rank 0 alone prints
    j = lines[0]
    assert j["n_gpus"] == n and j["backend"] == "gloo" and j["dry_run"] is True
    assert j["c1_layout_ok"] is True
    assert j["config"]["rewards_distinct_per_rank"] is True
    assert j["c2_sum_tokens"] == j["config"]["global_tokens"] == sum(j["config"]["tokens_per_rank"])
    assert j["c2_sum_steps"] == j["config"]["steps_total"]


def test_world_size_mismatch_is_refused():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = _run("--gpus", "2", "--dry-run", env=env)
    assert r.returncode != 0 and "does not match WORLD_SIZE" in r.stderr


def test_weak_layouts_per_rank_blocks():
    import bench
    lays, g, shards, V, _ = bench.weak_layouts("adaptive", 0, 3)
    assert V == 152064 and g.G == sum(L.G for L in lays)
    for r, (L, sh) in enumerate(zip(lays, shards)):
        # rank r's block of the global layout is its own layout, shifted
        assert sh.T_loc == L.T and sh.S_loc == L.S and sh.traj_end - sh.traj_begin == L.N_traj
        assert np.array_equal(g.traj_reward[sh.traj_begin:sh.traj_end], L.traj_reward)
        assert np.array_equal(g.step_tok_off[sh.step_begin:sh.step_end + 1] - sh.tok_begin, L.step_tok_off)
        assert np.array_equal(g.traj_group[sh.traj_begin:sh.traj_end] - int(g.traj_group[sh.traj_begin]),
                              L.traj_group)
    # rank 0 keeps the single-rank batch (N = 1 results unchanged)
    L0, _, _, _ = __import__("paper_2509_23866_b200.synth", fromlist=["x"]).config_layout("adaptive", seed=0)
    assert np.array_equal(lays[0].step_tok_off, L0.step_tok_off)
    assert not np.array_equal(lays[0].traj_reward, lays[1].traj_reward[:len(lays[0].traj_reward)]) \
        or len(lays[0].traj_reward) != len(lays[1].traj_reward)


def test_e2e_host_memory_guard():
    """The e2e leg is skipped (not run into an OOM) when the ranks' pinned
    inputs would not fit in host memory; small inputs always run."""
    import importlib.util
    import torch
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    ok, why = bench.e2e_host_memory_ok([torch.zeros(1024)], 1)
    assert ok and why is None
    os.environ["LOCAL_WORLD_SIZE"] = str(10 ** 9)     # pretend a billion ranks share this host
    try:
        ok, why = bench.e2e_host_memory_ok([torch.zeros(1 << 20)], 1)
    finally:
        del os.environ["LOCAL_WORLD_SIZE"]
    assert not ok and "host memory" in why
