"""Guard-band bounds checks of every write the library makes (the stand-in
for compute-sanitizer memcheck on pools where the sanitizer is closed).

Every device buffer the C ABI writes -- the per-token and per-step outputs,
keep / tau / norm / stats, the workspace and the gradient rows -- is placed
inside a larger allocation whose leading and trailing guard bands (and the
gradient's pad columns between V and the row pitch) hold a sentinel byte
pattern.  The inputs are placed the same way and must come back unchanged.
After the pass every sentinel byte must be intact: a single out-of-range
store anywhere (a wrong row pitch, a tail vector written whole, a masked row
written past V, a workspace overrun) fails the test.  Each case also checks
the pass's status word and, where the parity tests do not already cover the
shape, the loss against the oracle."""
import numpy as np
import pytest
import torch

from oracle import dart_oracle as O
from paper_2509_23866_b200 import dart, synth

pytestmark = pytest.mark.gpu

GUARD = 4096          # bytes on each side (keeps the interior 256-byte aligned)
SENT = 0xA5


class Guarded:
    """A byte buffer with sentinel guard bands around an interior view."""

    def __init__(self, shape, dtype, dev, fill=None):
        n = int(np.prod(shape)) * torch.empty((), dtype=dtype).element_size()
        self.raw = torch.full((GUARD + n + GUARD,), SENT, dtype=torch.uint8, device=dev)
        self.n = n
        self.view = self.raw[GUARD:GUARD + n].view(dtype).view(*shape) if n else \
            torch.empty(shape, dtype=dtype, device=dev)
        if fill is not None and n:
            self.view.copy_(fill)

    def intact(self):
        head = self.raw[:GUARD].cpu().numpy()
        tail = self.raw[GUARD + self.n:].cpu().numpy()
        return bool((head == SENT).all() and (tail == SENT).all())


def guard_outputs(dl, dev):
    """Re-home every buffer DartLoss hands to the ABI into guarded storage."""
    gs = {}
    for name in ("lse", "logp", "H", "ell", "dell", "step_H", "step_ell", "adv", "group_ok", "status", "keep",
                 "tau", "norm", "stats", "ws"):
        t = getattr(dl, name)
        g = Guarded(tuple(t.shape), t.dtype, dev, fill=torch.zeros_like(t) if name == "status" else None)
        setattr(dl, name, g.view)
        gs[name] = g
    if dl.dlogits_store is not None:
        T, ldg = dl.dlogits_store.shape
        g = Guarded((T, ldg), dl.dlogits_store.dtype, dev)
        dl.dlogits_store = g.view
        dl.dlogits = g.view[:, :dl.V]
        gs["dlogits"] = g
    return gs


def guard_inputs(tensors, dev):
    out, gs = [], []
    for t in tensors:
        if t is None:
            out.append(None)
            continue
        g = Guarded(tuple(t.shape), t.dtype, dev, fill=t.to(dev))
        out.append(g.view)
        gs.append((g, t.to(dev).clone()))
    return out, gs


def check(gs_out, gs_in, dl):
    bad = [n for n, g in gs_out.items() if not g.intact()]
    assert not bad, f"guard band overwritten: {bad}"
    for g, orig in gs_in:
        assert g.intact(), "guard band of an input overwritten"
        assert torch.equal(g.view.view(torch.uint8), orig.view(torch.uint8)), "an input was modified"
    if "dlogits" in gs_out and dl.dlogits_store.shape[1] > dl.V:
        pad = dl.dlogits_store[:, dl.V:].contiguous().view(torch.uint8).cpu().numpy()
        assert (pad == SENT).all(), "gradient pad columns (V..ldg) written"
    dl.check_status()


def _batch(name):
    if name == "odd":          # odd V, padded logits pitch, ragged groups
        layout, _, _, _ = synth.config_layout("small_multi", seed=1)
        return synth.make_batch("small_multi", seed=1, layout=layout, V=1001, dtype=torch.bfloat16, pad_ld=1008)
    if name == "tiny":         # fp32 logits, the tiny config
        return synth.make_batch("tiny", seed=0)
    if name == "midsplit":     # few rows at V = 152064 -> split-row mode, full bulk chunks + vocabulary tail
        layout, _, _, _ = synth.config_layout("grid1x2x2x16@152064", seed=0)
        return synth.make_batch("x", seed=0, layout=layout, V=152064, dtype=torch.bfloat16)
    if name == "tail":         # V not a multiple of the chunk, rows of 3 steps
        layout, _, _, _ = synth.config_layout("grid2x2x3x24@30001", seed=0)
        return synth.make_batch("x", seed=0, layout=layout, V=30001, dtype=torch.bfloat16, pad_ld=30016)
    raise KeyError(name)


def _dl(b, cfg, extra_pitch, grad_dtype=None):
    gd = grad_dtype or (torch.float32 if b.logits.dtype == torch.float32 else torch.bfloat16)
    per = 16 // gd.itemsize
    ldg = -(-b.V // per) * per + extra_pitch
    return dart.DartLoss(b.layout, dart.whole_shard(b.layout), b.V, cfg, "cuda", logits_dtype=b.logits.dtype,
                         grad_dtype=gd, ld=b.logits_store.stride(0), ldg=ldg)


def _inputs(b, dev):
    return guard_inputs([b.logits_store, b.target, b.logp_old, b.logp_rollout, b.logp_ref], dev)


@pytest.mark.parametrize("name", ["tiny", "odd", "midsplit", "tail"])
@pytest.mark.parametrize("zero_fill", [1, 0])
def test_main_path_writes_in_bounds(name, zero_fill):
    dev = torch.device("cuda")
    b = _batch(name)
    cfg = dart.Config(is_cap=2.0, zero_fill_masked=zero_fill, entropy_q=0.5)
    dl = _dl(b, cfg, extra_pitch=16)
    gs_out = guard_outputs(dl, dev)
    (lg, tg, lo, lr, lref), gs_in = _inputs(b, dev)
    dl.run(lg[:, :b.V], tg, lo, lr, lref)
    torch.cuda.synchronize()
    check(gs_out, gs_in, dl)
    if not zero_fill:     # masked rows are not written at all: their sentinel bytes stay
        keep = dl.keep.cpu().numpy()[:b.layout.S].astype(bool)
        n = np.diff(b.layout.step_tok_off)
        masked_rows = np.repeat(~keep, n)
        if masked_rows.any():
            rows = dl.dlogits_store[torch.as_tensor(np.nonzero(masked_rows)[0], device=dev)]
            assert (rows.contiguous().view(torch.uint8).cpu().numpy() == SENT).all()
    ref = O.loss_pass(b.oracle_dict(), cfg.as_f32(), keep_override=dl.keep.cpu().numpy())
    scale = float(np.sum(np.abs(ref["c_tok"] * ref["ell"]))) + 1e-30
    assert abs(dl.stats_dict()["loss"] - ref["loss"]) <= 1e-5 * scale


@pytest.mark.parametrize("name", ["odd", "midsplit", "tail"])
@pytest.mark.parametrize("zero_fill", [1, 0])
def test_fused_writes_in_bounds(name, zero_fill):
    dev = torch.device("cuda")
    b = _batch(name)
    cfg = dart.Config(zero_fill_masked=zero_fill, entropy_q=0.5)
    old = _dl(b, cfg, extra_pitch=0)
    args = (b.logits_store.to(dev)[:, :b.V], b.target.to(dev), b.logp_old.to(dev), b.logp_rollout.to(dev), b.logp_ref.to(dev))
    old.run(*args)
    torch.cuda.synchronize()
    keep, norm = Guarded((old.keep.numel(),), torch.uint8, dev, fill=old.keep), \
        Guarded((5,), torch.int64, dev, fill=old.norm)
    dl = _dl(b, cfg, extra_pitch=24)
    gs_out = guard_outputs(dl, dev)
    (lg, tg, lo, lr, lref), gs_in = _inputs(b, dev)
    dl.fused(lg[:, :b.V], tg, lo, lr, lref, keep=keep.view, norm=norm.view)
    torch.cuda.synchronize()
    gs_in += [(keep, old.keep.clone()), (norm, old.norm.clone())]
    check(gs_out, gs_in, dl)
    assert abs(dl.stats_dict()["loss"] - old.stats_dict()["loss"]) <= 1e-5 * max(1e-6, abs(old.stats_dict()["loss"]))


def test_exact_kl_writes_in_bounds():
    dev = torch.device("cuda")
    b = synth.make_batch("small_multi", seed=0, with_ref=True)
    cfg = dart.Config(kl_mode=dart.KL_EXACT)
    gd = torch.float32 if b.logits.dtype == torch.float32 else torch.bfloat16
    dl = dart.DartLoss(b.layout, dart.whole_shard(b.layout), b.V, cfg, "cuda", logits_dtype=b.logits.dtype,
                       grad_dtype=gd, ldg=-(-b.V // 8) * 8 + 8)
    gs_out = guard_outputs(dl, dev)
    (lg, tg, lo, lr, lref, rl), gs_in = guard_inputs(
        [b.logits, b.target, b.logp_old, b.logp_rollout, b.logp_ref, b.ref_logits], dev)
    dl.run(lg, tg, lo, lr, lref, rl)
    torch.cuda.synchronize()
    check(gs_out, gs_in, dl)


def test_lmhead_forward_writes_in_bounds():
    dev = torch.device("cuda")
    lb = synth.make_lmhead("grid2x4x3x20@3000", 256, seed=3)
    bb = lb.batch
    dl = dart.DartLoss(bb.layout, dart.whole_shard(bb.layout), bb.V, dart.Config(), "cuda", with_grad=False)
    gs_out = guard_outputs(dl, dev)
    (h, w, tg, lo, lr, lref), gs_in = guard_inputs(
        [lb.hidden, lb.weight, bb.target, bb.logp_old, bb.logp_rollout, bb.logp_ref], dev)
    dl.forward_lmhead(h, w, tg, lo, lr, lref)
    dl.select()
    torch.cuda.synchronize()
    check(gs_out, gs_in, dl)


def test_guard_detects_an_overrun():
    """The harness itself: one byte written past an interior is caught."""
    g = Guarded((7, 9), torch.bfloat16, torch.device("cuda"))
    assert g.intact()
    g.raw[GUARD + g.n] = 0
    assert not g.intact()
