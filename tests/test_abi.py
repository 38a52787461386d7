"""The C-ABI library builds, loads and exports every symbol include/dart_loss.h
declares; host-side argument validation rejects bad calls before any launch
(CPU only: these paths never touch the GPU)."""
import ctypes
import os
import re

import pytest

from paper_2509_23866_b200 import build as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "dart_loss.h")


@pytest.fixture(scope="module")
def L():
    B.build()
    from paper_2509_23866_b200 import dart
    return dart.lib()


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dart_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_three_calls():
    names = declared_functions()
    for n in ("dart_loss_fwd", "dart_select_steps", "dart_loss_bwd"):
        assert n in names


def test_library_exports_every_declared_symbol(L):
    for n in declared_functions():
        assert hasattr(L, n), n
    from paper_2509_23866_b200 import dart
    assert sorted(dart.EXPORTED) == declared_functions()


def test_sm100a_cubin_inside():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", B.OUT], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_and_status_strings(L):
    from paper_2509_23866_b200 import dart
    assert L.dart_abi_version() == dart.ABI_VERSION == 6
    for c in range(5):
        assert L.dart_status_str(c).startswith(b"DART_")
    assert L.dart_status_str(99) == b"DART_UNKNOWN_STATUS"


def _structs():
    from paper_2509_23866_b200 import dart
    cfg = dart.Config().c()
    fake = ctypes.c_void_p(0x100000)   # never dereferenced: validation fails first
    meta = dart.dart_meta(1, 2, 3, 48, fake, fake, fake, fake)
    batch = dart.dart_batch(fake, dart.DART_BF16, 48, 512, 512, 0, 0, 3, fake, fake, fake, fake)
    out = dart.dart_fwd_out(*([fake] * 10))
    return dart, cfg, meta, batch, out


def _fwd(L, dart, cfg, meta, batch, out, ws=ctypes.c_void_p(0x200000), ws_bytes=1 << 40):
    return L.dart_loss_fwd(ctypes.byref(batch), ctypes.byref(meta), ctypes.byref(cfg), ctypes.byref(out),
                           ws, ws_bytes, None)


def test_invalid_arguments_rejected_without_launch(L):
    dart, cfg, meta, batch, out = _structs()
    E = dart.DART_ERR_INVALID_ARG
    assert L.dart_loss_fwd(None, ctypes.byref(meta), ctypes.byref(cfg), ctypes.byref(out), None, 0, None) == E
    b = dart.dart_batch.from_buffer_copy(batch); b.logits = None
    assert _fwd(L, dart, cfg, meta, b, out) == E
    b = dart.dart_batch.from_buffer_copy(batch); b.ld = 100                 # ld < V
    assert _fwd(L, dart, cfg, meta, b, out) == E
    b = dart.dart_batch.from_buffer_copy(batch); b.ld = 513                 # row pitch not 16 B multiple
    assert _fwd(L, dart, cfg, meta, b, out) == E
    b = dart.dart_batch.from_buffer_copy(batch); b.logits = ctypes.c_void_p(0x100002)   # misaligned
    assert _fwd(L, dart, cfg, meta, b, out) == E
    b = dart.dart_batch.from_buffer_copy(batch); b.logits_dtype = 7
    assert _fwd(L, dart, cfg, meta, b, out) == dart.DART_ERR_UNSUPPORTED
    b = dart.dart_batch.from_buffer_copy(batch); b.T_loc = 49               # beyond meta.T
    assert _fwd(L, dart, cfg, meta, b, out) == E
    b = dart.dart_batch.from_buffer_copy(batch); b.logp_ref = None          # beta > 0 needs logp_ref
    assert _fwd(L, dart, cfg, meta, b, out) == E
    for field, val in (("eps_low", 0.0), ("eps_high", 1.0), ("is_cap", 0.0), ("beta_kl", -1.0),
                       ("entropy_q", 1.0), ("inv_temperature", 0.0), ("norm_mode", 9), ("select_rule", -1),
                       ("ratio_level", 2)):
        c = dart.dart_cfg.from_buffer_copy(cfg)
        setattr(c, field, val)
        assert _fwd(L, dart, c, meta, batch, out) == E, field
    o = dart.dart_fwd_out.from_buffer_copy(out); o.status = None
    assert _fwd(L, dart, cfg, meta, batch, o) == E
    # workspace
    assert _fwd(L, dart, cfg, meta, batch, out, ws=None) == dart.DART_ERR_WORKSPACE
    assert _fwd(L, dart, cfg, meta, batch, out, ws_bytes=16) == dart.DART_ERR_WORKSPACE


def test_select_and_bwd_validation(L):
    dart, cfg, meta, batch, out = _structs()
    fake = ctypes.c_void_p(0x100000)
    E = dart.DART_ERR_INVALID_ARG
    sel = lambda world, spad, rso=fake, ws_bytes=1 << 30: L.dart_select_steps(  # noqa: E731
        fake, rso, world, spad, ctypes.byref(meta), ctypes.byref(cfg), fake, fake, fake, fake,
        ctypes.c_void_p(0x200000), ws_bytes, None)
    assert sel(0, 3) == E
    assert sel(1, 2) == E                  # S_pad < S at one rank
    assert sel(2, 1) == E                  # world * S_pad < S
    assert sel(2, 3, rso=None) == E
    assert sel(1, 3, ws_bytes=8) == dart.DART_ERR_WORKSPACE
    bwd = lambda gdt, ldg, dl=fake: L.dart_loss_bwd(  # noqa: E731
        ctypes.byref(batch), ctypes.byref(meta), ctypes.byref(cfg), ctypes.byref(out), fake, fake, dl, gdt, ldg,
        fake, ctypes.c_void_p(0x200000), 1 << 40, None)
    assert bwd(5, 512) == dart.DART_ERR_UNSUPPORTED
    assert bwd(dart.DART_BF16, 511) == E
    assert bwd(dart.DART_BF16, 513) == E
    # dlogits = NULL is the loss-only mode: validation passes (ld / grad dtype ignored) up to the workspace
    assert L.dart_loss_bwd(ctypes.byref(batch), ctypes.byref(meta), ctypes.byref(cfg), ctypes.byref(out), fake, fake,
                           None, 5, 0, fake, ctypes.c_void_p(0x200000), 8, None) == dart.DART_ERR_WORKSPACE
    assert L.dart_loss_bwd(ctypes.byref(batch), ctypes.byref(meta), ctypes.byref(cfg), ctypes.byref(out), fake, None,
                           None, 5, 0, fake, ctypes.c_void_p(0x200000), 1 << 40, None) == E   # norm required
    # whole-batch convenience call requires the shard to be the whole batch
    b = dart.dart_batch.from_buffer_copy(batch); b.T_loc = 40
    assert L.dart_loss_pass(ctypes.byref(b), ctypes.byref(meta), ctypes.byref(cfg), ctypes.byref(out), fake, fake,
                            fake, fake, dart.DART_BF16, 512, fake, ctypes.c_void_p(0x200000), 1 << 40, None) == E


def test_workspace_size_is_host_only_and_monotone(L):
    dart, cfg, meta, batch, out = _structs()
    w1 = L.dart_workspace_size(ctypes.byref(batch), ctypes.byref(meta), ctypes.byref(cfg))
    b = dart.dart_batch.from_buffer_copy(batch); b.T_loc = 20000
    m = dart.dart_meta.from_buffer_copy(meta); m.T = 40000
    w2 = L.dart_workspace_size(ctypes.byref(b), ctypes.byref(m), ctypes.byref(cfg))
    assert 0 < w1 < w2


def test_lmhead_validation(L):
    """dart_lmhead_fwd rejects bad LM-head operands before any launch."""
    dart, cfg, meta, batch, out = _structs()
    E = dart.DART_ERR_INVALID_ARG
    fake = ctypes.c_void_p(0x100000)
    good = dart.dart_lmhead(fake, ctypes.c_void_p(0x300000), 64, 64, 72)

    def call(head, b=batch, c=cfg, ws_bytes=1 << 40):
        return L.dart_lmhead_fwd(None if head is None else ctypes.byref(head), ctypes.byref(b), ctypes.byref(meta),
                                 ctypes.byref(c), ctypes.byref(out), ctypes.c_void_p(0x200000), ws_bytes, None)
    assert call(None) == E
    for field, val in (("d", 0), ("d", 60), ("ld_h", 32), ("ld_w", 68), ("hidden", None),
                       ("weight", ctypes.c_void_p(0x300008))):
        h = dart.dart_lmhead.from_buffer_copy(good)
        setattr(h, field, val)
        assert call(h) == E, field
    b = dart.dart_batch.from_buffer_copy(batch); b.logits = None            # logits are not needed here
    assert call(good, b=b, ws_bytes=8) == dart.DART_ERR_WORKSPACE
    c = dart.dart_cfg.from_buffer_copy(cfg); c.kl_mode = dart.KL_EXACT       # needs the reference logits
    assert call(good, c=c) == dart.DART_ERR_UNSUPPORTED
    b = dart.dart_batch.from_buffer_copy(batch); b.logits = None
    w0 = L.dart_workspace_size(ctypes.byref(batch), ctypes.byref(meta), ctypes.byref(cfg))
    w1 = L.dart_lmhead_workspace_size(ctypes.byref(good), ctypes.byref(b), ctypes.byref(meta), ctypes.byref(cfg))
    assert w1 > w0


def test_binding_refuses_cpu_tensors():
    import torch
    from paper_2509_23866_b200 import dart
    with pytest.raises(dart.DartError):
        dart._require_cuda(torch.zeros(3))


def test_lmhead_bwd_validation(L):
    """dart_lmhead_bwd (training half) rejects bad buffers
    before any launch; stats_accumulate must be 0 or 1."""
    dart, cfg, meta, batch, out = _structs()
    E = dart.DART_ERR_INVALID_ARG
    fake = ctypes.c_void_p(0x100000)
    head = dart.dart_lmhead(fake, ctypes.c_void_p(0x300000), 64, 64, 72)
    b = dart.dart_batch.from_buffer_copy(batch); b.logits = None

    def call(dz=fake, ldg=512, hk=fake, ld_hk=64, rows=fake, nk=fake, norm=fake, stats=fake, c=cfg, ws_bytes=1 << 40):
        return L.dart_lmhead_bwd(ctypes.byref(head), ctypes.byref(b), ctypes.byref(meta), ctypes.byref(c),
                                 ctypes.byref(out), fake, norm, dz, ldg, hk, ld_hk, rows, nk, stats,
                                 ctypes.c_void_p(0x200000), ws_bytes, None)
    assert call(ws_bytes=8) == dart.DART_ERR_WORKSPACE      # everything else valid
    assert call(dz=None) == E
    assert call(ldg=500) == E                                # < V
    assert call(ldg=516) == E                                # % 8
    assert call(dz=ctypes.c_void_p(0x100008)) == E           # misaligned
    assert call(hk=None) == E
    assert call(ld_hk=32) == E                               # < d
    assert call(rows=None) == E
    assert call(nk=None) == E
    assert call(norm=None) == E
    assert call(stats=None) == E
    c = dart.dart_cfg.from_buffer_copy(cfg); c.stats_accumulate = 2
    assert call(c=c) == E
