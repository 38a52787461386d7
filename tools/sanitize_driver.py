"""Small driver for compute-sanitizer: one pass of a few configs through the C ABI."""
import sys
sys.path.insert(0, '.')
import torch
from paper_2509_23866_b200 import dart, synth
from tests.gpu_helpers import run_gpu

which = sys.argv[1:] or ["tiny", "small_multi", "odd"]
for name in which:
    if name == "odd":
        layout, _, _, _ = synth.config_layout("small_multi", seed=1)
        b = synth.make_batch("small_multi", seed=1, layout=layout, V=1001, dtype=torch.bfloat16, pad_ld=1008)
    elif name == "midsplit":   # V = 152064, few rows -> split-row mode + bulk copies of full chunks
        layout, _, _, _ = synth.config_layout("grid1x2x2x16@152064", seed=0)
        b = synth.make_batch("x", seed=0, layout=layout, V=152064, dtype=torch.bfloat16)
    else:
        b = synth.make_batch(name, seed=0)
    dl = run_gpu(b, dart.Config(is_cap=2.0 if name.startswith("tiny") else 1.0))
    dl.check_status()
    print(name, "ok", dl.stats_dict()["loss"])
