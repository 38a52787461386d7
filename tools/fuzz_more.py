"""Extended randomised parity sweep (on the GPU box): the cases of
tests/test_fuzz_gpu.py / test_fuzz_paths_gpu.py for seeds [a, b) -- main
path, fused update (even seeds), virtual ranks, exact KL, LM-head forward and
the streamed pass (subsets of seeds) -- each against the float64 oracle or the
resident pass.
Usage: python tools/fuzz_more.py 96 600"""
import sys
import traceback
sys.path.insert(0, ".")
from tests import test_fuzz_gpu as F
from tests import test_fuzz_paths_gpu as P

a, b = (int(x) for x in sys.argv[1:3])
fails = []
for seed in range(a, b):
    tests = [("main", F.test_fuzz_main_path_vs_oracle)]
    if seed % 2 == 0:
        tests.append(("fused", F.test_fuzz_fused_vs_oracle))
    else:
        tests.append(("fused_hard", F.test_fuzz_fused_hard_inputs_vs_oracle))
    if seed % 6 == 1:
        tests.append(("vranks", F.test_fuzz_virtual_ranks_vs_oracle))
    if seed % 8 == 5:
        tests.append(("zero_fill_off", F.test_fuzz_zero_fill_off))
    if seed % 3 == 0:
        tests.append(("exact_kl", P.test_fuzz_exact_kl_vs_oracle))
    if seed % 3 == 1:
        tests.append(("exact_kl_hard", P.test_fuzz_exact_kl_hard_inputs_vs_oracle))
    if seed % 6 == 1:
        tests.append(("lmhead", P.test_fuzz_lmhead_forward_vs_oracle))
    if seed % 6 == 2:
        tests.append(("stream", P.test_fuzz_streamed_equals_resident))
    if seed % 8 == 3:
        tests.append(("lmupdate", P.test_fuzz_lmhead_update_vs_oracle))
    for name, fn in tests:
        try:
            fn(seed)
        except BaseException as e:   # noqa: BLE001  (report and continue; pytest.skip is a BaseException)
            if type(e).__name__ == "Skipped":
                continue
            if isinstance(e, KeyboardInterrupt):
                raise
            fails.append((seed, name, repr(e)[:300]))
            print("FAIL", seed, name, repr(e)[:300], flush=True)
            traceback.print_exc(limit=3)
print(f"seeds {a}..{b - 1}: {len(fails)} failures", flush=True)
