"""Randomised multi-process check (on the GPU box): the tests/test_fuzz_gpu.py
cases for seeds 100..139 over 2-5 real gloo process groups sharing one GPU,
every rank against the oracle (tests/test_multi_gpu.py machinery)."""
import sys; sys.path.insert(0, ".")
from tests import test_multi_gpu as M

def main():
    fails = 0
    for seed in range(100, 140):
        world = 2 + seed % 4
        name = f"fuzz/{seed}"
        try:
            M._check(M._run("gloo", world, name, seed), name, seed, None); print("ok", seed, world, flush=True)
        except BaseException as e:
            if type(e).__name__ == "Skipped": continue
            fails += 1; print("FAIL", seed, world, repr(e)[:300], flush=True)
    print("failures", fails)


if __name__ == "__main__":
    main()
