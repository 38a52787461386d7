"""paper_2509_23866_b200 -- B200-native DART policy-loss pass.

The product is the C-ABI CUDA library `libdart_loss.so` (include/dart_loss.h);
`paper_2509_23866_b200.dart` is the thin ctypes binding with the same names.
Importing this package does not load the library; `synth` (the seeded input
generator) is importable on a CPU-only box.
"""
__all__ = ["dart", "synth", "dist"]


def __getattr__(name):
    import importlib
    if name in __all__:
        return importlib.import_module(f"{__name__}.{name}")
    raise AttributeError(name)
