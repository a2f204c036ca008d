"""B200-native PPO/RLVR logits -> training-signal path (OpenRLHF, arXiv 2405.11143).

The product is ``liborl.so`` (hand-written sm_100a CUDA behind a C ABI,
``include/orl.h``); ``paper_2405_11143_b200.orl`` is its thin ctypes binding
(imported on first use, so that ``synth`` can be used without the library).
``synth`` generates seeded synthetic inputs and holds none of the method.
"""
import importlib

__all__ = ["orl", "synth", "pipeline"]


def __getattr__(name):
    if name in ("orl", "pipeline"):
        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)
