"""B200-native PPO/RLVR logits -> training-signal path (OpenRLHF, arXiv 2405.11143).

The product is ``liborl.so`` (hand-written sm_100a CUDA behind a C ABI,
``include/orl.h``); ``paper_2405_11143_b200.orl`` is its thin ctypes binding.
``synth`` generates seeded synthetic inputs and holds none of the method.
"""
__all__ = ["orl", "synth"]


def __getattr__(name):
    if name == "orl":
        from . import orl as _orl
        return _orl
    raise AttributeError(name)
