"""paper_2512_00722_b200 — B200-native (sm_100a) SpeContext decode-step hot path.

The compute path is libspc.so (hand-written CUDA, C ABI in include/spc.h).
This package is a thin binding: ``spc`` (ctypes marshalling of the five
calls), ``pipeline`` (one decode step from those calls), ``dist``
(context-sharded driver over torch.distributed), ``synth`` (seeded inputs) and
``roofline`` (byte accounting).  Importing the package does not load CUDA; the
first call into ``spc`` does, and raises if libspc.so is missing — there is no
CPU fallback.
"""
__all__ = ["spc", "pipeline", "dist", "synth", "roofline"]
