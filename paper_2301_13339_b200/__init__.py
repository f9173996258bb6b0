"""B200-native QTT convolution (arXiv 2301.13339 hot path).

The compute path is the C-ABI library `libqtt.so` (include/qtt.h) built from
hand-written sm_100a CUDA; `paper_2301_13339_b200.qtt` is the thin ctypes
binding.  Importing this package does not load the library (so the seeded
input generators in `synth` stay importable without it); the first call into
`paper_2301_13339_b200.qtt` loads it and fails loudly if it is missing.
"""

__all__ = ["qtt", "synth"]
