"""B200-native reconstruction hot path of arXiv 2010.15491 (3D-FSR).

The product is `_lib/libvsr_b200.so` (hand-written sm_100a CUDA kernels behind
the C ABI in include/vsr.h).  `paper_2010_15491_b200.volsr` is the Python
mirror of the reference `volsr` C++ solver API over that ABI;
`paper_2010_15491_b200.synth` builds seeded synthetic inputs.
"""
__all__ = ["volsr", "synth"]
