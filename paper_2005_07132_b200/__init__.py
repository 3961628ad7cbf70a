"""B200-native fKK-EC (arxiv 2005.07132): factorized Kramers-Kronig + phase/scale error correction,
ML reuse and the direct per-spectrum KK path, behind the C-ABI of include/fkk.h.

``paper_2005_07132_b200.fkk`` is the ctypes binding of lib/libfkk.so (built by build.py).
Importing the package does not import torch or load the library; ``from paper_2005_07132_b200
import fkk`` does, and fails loudly if the library is missing.
"""
__all__ = ["fkk", "build"]
