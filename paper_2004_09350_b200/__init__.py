"""paper_2004_09350_b200 — B200-native (sm_100a) compression-enabled
operator-at-a-time hot path of MorphStore (arXiv 2004.09350).

The product is libms.so (C ABI in include/ms.h, kernels in csrc/); `ms` is its
Python binding. Importing `ms` fails loudly if libms.so is missing.
"""
import os

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIBMS = os.path.join(PKG_DIR, "libms.so")
