"""hetreco-b200: B200-native (sm_100a) MRI reconstruction process chain with
the OpenCLIPER/hetreco operator API.

The product is ``libhetreco_b200.so`` (C++ host library + sm_100a kernels +
C-ABI, built in-tree by ``paper_1807_11830_b200.build``); ``hetreco`` is the
Python ctypes mirror of the API.
"""
from . import hetreco  # noqa: F401

__all__ = ["hetreco"]
