"""B200-native Ok-Topk sparse allreduce (arXiv 2201.07598).

The product is the C-ABI library ``libokt.so`` (include/okt.h): hand-written
sm_100a kernels plus C++ orchestration over NVLink (NCCL or peer copies).
``oktopk`` mirrors the reference's C++ interface for Python callers and tests.
"""
from ._lib import LIB_PATH, lib  # noqa: F401

__all__ = ["lib", "LIB_PATH"]
