"""vexbayes-b200: B200-native hot path of arXiv 1902.09046 ("vexbayes").

Batched, independent prior-predictive simulation inside likelihood-free
samplers, as hand-written sm_100a kernels behind a C ABI
(include/vexbayes_cuda.h, built into libvexbayes_cuda.so by ``build``).

Layout: ``csrc/`` CUDA kernels + the C ABI; ``cpp/vexbayes/`` the C++ shim that
keeps the reference's vexbayes:: signatures; ``lib`` the ctypes binding;
``models`` POD model descriptors; ``abc`` / ``dist`` the host layer used by
bench.py (single GPU and torch.distributed sharding).
"""
from . import _abi, models  # noqa: F401

__all__ = ["_abi", "models", "lib", "build"]
