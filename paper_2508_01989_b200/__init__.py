"""taichi-b200: B200-native hybrid iteration of TaiChi (arXiv 2508.01989).

The host engine (C++, include/pdsim) keeps the reference simulator's
instance/scheduler API; the hot path -- the hybrid prefill/decode step and the
KV migration copy -- runs as sm_100a kernels behind the C ABI in
include/taichi_b200.h (lib/libtaichi_b200.so). `runtime` binds that ABI.
"""
from .runtime import (ModelDims, Instance, RemotePool, MigrationEvent, load_library, model_preset,  # noqa: F401
                      gemm, copy_pages, TaichiError)

__all__ = ["ModelDims", "Instance", "RemotePool", "MigrationEvent", "load_library", "model_preset", "gemm",
           "copy_pages", "TaichiError"]
