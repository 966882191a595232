"""ctypes binding of the C ABI in include/taichi_b200.h (lib/libtaichi_b200.so).

This is the Python face of the drop-in boundary: tests and bench.py call the
GPU path exactly as the C++ host engine does. There is no CPU fallback -- if
the CUDA library is missing or no B200 is visible, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os
import pathlib
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

_PKG = pathlib.Path(__file__).resolve().parent
LIB_PATH = _PKG / "lib" / "libtaichi_b200.so"

EXPORTED = [
    "tc_model_preset", "tc_instance_create", "tc_instance_destroy", "tc_step_launch", "tc_step_wait",
    "tc_kv_reserve", "tc_kv_release", "tc_kv_stats", "tc_kv_migrate", "tc_kv_migrate_wait",
    "tc_kv_pool_info", "tc_kv_pages", "tc_weight_ptr", "tc_read_device", "tc_weight_value", "tc_gemm",
    "tc_copy_pages", "tc_set_profiling", "tc_phase_ms", "tc_last_error", "tc_version",
    "tc_kv_migrate_async", "tc_event_query", "tc_event_wait", "tc_event_destroy", "tc_set_migration_ctas",
    "tc_kv_pool_export", "tc_kv_pool_import", "tc_remote_pool_close", "tc_kv_push_pages",
]
IPC_HANDLE_BYTES = 64  # TC_IPC_HANDLE_BYTES


class TaichiError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[tc_status {code}] {msg}")
        self.code = code


class ModelDims(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("d_model", C.c_int32), ("n_heads", C.c_int32),
                ("n_kv_heads", C.c_int32), ("head_dim", C.c_int32), ("ffn_dim", C.c_int32),
                ("vocab", C.c_int32), ("qkv_bias", C.c_int32), ("rope_theta", C.c_float),
                ("rms_eps", C.c_float)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class _InstanceDesc(C.Structure):
    _fields_ = [("device", C.c_int32), ("dims", ModelDims), ("weight_seed", C.c_uint64),
                ("page_size", C.c_int32), ("kv_pool_tokens", C.c_int64), ("max_step_tokens", C.c_int32),
                ("max_seqs", C.c_int32), ("max_context", C.c_int32), ("share_weights", C.c_void_p),
                ("share_kv_pool", C.c_void_p)]


class _PrefillSlice(C.Structure):
    _fields_ = [("req_id", C.c_int64), ("pos0", C.c_int32), ("n_tokens", C.c_int32),
                ("token_ids", C.POINTER(C.c_int32)), ("want_logits", C.c_int32)]


class _DecodeItem(C.Structure):
    _fields_ = [("req_id", C.c_int64), ("pos", C.c_int32), ("token_id", C.c_int32)]


class _StepDesc(C.Structure):
    _fields_ = [("n_prefill", C.c_int32), ("prefill", C.POINTER(_PrefillSlice)), ("n_decode", C.c_int32),
                ("decode", C.POINTER(_DecodeItem)), ("flags", C.c_int32)]


class _StepResult(C.Structure):
    _fields_ = [("n_sampled", C.c_int32), ("sampled_ids", C.POINTER(C.c_int32)),
                ("logits", C.POINTER(C.c_float)), ("gpu_ms", C.c_float), ("launches", C.c_int32),
                ("h2d_bytes", C.c_int64), ("d2h_bytes", C.c_int64), ("attn_pf_sms", C.c_int32)]


_lib: Optional[C.CDLL] = None


def load_library(path: Optional[os.PathLike] = None) -> C.CDLL:
    """Load libtaichi_b200.so (build it with `python -m paper_2508_01989_b200.build`)."""
    global _lib
    if _lib is not None:
        return _lib
    p = pathlib.Path(path) if path else pathlib.Path(os.environ.get("TAICHI_B200_LIB", LIB_PATH))
    if not p.exists():
        raise FileNotFoundError(f"{p} missing: the CUDA library is not built (no CPU fallback exists)")
    lib = C.CDLL(str(p))
    P, I32, I64, U64 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64
    sig = {
        "tc_model_preset": (I32, [C.c_char_p, C.POINTER(ModelDims)]),
        "tc_instance_create": (I32, [C.POINTER(_InstanceDesc), C.POINTER(P)]),
        "tc_instance_destroy": (I32, [P]),
        "tc_step_launch": (I32, [P, C.POINTER(_StepDesc)]),
        "tc_step_wait": (I32, [P, C.POINTER(_StepResult)]),
        "tc_kv_reserve": (I32, [P, I64, I64]),
        "tc_kv_release": (I32, [P, I64]),
        "tc_kv_stats": (I32, [P, I64, C.POINTER(I64), C.POINTER(I64)]),
        "tc_kv_migrate": (I32, [P, P, I64, I64]),
        "tc_kv_migrate_wait": (I32, [P, C.POINTER(C.c_float), C.POINTER(I64)]),
        "tc_kv_migrate_async": (I32, [P, P, I64, I64, C.POINTER(P)]),
        "tc_event_query": (I32, [P, C.POINTER(I32)]),
        "tc_event_wait": (I32, [P, C.POINTER(C.c_float), C.POINTER(I64)]),
        "tc_event_destroy": (I32, [P]),
        "tc_set_migration_ctas": (I32, [P, I32]),
        "tc_kv_pool_export": (I32, [P, P, C.POINTER(I64), C.POINTER(I64)]),
        "tc_kv_pool_import": (I32, [I32, P, I64, I64, C.POINTER(P)]),
        "tc_remote_pool_close": (I32, [P]),
        "tc_kv_push_pages": (I32, [P, P, C.POINTER(I32), C.POINTER(I32), I32, C.POINTER(P)]),
        "tc_kv_pool_info": (I32, [P, C.POINTER(P), C.POINTER(I64), C.POINTER(I64)]),
        "tc_kv_pages": (I32, [P, I64, C.POINTER(I32), I32, C.POINTER(I32)]),
        "tc_weight_ptr": (I32, [P, C.c_char_p, C.POINTER(P), C.POINTER(I64), C.POINTER(I64)]),
        "tc_read_device": (I32, [P, P, C.c_size_t]),
        "tc_weight_value": (C.c_uint16, [U64, U64, I64, C.c_float, C.c_float]),
        "tc_gemm": (I32, [I32, P, P, P, P, I32, I32, I32, I32, I32, I32, P]),
        "tc_copy_pages": (I32, [P, P, P, P, I32, I64, P]),
        "tc_set_profiling": (I32, [P, I32]),
        "tc_phase_ms": (I32, [P, C.c_char_p, C.POINTER(C.c_float)]),
        "tc_last_error": (C.c_char_p, []),
        "tc_version": (C.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def _check(status: int) -> None:
    if status != 0:
        raise TaichiError(status, load_library().tc_last_error().decode())


def model_preset(name: str) -> ModelDims:
    d = ModelDims()
    _check(load_library().tc_model_preset(name.encode(), C.byref(d)))
    return d


@dataclass
class StepOutput:
    sampled: np.ndarray           # int32 [n_sampled]
    logits: Optional[np.ndarray]  # fp32 [n_sampled, vocab] when requested
    gpu_ms: float
    launches: int = 0
    h2d_bytes: int = 0
    d2h_bytes: int = 0
    attn_pf_sms: int = 0          # SMs prefill attention ran on beside decode attention (0 = serial)


class Instance:
    """One TaiChi instance on one GPU (tc_instance)."""

    def __init__(self, model: str | ModelDims = "tiny", device: int = 0, weight_seed: int = 0,
                 kv_pool_tokens: int = 1 << 16, max_step_tokens: int = 2048, max_seqs: int = 256,
                 max_context: int = 4096, page_size: int = 16, share_weights: "Instance | None" = None,
                 share_kv_pool: "Instance | None" = None):
        lib = load_library()
        self.dims = model_preset(model) if isinstance(model, str) else model
        desc = _InstanceDesc(device, self.dims, weight_seed, page_size, kv_pool_tokens, max_step_tokens,
                             max_seqs, max_context, share_weights._h.value if share_weights is not None else None,
                             share_kv_pool._h.value if share_kv_pool is not None else None)
        self._shared_from = (share_weights, share_kv_pool)  # keep the owners alive
        h = C.c_void_p()
        _check(lib.tc_instance_create(C.byref(desc), C.byref(h)))
        self._h = h
        self.device = device
        self.page_size = page_size
        self.max_context = max_context
        self._pending_keep = False

    # ---------------------------------------------------------------- lifetime
    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            _check(load_library().tc_instance_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def handle(self):
        return self._h

    # ---------------------------------------------------------------- steps
    def launch(self, prefill: Sequence[tuple] = (), decode: Sequence[tuple] = (), keep_logits=False):
        """prefill: (req_id, pos0, token_ids, want_logits); decode: (req_id, pos, token_id)."""
        lib = load_library()
        self._keep_alive = []
        slices = (_PrefillSlice * max(1, len(prefill)))()
        for i, (rid, pos0, toks, want) in enumerate(prefill):
            arr = np.ascontiguousarray(toks, dtype=np.int32)
            self._keep_alive.append(arr)
            slices[i] = _PrefillSlice(rid, pos0, len(arr), arr.ctypes.data_as(C.POINTER(C.c_int32)), int(want))
        items = (_DecodeItem * max(1, len(decode)))()
        for i, (rid, pos, tok) in enumerate(decode):
            items[i] = _DecodeItem(rid, pos, tok)
        self._keep_alive += [slices, items]
        desc = _StepDesc(len(prefill), slices, len(decode), items, 1 if keep_logits else 0)
        _check(lib.tc_step_launch(self._h, C.byref(desc)))
        self._pending_keep = keep_logits
        self._pending_n = sum(1 for p in prefill if p[3]) + len(decode)

    def wait(self) -> StepOutput:
        lib = load_library()
        n = self._pending_n
        ids = np.zeros(max(1, n), dtype=np.int32)
        logits = np.zeros((max(1, n), self.dims.vocab), dtype=np.float32) if self._pending_keep else None
        res = _StepResult(0, ids.ctypes.data_as(C.POINTER(C.c_int32)),
                          logits.ctypes.data_as(C.POINTER(C.c_float)) if logits is not None else None, 0.0, 0, 0, 0, 0)
        _check(lib.tc_step_wait(self._h, C.byref(res)))
        return StepOutput(ids[:res.n_sampled].copy(),
                          logits[:res.n_sampled].copy() if logits is not None else None, float(res.gpu_ms),
                          int(res.launches), int(res.h2d_bytes), int(res.d2h_bytes), int(res.attn_pf_sms))

    def step(self, prefill=(), decode=(), keep_logits=False) -> StepOutput:
        self.launch(prefill, decode, keep_logits)
        return self.wait()

    # ---------------------------------------------------------------- KV
    def kv_reserve(self, rid: int, n_tokens: int):
        _check(load_library().tc_kv_reserve(self._h, rid, n_tokens))

    def kv_release(self, rid: int):
        _check(load_library().tc_kv_release(self._h, rid))

    def kv_stats(self, rid: int = -1):
        a, b = C.c_int64(), C.c_int64()
        _check(load_library().tc_kv_stats(self._h, rid, C.byref(a), C.byref(b)))
        return a.value, b.value

    def kv_pages(self, rid: int) -> np.ndarray:
        n = C.c_int32()
        _check(load_library().tc_kv_pages(self._h, rid, None, 0, C.byref(n)))
        buf = np.zeros(max(1, n.value), dtype=np.int32)
        _check(load_library().tc_kv_pages(self._h, rid, buf.ctypes.data_as(C.POINTER(C.c_int32)), n.value,
                                          C.byref(n)))
        return buf[:n.value]

    def pool_info(self):
        base, pb, npg = C.c_void_p(), C.c_int64(), C.c_int64()
        _check(load_library().tc_kv_pool_info(self._h, C.byref(base), C.byref(pb), C.byref(npg)))
        return base.value, pb.value, npg.value

    def read_pages(self, pages: Sequence[int]) -> np.ndarray:
        """Raw bytes of whole KV pages (host copy) -> uint8 [n, page_bytes]."""
        base, pb, _ = self.pool_info()
        out = np.zeros((len(pages), pb), dtype=np.uint8)
        for i, p in enumerate(pages):
            _check(load_library().tc_read_device(out[i].ctypes.data_as(C.c_void_p), C.c_void_p(base + int(p) * pb), pb))
        return out

    def migrate_to(self, dst: "Instance", rid: int, n_tokens: int):
        _check(load_library().tc_kv_migrate(self._h, dst._h, rid, n_tokens))

    def migrate_wait(self):
        ms, nbytes = C.c_float(), C.c_int64()
        _check(load_library().tc_kv_migrate_wait(self._h, C.byref(ms), C.byref(nbytes)))
        return float(ms.value), int(nbytes.value)

    def migrate_async(self, dst: "Instance", rid: int, n_tokens: int) -> "MigrationEvent":
        """Asynchronous KV migration (tc_kv_migrate_async): returns at once; several may be in flight."""
        ev = C.c_void_p()
        _check(load_library().tc_kv_migrate_async(self._h, dst._h, rid, n_tokens, C.byref(ev)))
        return MigrationEvent(ev)

    def set_migration_ctas(self, ctas: int):
        _check(load_library().tc_set_migration_ctas(self._h, ctas))

    # ------------------------------------------------- cross-process migration (one process per GPU)
    def export_pool(self) -> dict:
        """IPC description of this instance's KV pool, picklable (send it to the pushing process)."""
        h = (C.c_uint8 * IPC_HANDLE_BYTES)()
        pb, npg = C.c_int64(), C.c_int64()
        _check(load_library().tc_kv_pool_export(self._h, C.cast(h, C.c_void_p), C.byref(pb), C.byref(npg)))
        return {"handle": bytes(h), "page_bytes": pb.value, "n_pages": npg.value, "device": self.device}

    def push_pages(self, remote: "RemotePool", src_pages: Sequence[int], dst_pages: Sequence[int]) -> "MigrationEvent":
        """Copy whole KV pages of this instance into another process's pool (tc_kv_push_pages):
        asynchronous, after this instance's in-flight step; NVLink P2P when the pool is on a peer GPU."""
        assert len(src_pages) == len(dst_pages)
        n = len(src_pages)
        sp = (C.c_int32 * max(n, 1))(*[int(x) for x in src_pages])
        dp = (C.c_int32 * max(n, 1))(*[int(x) for x in dst_pages])
        ev = C.c_void_p()
        _check(load_library().tc_kv_push_pages(self._h, remote._h, sp, dp, n, C.byref(ev)))
        return MigrationEvent(ev)

    # ---------------------------------------------------------------- weights / profiling
    def weight(self, name: str, dtype=np.uint16) -> np.ndarray:
        ptr, r, c = C.c_void_p(), C.c_int64(), C.c_int64()
        _check(load_library().tc_weight_ptr(self._h, name.encode(), C.byref(ptr), C.byref(r), C.byref(c)))
        out = np.zeros((r.value, c.value), dtype=dtype)
        _check(load_library().tc_read_device(out.ctypes.data_as(C.c_void_p), ptr, out.nbytes))
        return out

    def set_profiling(self, on: bool):
        _check(load_library().tc_set_profiling(self._h, 1 if on else 0))

    def phase_ms(self, phase: str) -> float:
        v = C.c_float()
        _check(load_library().tc_phase_ms(self._h, phase.encode(), C.byref(v)))
        return float(v.value)


class RemotePool:
    """Another process's KV pool mapped into this process (tc_kv_pool_import), on `device` -- the
    device of the instance that will push into it."""

    def __init__(self, exported: dict, device: int):
        h = C.create_string_buffer(bytes(exported["handle"]), IPC_HANDLE_BYTES)
        self._h = C.c_void_p()
        _check(load_library().tc_kv_pool_import(device, C.cast(h, C.c_void_p), exported["page_bytes"],
                                                exported["n_pages"], C.byref(self._h)))
        self.page_bytes, self.n_pages = exported["page_bytes"], exported["n_pages"]

    def close(self):
        if self._h is not None and self._h.value:
            _check(load_library().tc_remote_pool_close(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class MigrationEvent:
    """Completion handle of one asynchronous migration (tc_event)."""

    def __init__(self, h: C.c_void_p):
        self._h = h

    def done(self) -> bool:
        d = C.c_int32()
        _check(load_library().tc_event_query(self._h, C.byref(d)))
        return bool(d.value)

    def wait(self):
        """Blocks until the copy finished; returns (copy device ms, bytes)."""
        ms, nbytes = C.c_float(), C.c_int64()
        _check(load_library().tc_event_wait(self._h, C.byref(ms), C.byref(nbytes)))
        return float(ms.value), int(nbytes.value)

    def close(self):
        if self._h is not None and self._h.value:
            _check(load_library().tc_event_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def gemm(a, b, out, m, n, k, epilogue=0, bias=None, bn=0, k_splits=0, device=0, stream=None):
    """Kernel-level GEMM on device pointers (ints): out = epi(a[m,k] @ b[n,k]^T)."""
    _check(load_library().tc_gemm(device, C.c_void_p(a), C.c_void_p(b), C.c_void_p(out),
                                  C.c_void_p(bias) if bias else None, m, n, k, epilogue, bn, k_splits,
                                  C.c_void_p(stream) if stream else None))


def copy_pages(src_pool, dst_pool, src_pages_dev, dst_pages_dev, n_pages, page_bytes, stream=None):
    _check(load_library().tc_copy_pages(C.c_void_p(src_pool), C.c_void_p(dst_pool), C.c_void_p(src_pages_dev),
                                        C.c_void_p(dst_pages_dev), n_pages, page_bytes,
                                        C.c_void_p(stream) if stream else None))
