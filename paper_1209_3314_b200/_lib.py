"""ctypes binding of libiwpp_b200.so (the C ABI in include/iwpp_b200.h).

There is no CPU fallback: if the shared object is missing or no CUDA
device is visible, every operator raises ``RuntimeError``.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from .errors import ContractViolation, EngineError, NoBackgroundError

HERE = os.path.dirname(os.path.abspath(__file__))
# IWPP_B200_LIB: load another build (development: compile-time variants)
LIB_PATH = os.environ.get("IWPP_B200_LIB") or os.path.join(HERE, "libiwpp_b200.so")

IWPP_OK = 0
IWPP_E_CONTRACT = -1
IWPP_E_NO_BACKGROUND = -2
IWPP_E_ENGINE_LIMIT = -3
IWPP_E_CUDA = -4
IWPP_E_WORKSPACE = -5
IWPP_E_OVERFLOW = -6

# every symbol the header declares (checked by tests/test_capi.py)
EXPORTS = (
    "iwpp_last_error", "iwpp_version", "iwpp_device_info",
    "iwpp_recon_workspace_bytes", "iwpp_recon", "iwpp_recon_host_workspace_bytes",
    "iwpp_recon_host", "iwpp_recon_engine_counters", "iwpp_check_le", "iwpp_edt_set_engine",
    "iwpp_recon_sweep_rows", "iwpp_recon_sweep_cols",
    "iwpp_recon_seed_scan", "iwpp_recon_pass_workspace_bytes", "iwpp_recon_pass",
    "iwpp_edt_workspace_bytes", "iwpp_edt", "iwpp_edt_propagate",
    "iwpp_edt_finalize", "iwpp_edt_host_workspace_bytes", "iwpp_edt_host",
    "iwpp_event_create", "iwpp_event_destroy", "iwpp_event_record", "iwpp_event_elapsed_ms",
    "iwpp_edt_slab_workspace_bytes", "iwpp_edt_slab_init", "iwpp_edt_slab_round",
    "iwpp_edt_slab_finalize", "iwpp_pgm_decode", "iwpp_pgm_encode", "iwpp_gen_marker",
    "iwpp_quantize_u8", "iwpp_edt_init_workspace_bytes", "iwpp_edt_init",
    "iwpp_edt_exact_workspace_bytes", "iwpp_edt_exact", "iwpp_debug_atrace",
    "iwpp_edt_mg_workspace_bytes", "iwpp_edt_mg_mailbox_bytes", "iwpp_edt_mg_init", "iwpp_edt_mg_run",
)


class Stats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in (
        "rounds", "executions", "overflow_count", "queued_total", "seeds",
        "tiles_processed", "tile_reruns", "contract_violations", "n_inf")]

    def as_dict(self) -> dict:
        return {n: int(getattr(self, n)) for n, _ in self._fields_}


class MgSlab(ctypes.Structure):
    """iwpp_edt_mg_slab (include/iwpp_b200.h)."""
    _fields_ = [("workspace", ctypes.c_void_p), ("W", ctypes.c_int64), ("h", ctypes.c_int64),
                ("y0", ctypes.c_int64), ("H", ctypes.c_int64), ("has_up", ctypes.c_int),
                ("has_down", ctypes.c_int), ("rank", ctypes.c_int), ("world", ctypes.c_int),
                ("mailbox", ctypes.c_void_p * 16)]


class ReconOpts(ctypes.Structure):
    _fields_ = [("sweeps", ctypes.c_int), ("max_blocks", ctypes.c_int),
                ("check_contract", ctypes.c_int), ("queue_capacity", ctypes.c_int),
                ("tile_sweeps", ctypes.c_int), ("halo_sweep_threshold", ctypes.c_int),
                ("ev_begin", ctypes.c_void_p), ("ev_end", ctypes.c_void_p),
                ("slab_rows", ctypes.c_int), ("pipeline_rows", ctypes.c_int), ("engine", ctypes.c_int),
                ("max_rounds", ctypes.c_int), ("marker", ctypes.c_void_p)]


_lib = None
_lock = threading.Lock()


def load_library(path: str = LIB_PATH):
    """Load and prototype the library without touching the GPU."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise RuntimeError(
                f"libiwpp_b200.so not built ({path}); run __graft_entry__.build() "
                "or python -m paper_1209_3314_b200.build")
        L = ctypes.CDLL(path)
        P, I64, I, SZ = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_size_t
        SP = ctypes.POINTER(Stats)
        OP = ctypes.POINTER(ReconOpts)
        proto = {
            "iwpp_last_error": ([], ctypes.c_char_p),
            "iwpp_version": ([], ctypes.c_char_p),
            "iwpp_device_info": ([I, ctypes.POINTER(I), ctypes.POINTER(I), ctypes.POINTER(I)], I),
            "iwpp_recon_workspace_bytes": ([I64, I64, I, I], SZ),
            "iwpp_recon": ([P, P, I64, I64, I, I, P, SZ, OP, SP, P], I),
            "iwpp_recon_host_workspace_bytes": ([I64, I64, I, I], SZ),
            "iwpp_recon_host": ([P, P, P, I64, I64, I, I, P, SZ, OP, SP, P], I),
            "iwpp_recon_engine_counters": ([P, I64, I64, ctypes.POINTER(ctypes.c_uint64), I, P], I),
            "iwpp_check_le": ([P, P, I64, I, P, ctypes.POINTER(I64), P], I),
            "iwpp_recon_sweep_rows": ([P, P, I64, I64, I, P], I),
            "iwpp_recon_sweep_cols": ([P, P, I64, I64, I, P, P], I),
            "iwpp_recon_seed_scan": ([P, P, I64, I64, I, I, P, ctypes.POINTER(I64), P, P], I),
            "iwpp_recon_pass_workspace_bytes": ([I64, I64, I], ctypes.c_size_t),
            "iwpp_recon_pass": ([P, P, I64, I64, I, I, I, P, ctypes.POINTER(I64),
                                 ctypes.POINTER(I), P, P], I),
            "iwpp_edt_workspace_bytes": ([I64, I64, I], SZ),
            "iwpp_edt": ([P, I64, I64, I, P, P, P, SZ, I64, SP, P], I),
            "iwpp_edt_propagate": ([P, I64, I64, I, P, I64, P, SZ, I64, SP, P], I),
            "iwpp_edt_finalize": ([P, I64, I64, P, P, P, P], I),
            "iwpp_edt_set_engine": ([I], I),
            "iwpp_edt_host_workspace_bytes": ([I64, I64, I], SZ),
            "iwpp_edt_host": ([P, I64, I64, I, P, P, P, SZ, I64, SP, P], I),
            "iwpp_event_create": ([ctypes.POINTER(P)], I),
            "iwpp_event_destroy": ([P], I),
            "iwpp_event_record": ([P, P], I),
            "iwpp_event_elapsed_ms": ([P, P, ctypes.POINTER(ctypes.c_float)], I),
            "iwpp_edt_slab_workspace_bytes": ([I64, I64], SZ),
            "iwpp_edt_slab_init": ([P, I64, I64, I64, I64, I, I, I, P, P, P, P], I),
            "iwpp_edt_slab_round": ([P, I64, I64, I64, I, I64, P, P, P, P,
                                     ctypes.POINTER(I64), P], I),
            "iwpp_edt_slab_finalize": ([P, I64, I64, I64, I64, P, P, P], I),
            "iwpp_pgm_decode": ([P, P, I64, I, I, P, ctypes.POINTER(I64), P], I),
            "iwpp_pgm_encode": ([P, P, I64, I, P], I),
            "iwpp_gen_marker": ([P, P, I64, I, ctypes.c_double, P], I),
            "iwpp_quantize_u8": ([P, P, I64, P], I),
            "iwpp_edt_init_workspace_bytes": ([I64, I64], SZ),
            "iwpp_edt_init": ([P, I64, I64, I, P, P, ctypes.POINTER(I64), P, SZ, P], I),
            "iwpp_edt_exact_workspace_bytes": ([I64, I64], SZ),
            "iwpp_edt_exact": ([P, I64, I64, P, P, P, SZ, P], I),
            "iwpp_debug_atrace": ([P, ctypes.c_uint32, ctypes.POINTER(ctypes.c_uint32)], I),
            "iwpp_edt_mg_workspace_bytes": ([I64, I64], SZ),
            "iwpp_edt_mg_mailbox_bytes": ([I64], SZ),
            "iwpp_edt_mg_init": ([P, I64, I64, I64, I64, I, I, I, P, P, P, P], I),
            "iwpp_edt_mg_run": ([ctypes.POINTER(MgSlab), I, I, I64, ctypes.POINTER(I64), P], I),
        }
        for name, (args, res) in proto.items():
            if os.environ.get("IWPP_B200_LIB") and not hasattr(L, name):
                continue  # (development: an older build under A/B lacks newer entry points)
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
        return L


def lib():
    """The library, with a CUDA device required (fails loudly otherwise)."""
    L = load_library()
    torch = _torch()
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1209_3314_b200 needs a CUDA device (B200, sm_100a); none visible")
    return L


def _torch():
    import torch
    return torch


def check(rc: int, what: str = ""):
    if rc == IWPP_OK:
        return
    msg = _lib.iwpp_last_error().decode(errors="replace") if _lib else ""
    msg = f"{what}: {msg}" if what else msg
    if rc == IWPP_E_CONTRACT:
        raise ContractViolation(msg)
    if rc == IWPP_E_NO_BACKGROUND:
        raise NoBackgroundError(msg)
    if rc == IWPP_E_ENGINE_LIMIT:
        raise EngineError(msg)
    raise RuntimeError(f"iwpp error {rc}: {msg}")


# -- workspace cache: one growable device buffer per (device, stream) ------
_ws = {}
_ws_lock = threading.Lock()


def workspace(nbytes: int):
    """A device byte buffer of at least nbytes on the current device, private
    to torch's current stream there.  Calls on one stream are ordered, so they
    share it safely; calls on different streams (e.g. from several host
    threads, SURVEY 8(b) "Threading") get different buffers.  A buffer that
    is replaced by a larger one is released to torch's caching allocator,
    which reuses it only in that stream's order."""
    torch = _torch()
    dev = torch.cuda.current_device()
    key = (dev, torch.cuda.current_stream(dev).cuda_stream)
    with _ws_lock:
        buf = _ws.get(key)
        if buf is None or buf.numel() < nbytes:
            buf = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=f"cuda:{dev}")
            _ws[key] = buf
        return buf


def stream_ptr():
    return ctypes.c_void_p(_torch().cuda.current_stream().cuda_stream)


class Event:
    """A CUDA event owned by libiwpp_b200 (same runtime as its kernels)."""

    def __init__(self):
        L = lib()
        h = ctypes.c_void_p()
        check(L.iwpp_event_create(ctypes.byref(h)), "event_create")
        self.handle = h

    def record(self, stream=None):
        check(lib().iwpp_event_record(self.handle, stream if stream is not None else stream_ptr()))

    def elapsed_ms(self, end: "Event") -> float:
        ms = ctypes.c_float()
        check(lib().iwpp_event_elapsed_ms(self.handle, end.handle, ctypes.byref(ms)))
        return float(ms.value)

    def __del__(self):
        try:
            if _lib is not None and self.handle:
                _lib.iwpp_event_destroy(self.handle)
        except Exception:
            pass


def ptr(a):
    """Raw pointer of a numpy array or torch tensor."""
    if isinstance(a, np.ndarray):
        return ctypes.c_void_p(a.ctypes.data)
    return ctypes.c_void_p(a.data_ptr())


def device_of(*arrays):
    """``with device_of(t, ...)``: run the call on the device of the CUDA
    tensors among ``arrays`` (all must share it), so kernels launch on the
    device that owns the pointers and pick that device's workspace and
    current stream.  Host arrays impose nothing; with no tensor at all the
    current device is used."""
    import contextlib
    torch = _torch()
    devs = {a.device for a in arrays if isinstance(a, torch.Tensor)}
    if len(devs) > 1:
        raise ContractViolation(f"arrays live on different devices: {sorted(map(str, devs))}")
    if not devs:
        return contextlib.nullcontext()
    (d,) = devs
    if d.type != "cuda":
        raise ContractViolation(f"tensor on {d}; the B200 engines need CUDA tensors or numpy arrays")
    return torch.cuda.device(d)
