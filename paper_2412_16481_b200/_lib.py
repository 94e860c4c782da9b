"""ctypes binding of libf3d.so (include/f3d.h) and device-array plumbing.

The library is built in-tree by ``make -C paper_2412_16481_b200/csrc`` (or
``__graft_entry__.build()``).  There is no CPU fallback: if the shared
library or a CUDA device is missing, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

from .errors import (ConfigError, EmptyInputError, IntegrityError, NumericError,
                     RangeError)

_HERE = os.path.dirname(os.path.abspath(__file__))
# F3D_LIB_PATH: developer override (A/B builds of the same sources under tools/)
LIB_PATH = os.environ.get("F3D_LIB_PATH") or os.path.join(_HERE, "libf3d.so")

_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_INT = ctypes.c_int
_F64 = ctypes.c_double
_SZ = ctypes.c_size_t

# name -> (restype, argtypes); mirrors include/f3d.h
SIGNATURES = {
    "f3d_abi_version": (_INT, []),
    "f3d_last_error": (ctypes.c_char_p, []),
    "f3d_voxelize": (_INT, [_P, _I64, _P, _F64, _P, _P]),
    "f3d_remap_nonnegative": (_INT, [_P, _P, _I64, _I32, _P, _P, _P]),
    "f3d_hash_bucket": (_INT, [_P, _I64, _INT, _I32, _I64, _INT, _P, _P, _P, _P]),
    "f3d_morton_encode": (_INT, [_P, _I64, _INT, _P, _P, _P]),
    "f3d_voxel_hash": (_INT, [_P, _P, _I64, _I32, _P, _F64, _INT, _I32, _I64, _INT, _P, _P, _P,
                              _P, _P, _P]),
    "f3d_psh_workspace_size": (_SZ, [_I64, _I32, _I32]),
    "f3d_psh_assign": (_INT, [_P, _P, _P, _I64, _I32, _I32, _I32, _INT, _I64, _INT, _INT, _P,
                              _I32, _I32, _P, _P, _P, _P, _P, _P, _P, _SZ, _P, _P]),
    "f3d_psh_coords_workspace_size": (_SZ, [_I64, _I32]),
    "f3d_psh_assign_coords": (_INT, [_P, _I64, _P, _F64, _INT, _I32, _I32, _I64, _INT, _INT, _P,
                                     _I32, _I32, _P, _P, _P, _P, _P, _P, _P, _P, _SZ, _P, _P]),
    "f3d_validate_workspace_size": (_SZ, [_I64, _I64]),
    "f3d_validate_assignment": (_INT, [_P, _P, _P, _P, _P, _I64, _I32, _I32, _I32, _P, _P, _P]),
    "f3d_scatter_rows": (_INT, [_P, _P, _I64, _I64, _P, _P, _P]),
    "f3d_gather_rows": (_INT, [_P, _P, _I64, _I64, _P, _P, _P]),
    "f3d_scatter_rows_bf16_f32": (_INT, [_P, _I64, _P, _I64, _INT, _P, _I64, _P, _P]),
    "f3d_bswin_attention": (_INT, [_P, _P, _P, _I64, _I64, _I64, _P, _I64, _INT, _INT, _INT, _P,
                                   _P, _P, _P, _P, _P, _INT, _P, _INT, _INT, _P, _P, _P, _P]),
    "f3d_bswin_attention_tc": (_INT, [_P, _P, _P, _I64, _I64, _I64, _P, _I64, _INT, _INT, _INT,
                                      _P, _P, _P, _P, _P, _P, _INT, _P, _I64, _P, _I64, _P]),
    "f3d_attention_tc_qstep": (_INT, [_INT]),
    "f3d_plan_round": (_INT, [_P, _P, _INT, _INT, _INT, _INT, _INT, _INT, _INT, _P, _P, _P, _P, _P,
                              _P, _P, _INT, _INT, _P, _P]),
    "f3d_plan_rounds": (_INT, [_P, _P, _INT, _INT, _INT, _INT, _INT, _INT, _INT, _I64, _INT, _P,
                               _P, _P, _P, _P, _P, _P, _INT, _INT, _P, _P]),
    "f3d_plan_pool": (_INT, [_P, _P, _INT, _INT, _INT, _P, _P, _P, _P, _P]),
    "f3d_positional_encoding": (_INT, [_P, _I64, _INT, _F64, _INT, _P, _I64, _P]),
    "f3d_stage_pe": (_INT, [_P, _I64, _INT, _F64, _P, _INT, _P, _I64, _P]),
    "f3d_coord_bbox": (_INT, [_P, _I64, _P, _P, _P, _P]),
    "f3d_row_ln": (_INT, [_P, _INT, _I64, _P, _I64, _P, _P, _P, _P, _P, _F64, _P, _INT, _I64,
                          _I64, _INT, _F64, _P]),
    "f3d_gelu_f64": (_INT, [_P, _I64, _P, _P]),
    "f3d_pool_build": (_INT, [_P, _P, _P, _P, _INT, _INT, _P, _P, _P, _P, _P, _P, _P, _P]),
    "f3d_pool_reduce": (_INT, [_P, _INT, _I64, _INT, _P, _P, _I64, _INT, _INT, _P, _I64, _P, _P]),
    "f3d_bias_gelu": (_INT, [_P, _I64, _INT, _P, _P]),
    "f3d_pool_parent": (_INT, [_P, _P, _I64, _INT, _P, _P, _P]),
    "f3d_residual_out": (_INT, [_P, _I64, _P, _I64, _P, _P, _I64, _I64, _INT, _P]),
    "f3d_pool_reduce_res": (_INT, [_P, _I64, _P, _I64, _P, _INT, _P, _P, _I64, _INT, _INT, _P,
                                   _I64, _P, _P]),
    "f3d_scatter_ln_pe": (_INT, [_P, _INT, _I64, _P, _P, _P, _F64, _P, _P, _P, _I64, _P, _I64,
                                 _I64, _INT, _F64, _P, _P]),
    "f3d_gemm_supported": (_INT, [_INT, _INT]),
    "f3d_gemm": (_INT, [_P, _I64, _I64, _INT, _P, _INT, _P, _INT, _P, _I64, _P, _P]),
    "f3d_gemm_res_ln_supported": (_INT, [_INT, _INT]),
    "f3d_gemm_res_ln": (_INT, [_P, _I64, _I64, _INT, _P, _INT, _P, _P, _I64, _P, _P, _P, _P, _F64,
                               _F64, _P, _I64, _P, _P]),
    "f3d_ln_bwd": (_INT, [_P, _I64, _P, _INT, _I64, _P, _P, _I64, _P, _I64, _P, _P, _I64, _INT, _F64,
                          _P]),
    "f3d_gelu_bwd": (_INT, [_P, _I64, _P, _P, _I64, _P, _I64, _P, _I64, _INT, _P]),
    "f3d_colsum": (_INT, [_P, _INT, _I64, _I64, _INT, _P, _P]),
    "f3d_softmax_bwd": (_INT, [_P, _P, _P, _P, _INT, _INT, _F64, _F64, _INT, _P, _P]),
    "f3d_attn_bwd": (_INT, [_P, _P, _P, _P, _I64, _I64, _I64, _I64, _P, _I64, _P, _I64, _P, _I64,
                            _P, _I64, _P, _I64, _INT, _INT, _P, _P, _P, _P, _P, _INT, _INT, _P]),
}

_lib = None


def load():
    """Load libf3d.so and bind every declared symbol (raises if absent)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `make -C {os.path.join(_HERE, 'csrc')}` "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


_ERRS = {1: ConfigError, 2: RangeError, 3: IntegrityError, 5: EmptyInputError, 6: NumericError}


# kernels each entry point launches (for the bench's gpu_launches count)
KERNELS_PER_CALL = {
    "f3d_voxelize": 1, "f3d_remap_nonnegative": 3, "f3d_hash_bucket": 2, "f3d_morton_encode": 2,
    "f3d_voxel_hash": 3, "f3d_psh_assign": 2, "f3d_psh_assign_coords": 1, "f3d_validate_assignment": 5,
    "f3d_scatter_rows": 1, "f3d_gather_rows": 1, "f3d_scatter_rows_bf16_f32": 1, "f3d_bswin_attention": 1,
    "f3d_bswin_attention_tc": 1,
    "f3d_positional_encoding": 1, "f3d_stage_pe": 1, "f3d_coord_bbox": 2, "f3d_row_ln": 1,
    "f3d_gelu_f64": 1, "f3d_bias_gelu": 1, "f3d_pool_build": 2, "f3d_pool_reduce": 1, "f3d_pool_parent": 1, "f3d_gemm": 1, "f3d_gemm_res_ln": 1, "f3d_scatter_ln_pe": 1, "f3d_pool_reduce_res": 1, "f3d_residual_out": 1, "f3d_ln_bwd": 1, "f3d_gelu_bwd": 1, "f3d_colsum": 1,
    "f3d_softmax_bwd": 1, "f3d_attn_bwd": 2,
    "f3d_plan_round": 1, "f3d_plan_rounds": 1, "f3d_plan_pool": 1,
}


class Probe:
    """Optional instrumentation used by bench.py: counts launches and records
    CUDA events around every entry point on the launching stream."""

    active = None

    def __init__(self, events: bool = True):
        self.launches = 0
        self.events = events
        self.records = []   # (name, start_event, end_event)

    def __enter__(self):
        Probe.active = self
        return self

    def __exit__(self, *exc):
        Probe.active = None

    def totals_ms(self):
        torch.cuda.synchronize()
        out = {}
        for name, a, b in self.records:
            out[name] = out.get(name, 0.0) + a.elapsed_time(b)
        return out


class Recorder:
    """Optional instrumentation used by bench.py: keeps (name, args) of every
    entry point called while active (e.g. during a CUDA-graph capture, whose
    buffers stay alive with the graph), so a family of launches can be
    re-issued alone -- in its own graph, on one stream -- and timed with CUDA
    events (``replay_calls``).  The last argument of every entry point that
    launches work is its stream."""

    active = None

    def __init__(self):
        self.calls = []
        # every tensor handed to an entry point while recording stays alive, so
        # no buffer of a recorded call is reused by a later allocation of the
        # capture: any family of recorded calls can then be re-issued alone
        self.keep = []

    def __enter__(self):
        self._prev, Recorder.active = Recorder.active, self
        return self

    def __exit__(self, *exc):
        Recorder.active = self._prev

    def launches(self):
        return sum(KERNELS_PER_CALL.get(n, 0) for n, _ in self.calls)


def replay_calls(calls, stream_ptr):
    """Re-issue recorded entry-point calls with their stream replaced."""
    lib = load()
    for name, args in calls:
        st = getattr(lib, name)(*args[:-1], stream_ptr)
        if st != 0:
            raise RuntimeError(f"replay of {name} failed (status {st})")


def call(name, *args):
    """Invoke an f3d_* entry point and map a non-zero status to the
    reference exception classes (bw/errors.py)."""
    rec = Recorder.active
    if rec is not None and torch.cuda.is_current_stream_capturing():
        rec.calls.append((name, args))
    pr = Probe.active
    if pr is not None:
        pr.launches += KERNELS_PER_CALL.get(name, 0)
        if pr.events:
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
    st = getattr(load(), name)(*args)
    if pr is not None and pr.events:
        e1.record()
        pr.records.append((name, e0, e1))
    if st != 0:
        msg = load().f3d_last_error().decode(errors="replace")
        if st == 4:
            raise RuntimeError(f"{name}: {msg}")
        raise _ERRS.get(st, RuntimeError)(f"{name} failed (status {st}) {msg}".strip())
    return st


# ------------------------------------------------------------ device plumbing

def device():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2412_16481_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def stream():
    return _P(torch.cuda.current_stream().cuda_stream)


def ptr(t):
    if t is None:
        return None
    rec = Recorder.active
    if rec is not None:
        rec.keep.append(t)
    return _P(t.data_ptr())


def is_host(x) -> bool:
    """True when the caller passed host data (numpy / lists / CPU tensors):
    results are then handed back as numpy, like the reference."""
    return not (isinstance(x, torch.Tensor) and x.is_cuda)


def to_dev(x, dtype) -> torch.Tensor:
    """Any array-like -> contiguous CUDA tensor of dtype."""
    if isinstance(x, torch.Tensor):
        return x.to(device=device(), dtype=dtype).contiguous()
    arr = np.asarray(x)
    return torch.from_numpy(np.ascontiguousarray(arr)).to(device=device(), dtype=dtype)


def out(t: torch.Tensor, host: bool):
    return t.cpu().numpy() if host else t


def empty(shape, dtype):
    return torch.empty(shape, dtype=dtype, device=device())


class _Uploader:
    """Packs many small int32 host arrays into one pinned staging buffer and
    issues a single non-blocking H2D copy on the current stream (plans are
    rebuilt once per stage; a blocking pageable copy per array would drain the
    stream each time)."""

    def __init__(self):
        self.host = None
        self.event = None

    def __call__(self, arrays):
        items = [(k, np.ascontiguousarray(v, dtype=np.int32)) for k, v in arrays.items()]
        total = 0
        spans = []
        for k, a in items:
            spans.append((k, total, a))
            total += (a.size + 3) & ~3          # 16-byte aligned slices
        total = max(total, 4)
        if self.event is not None:
            self.event.synchronize()
        if self.host is None or self.host.numel() < total:
            self.host = torch.empty(max(total, 1 << 20), dtype=torch.int32).pin_memory()
        hv = self.host.numpy()
        for k, o, a in spans:
            hv[o:o + a.size] = a.ravel()
        dev = torch.empty(total, dtype=torch.int32, device=device())
        dev.copy_(self.host[:total], non_blocking=True)
        self.event = torch.cuda.Event()
        self.event.record()
        return {k: dev[o:o + a.size].view(a.shape) for k, o, a in spans}


upload = _Uploader()
