"""ctypes binding of ``libfastcdf_b200.so`` (declared in include/fastcdf_b200.h) plus the torch
plumbing: device tensors, the caller's CUDA stream, workspace allocation and status mapping.

There is no CPU fallback: if the library or a CUDA device is missing, every entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import numpy as np

from .core import OverflowGuardError, ParameterError, ShapeError

_HERE = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ["FCG_LIB_PATH"]) if os.environ.get("FCG_LIB_PATH") else _HERE / "libfastcdf_b200.so"  # dev A/B override
ABI_VERSION = 1

FCG_OK = 0
FCG_EINVAL = 22
FCG_EUNSUPPORTED = 95
FCG_ERANGE = 34
FCG_ECUDA = 100
FCG_EWORKSPACE = 101

LAT_I32 = 0
LAT_F64 = 1

_P = C.c_void_p
_I64 = C.c_int64
_I32 = C.c_int32
_SZP = C.POINTER(C.c_size_t)

_SIGS = {
    "fcg_abi_version": ([], C.c_int),
    "fcg_last_error": ([], C.c_char_p),
    "fcg_device_sm_count": ([], C.c_int),
    "fcg_profile_enable": ([C.c_int], C.c_int),
    "fcg_profile_report": ([C.c_char_p, C.c_size_t], C.c_int),
    "fcg_profile_launches": ([], C.c_int64),
    "fcg_local_sums": ([_P, _I64, _I32, _P, _P, _P, _P, _I32, _P, _P, _SZP, _P], C.c_int),
    "fcg_directional_sweep": ([_P, _I32, _I32, _P, _P, _P, _SZP, _P], C.c_int),
    "fcg_ecdf_grid": ([_P, _I64, _I32, _P, _P, _P, _P, _I32, _I32, _I32, _P, _P, _SZP, _P], C.c_int),
    "fcg_minmax": ([_P, _I64, _I32, _P, _P, _SZP, _P], C.c_int),
    "fcg_kde_grid_laplacian": ([_P, _I64, _I32, _P, _P, _P, _P, _P, _P, _P, _SZP, _P], C.c_int),
    "fcg_kde_grid_matern32": ([_P, _I64, _I32, _P, _P, _P, _P, _P, _P, _P, _SZP, _P], C.c_int),
    "fcg_multilinear_interp": ([_P, _P, _I32, _P, _P, _I64, _P, _P, _P, _SZP, _P], C.c_int),
    "fcg_rank_f64": ([_P, _I64, _I64, _P, _P, _P, _P, _P, _P, _SZP, _P], C.c_int),
    "fcg_distinct": ([_P, _I64, _I32, _P, _P, _SZP, _P], C.c_int),
    "fcg_ecdf_points": ([_P, _I64, _I32, _P, _P, _I32, _I32, _P, _P, _SZP, _P], C.c_int),
    "fcg_ecdf_esf_points": ([_P, _I64, _I32, _P, _P, _I32, _P, _P, _P, _SZP, _P], C.c_int),
    "fcg_dnc_ecdf": ([_P, _I64, _I32, _P, _I32, _I32, _P, _P, _SZP, _P], C.c_int),
    "fcg_kde_points_laplacian": ([_P, _I64, _I32, _P, _I32, _P, _P, _P, _P, _SZP, _P], C.c_int),
    "fcg_kde_points_matern32": ([_P, _I64, _I32, _P, _P, _P, _P, _P, _SZP, _P], C.c_int),
    "fcg_kde_points_laplacian_w2": ([_P, _I64, _I32, _P, _P, _I32, _P, _P, _P, _P, _SZP, _P],
                                    C.c_int),
    "fcg_dominance_terms": ([_P, _I64, _I32, _P, _P, _P, _SZP, _P], C.c_int),
    "fcg_kde_points_laplacian_shard": ([_P, _I64, _I32, _P, _I32, _P, _P, _I32, _I32, _P, _P, _SZP,
                                        _P], C.c_int),
    "fcg_dnc_ecdf_shard": ([_P, _I64, _I32, _P, _I32, _I32, _I32, _I32, _P, _P, _SZP, _P], C.c_int),
    "fcg_copy_h2d": ([_P, _P, C.c_size_t, _P], C.c_int),
    "fcg_copy_d2h": ([_P, _P, C.c_size_t, _P], C.c_int),
    "fcg_axis_owner": ([_P, _I64, _I32, _I32, _P, _I64, _I32, _I32, _P, _I32, _P, _P], C.c_int),
    "fcg_partition_rows": ([_P, _I64, _I32, _P, _P, _I32, _P, _P, _P, _P, _SZP, _P], C.c_int),
    "fcg_slab_finish": ([_P, _I32, _P, _I64, _I64, _I64, C.c_double, _P, _P], C.c_int),
    "fcg_kde_grid_laplacian_ex": ([_P, _I64, _I32, _P, _P, _P, _P, _P, C.c_double, C.c_double,
                                   _P, _P, _P, _SZP, _P], C.c_int),
    "fcg_kde_carry_fixup": ([_P, _I32, _P, _P, _P, _P, _P, C.c_double, _P, _SZP, _P], C.c_int),
}

EXPORTED = tuple(_SIGS)

_lock = threading.Lock()
_lib = None


def load_library(path: Path | str | None = None, require_all: bool = True):
    """Load and type the shared library (no GPU needed)."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path) if path is not None else LIB_PATH
        if not p.exists():
            raise RuntimeError(
                f"{p.name} is not built; run `python -m paper_2005_03246_b200._build` "
                "(the GPU path has no CPU fallback)")
        lib = C.CDLL(str(p))
        for name, (args, res) in _SIGS.items():
            fn = getattr(lib, name, None)
            if fn is None:
                if require_all:
                    raise RuntimeError(f"{p.name} does not export {name}")
                continue
            fn.argtypes = args
            fn.restype = res
        if lib.fcg_abi_version() != ABI_VERSION:
            raise RuntimeError("ABI version mismatch between Python host and libfastcdf_b200.so")
        if path is None:
            _lib = lib
        return lib


_torch_ok = None


def _torch():
    global _torch_ok
    if _torch_ok is not None:
        return _torch_ok
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_2005_03246_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    _torch_ok = torch
    return torch


def device():
    torch = _torch()
    return torch.device("cuda", torch.cuda.current_device())


def _raw_stream(torch, dev: int) -> int:
    """The current CUDA stream of device `dev` as an integer handle (the cheap accessor when
    this torch build has it: current_stream() builds a Stream object per call)."""
    f = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    return f(dev) if f is not None else torch.cuda.current_stream(dev).cuda_stream


def stream_handle():
    torch = _torch()
    return C.c_void_p(_raw_stream(torch, torch.cuda.current_device()))


def ptr(t) -> C.c_void_p:
    return C.c_void_p(0 if t is None else t.data_ptr())


def check(rc: int, name: str):
    if rc == FCG_OK:
        return
    msg = load_library().fcg_last_error().decode(errors="replace")
    if rc in (FCG_EINVAL, FCG_EUNSUPPORTED):
        raise ParameterError(f"{name}: {msg}")
    if rc == FCG_ERANGE:
        raise OverflowGuardError(msg)
    raise RuntimeError(f"{name} failed (status {rc}): {msg}")


def call_ws(name: str, *args):
    """Two-phase workspace call: size query, torch allocation (the caching allocator, so the
    buffer is stream-ordered), real call on the current stream."""
    torch = _torch()
    lib = _lib if _lib is not None else load_library()
    fn = getattr(lib, name)
    dev = torch.cuda.current_device()
    raw = _raw_stream(torch, dev)
    sh = C.c_void_p(raw)
    nbytes = C.c_size_t(0)
    check(fn(*args, None, C.byref(nbytes), sh), name)
    need = max(int(nbytes.value), 1)
    key = (threading.get_ident(), dev, raw)
    ws = _ws_cache.get(key)
    if ws is None or ws.numel() < need:
        ws = torch.empty(need, dtype=torch.uint8, device=torch.device("cuda", dev))
        if need <= _WS_CACHE_MAX:
            _ws_cache[key] = ws
    check(fn(*args, C.c_void_p(ws.data_ptr()), C.byref(nbytes), sh), name)
    return ws


# Small workspaces are reused per (host thread, stream): one thread's calls on one stream are
# issued in order, so the next call's kernels only touch the scratch after the previous call's
# kernels are done (threads sharing a stream get separate buffers); launch-bound
# configurations otherwise pay an allocator round trip per call.  Large ones go back to torch's
# caching allocator so the memory stays available to other tensors.
_ws_cache: dict = {}
_WS_CACHE_MAX = 64 << 20


def i64_array(vals) -> C.Array:
    arr = (C.c_int64 * len(vals))(*[int(v) for v in vals])
    return arr


def i32_array(vals) -> C.Array:
    return (C.c_int32 * len(vals))(*[int(v) for v in vals])


def f64_array(vals) -> C.Array:
    return (C.c_double * len(vals))(*[float(v) for v in vals])


# ---- tensors ---------------------------------------------------------------------------

def is_torch(a) -> bool:
    return type(a).__module__.startswith("torch")


def to_device_f64(a):
    """numpy / array-like / torch -> contiguous fp64 CUDA tensor."""
    torch = _torch()
    if is_torch(a):
        t = a
        if t.device.type != "cuda":
            t = t.to(device(), non_blocking=True)
        elif t.device.index != torch.cuda.current_device():
            # kernels launch on the current device's stream with workspace allocated there
            raise ParameterError(
                f"tensor is on {t.device} but the current CUDA device is "
                f"cuda:{torch.cuda.current_device()}; call under torch.cuda.device({t.device})")
        return t.to(torch.float64).contiguous()
    arr = np.ascontiguousarray(a, dtype=np.float64)
    if arr.nbytes >= _STAGED_MIN:  # large uploads: pinned ring + threaded staging
        t = torch.empty(arr.shape, dtype=torch.float64, device=device())
        lib = _lib if _lib is not None else load_library()
        check(lib.fcg_copy_h2d(C.c_void_p(t.data_ptr()), arr.ctypes.data_as(C.c_void_p),
                               arr.nbytes, stream_handle()), "fcg_copy_h2d")
        return t
    return torch.from_numpy(arr).to(device(), non_blocking=True)


_STAGED_MIN = 8 << 20


def to_host(t) -> np.ndarray:
    """Device tensor -> freshly allocated numpy array (staged and threaded when large)."""
    if t.device.type != "cuda":
        return t.numpy()
    torch = _torch()
    dt = {torch.float64: np.float64, torch.int64: np.int64, torch.int32: np.int32}.get(t.dtype)
    if (dt is None or not t.is_contiguous()
            or t.numel() * t.element_size() < _STAGED_MIN):
        return t.cpu().numpy()
    out = np.empty(tuple(t.shape), dtype=dt)
    lib = _lib if _lib is not None else load_library()
    with _torch().cuda.device(t.device):
        check(lib.fcg_copy_d2h(out.ctypes.data_as(C.c_void_p), C.c_void_p(t.data_ptr()),
                               out.nbytes, stream_handle()), "fcg_copy_d2h")
    return out


def device_knots(grid):
    """Concatenated knot vectors of a grid on the device (cached on our own grid objects)."""
    torch = _torch()
    dev = device()
    cache = getattr(grid, "__dict__", {}).get("_fcg_knots")
    if cache is not None and cache.device == dev:
        return cache
    flat = np.concatenate([np.ascontiguousarray(z, dtype=np.float64).reshape(-1)
                           for z in grid.knots])
    t = torch.from_numpy(flat).to(dev)
    try:
        object.__setattr__(grid, "_fcg_knots", t)
    except (AttributeError, TypeError):
        pass
    return t


def distinct_flags(points) -> tuple:
    """Pairwise-distinct flag per dimension, computed on the device (syncs)."""
    pts = to_device_f64(points)
    if pts.dim() == 1:
        pts = pts.reshape(-1, 1)
    n, d = pts.shape
    flags = (C.c_int32 * d)()
    call_ws("fcg_distinct", ptr(pts), n, d, flags)
    return tuple(bool(v) for v in flags)


def minmax(points):
    """Per-dimension (min, max) host arrays from a device reduction (syncs)."""
    torch = _torch()
    pts = to_device_f64(points)
    n, d = pts.shape
    out = torch.empty(2 * d, dtype=torch.float64, device=pts.device)
    call_ws("fcg_minmax", ptr(pts), n, d, ptr(out))
    mm = out.cpu().numpy()
    return mm[:d].copy(), mm[d:].copy()


def profile_enable(on: bool = True):
    load_library().fcg_profile_enable(1 if on else 0)


def profile_report() -> dict:
    """{kernel label: (launches, total_ms)} since the last report (synchronises)."""
    lib = load_library()
    cap = 1 << 16
    buf = C.create_string_buffer(cap)
    nb = lib.fcg_profile_report(buf, cap)
    if nb < 0:
        raise RuntimeError("fcg_profile_report failed")
    out = {}
    for line in buf.value.decode().splitlines():
        name, cnt, ms = line.split()
        out[name] = (int(cnt), float(ms))
    return out


def check_rows(points, d: int):
    if points.shape[1] != d:
        raise ShapeError(f"expected {d} columns, got {points.shape[1]}")


def rank_f64(keys):
    """Device ranking of one fp64 key vector (``fcg_rank_f64``, subsystem 1): returns the int32
    CUDA tensors (order, pos, lower, upper, dense) — stable argsort, its inverse, #keys < key,
    #keys <= key and #distinct keys < key (-0.0 and +0.0 rank equal)."""
    torch = _torch()
    k = to_device_f64(keys).reshape(-1)
    n = k.numel()
    outs = [torch.empty(n, dtype=torch.int32, device=k.device) for _ in range(5)]
    call_ws("fcg_rank_f64", ptr(k), n, 1, *[ptr(o) for o in outs])
    return tuple(outs)
