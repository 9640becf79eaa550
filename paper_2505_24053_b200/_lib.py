"""ctypes binding of libgeer_b200.so (the C ABI declared in include/geer.h).

The library is built in-tree (``python -m paper_2505_24053_b200.build``) and
loaded from this package directory.  There is no fallback: if the shared
object is missing or a CUDA device is unavailable, calls raise.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libgeer_b200.so")

GEER_OK = 0
GEER_ERR_INVALID = 1
GEER_ERR_NOT_SYMMETRIC = 2
GEER_ERR_NOT_PD = 3
GEER_ERR_CUDA = 4
GEER_ERR_NOMEM = 5
GEER_ERR_STATE = 6
GEER_ERR_OVERFLOW = 7

MODEL_IDS = {"pinhole": 0, "kb": 1, "beap": 2}

# every symbol include/geer.h declares (checked by tests/test_abi.py)
EXPORTED = (
    "geer_abi_version", "geer_last_error", "geer_create", "geer_destroy", "geer_set_timing", "geer_forward",
    "geer_backward", "geer_frame_stats", "geer_graph_info", "geer_graph_export", "geer_build_graph_host",
    "geer_render_host", "geer_render_backward_host", "geer_l1_grad", "geer_adam", "geer_measure_fp32_peak",
    "geer_loss_workspace_bytes", "geer_loss", "geer_resample_to_beap", "geer_ply_to_soa",
    "geer_association_check", "geer_sync", "geer_clear_camera_cache", "geer_workspace_bytes",
    "geer_set_workspace", "geer_workspace_used", "geer_debug_n_eval",
    "geer_last_h2d_bytes",
)


class GeerCamera(ctypes.Structure):
    _fields_ = [
        ("width", ctypes.c_int32), ("height", ctypes.c_int32), ("model", ctypes.c_int32), ("pad_", ctypes.c_int32),
        ("rotation", ctypes.c_double * 9), ("translation", ctypes.c_double * 3),
        ("fov_x", ctypes.c_double), ("fov_y", ctypes.c_double),
        ("fx", ctypes.c_double), ("fy", ctypes.c_double), ("cx", ctypes.c_double), ("cy", ctypes.c_double),
        ("k", ctypes.c_double * 4),
    ]


class GeerConfig(ctypes.Structure):
    _fields_ = [
        ("lam", ctypes.c_double), ("background", ctypes.c_double * 3), ("tile_px", ctypes.c_int32),
        ("support_cutoff", ctypes.c_int32), ("threads", ctypes.c_int32), ("flags", ctypes.c_int32),
    ]


class GeerScene(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int64), ("n_bands", ctypes.c_int32), ("pad_", ctypes.c_int32),
        ("means", ctypes.c_void_p), ("log_scales", ctypes.c_void_p), ("quats", ctypes.c_void_p),
        ("opacity_logits", ctypes.c_void_p), ("sh", ctypes.c_void_p),
    ]


class GeerGrads(ctypes.Structure):
    _fields_ = [("dmeans", ctypes.c_void_p), ("dlog_scales", ctypes.c_void_p), ("dquats", ctypes.c_void_p),
                ("dopacities", ctypes.c_void_p), ("dsh", ctypes.c_void_p)]


GeerHostScene = GeerScene  # same layout, double pointers
GeerHostGrads = GeerGrads


class GeerStats(ctypes.Structure):
    _fields_ = [
        ("n_gaussians", ctypes.c_int64), ("n_entries", ctypes.c_int64), ("n_tiles", ctypes.c_int64),
        ("n_work_items", ctypes.c_int64), ("evaluated_pairs", ctypes.c_int64), ("kappa_rechecks", ctypes.c_int64),
        ("fixup_pixels", ctypes.c_int64),
        ("clamped", ctypes.c_int64), ("warp_entries", ctypes.c_int64), ("streamed_entries", ctypes.c_int64),
        ("ms_prep", ctypes.c_float), ("ms_dup", ctypes.c_float), ("ms_sort", ctypes.c_float),
        ("ms_render", ctypes.c_float), ("ms_total", ctypes.c_float), ("ms_backward", ctypes.c_float),
    ]

    def as_dict(self):
        return {name: getattr(self, name) for name, _ in self._fields_}


class GeerError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


_lib = None
_lock = threading.Lock()


def load():
    """Load libgeer_b200.so; raises ImportError (never falls back) if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is not built; run `python -m paper_2505_24053_b200.build` "
                              "(there is no CPU fallback for the render path)")
        lib = ctypes.CDLL(LIB_PATH)
        P, I, I64, F, D = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_float, ctypes.c_double
        sig = {
            "geer_abi_version": ([], I),
            "geer_last_error": ([], ctypes.c_char_p),
            "geer_create": ([I], P),
            "geer_destroy": ([P], None),
            "geer_set_timing": ([P, I], I),
            "geer_forward": ([P, P, P, P, P, P, P, P], I),
            "geer_backward": ([P, P, P, I, P], I),
            "geer_frame_stats": ([P, P], I),
            "geer_graph_info": ([P, P, P, P], I),
            "geer_graph_export": ([P, P, P, P, P, P, P, P, P, P, P], I),
            "geer_build_graph_host": ([P, P, P, D, ctypes.c_int32], I),
            "geer_render_host": ([P, P, P, P, P, P, P], I),
            "geer_render_backward_host": ([P, P, P, P, P, P], I),
            "geer_l1_grad": ([P, P, P, P, I64, F, P], I),
            "geer_adam": ([P, P, P, P, P, I64, F, F, F, ctypes.c_int32, P, P], I),
            "geer_measure_fp32_peak": ([I, P, P], I),
            "geer_loss_workspace_bytes": ([I, I], ctypes.c_size_t),
            "geer_loss": ([P, P, P, I, I, F, P, P, P, P], I),
            "geer_resample_to_beap": ([P, I, I, P, P, P, P, P], I),
            "geer_ply_to_soa": ([P, I64, I, P, I, P, P], I),
            "geer_association_check": ([P, ctypes.c_int32, P, P, ctypes.c_int32, P], I),
            "geer_sync": ([P, P], I),
            "geer_clear_camera_cache": ([P], I),
            "geer_workspace_bytes": ([P, I64, ctypes.c_int32, P, P, I64], ctypes.c_size_t),
            "geer_set_workspace": ([P, P, ctypes.c_size_t], I),
            "geer_workspace_used": ([P, P], I),
            "geer_debug_n_eval": ([P, P], I),
            "geer_last_h2d_bytes": ([P], ctypes.c_int64),
        }
        for name, (args, res) in sig.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _lib = lib
        return lib


def last_error() -> str:
    msg = load().geer_last_error()
    return msg.decode() if msg else ""


def check(code: int) -> None:
    """Map a geer_status to the reference's exception types (association.py:155-160)."""
    if code == GEER_OK:
        return
    msg = last_error()
    if code in (GEER_ERR_INVALID, GEER_ERR_NOT_PD, GEER_ERR_NOT_SYMMETRIC):
        raise ValueError(msg)
    if code == GEER_ERR_NOMEM:
        raise MemoryError(msg)
    raise GeerError(code, msg)


def camera_struct(camera) -> GeerCamera:
    c = GeerCamera()
    c.width = int(camera.width)
    c.height = int(camera.height)
    c.model = MODEL_IDS[camera.model]
    c.rotation[:] = [float(v) for v in np.asarray(camera.rotation, dtype=np.float64).ravel()]
    c.translation[:] = [float(v) for v in np.asarray(camera.translation, dtype=np.float64).ravel()]
    nan = float("nan")
    opt = lambda v: float(v) if v is not None else nan
    c.fov_x, c.fov_y = opt(camera.fov_x), opt(camera.fov_y)
    c.fx, c.fy, c.cx, c.cy = opt(camera.fx), opt(camera.fy), opt(camera.cx), opt(camera.cy)
    c.k[:] = [float(v) for v in np.asarray(getattr(camera, "k", np.zeros(4)), dtype=np.float64).ravel()]
    return c


GEER_CFG_NO_CULL = 1
GEER_CFG_EXHAUSTIVE = 2  # every tile composites all kept Gaussians (association oracle, forward only)


def config_struct(config, flags: int = 0) -> GeerConfig:
    g = GeerConfig()
    g.lam = float(config.lam)
    g.background[:] = [float(v) for v in np.asarray(config.background, dtype=np.float64).reshape(3)]
    g.tile_px = int(config.tile_px)
    g.support_cutoff = 1 if config.support_cutoff else 0
    g.threads = int(getattr(config, "threads", 1) or 0)
    g.flags = int(flags)
    return g


class Context:
    """Owns one geer_ctx (device workspaces + the state of its last forward)."""

    def __init__(self, device: int = 0):
        lib = load()
        self._lib = lib
        self.device = device
        self.ptr = lib.geer_create(device)
        if not self.ptr:
            raise GeerError(GEER_ERR_CUDA, last_error() or "geer_create failed (no CUDA device?)")

    def close(self):
        if getattr(self, "ptr", None):
            self._lib.geer_destroy(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_timing(self, on: bool):
        check(self._lib.geer_set_timing(self.ptr, 1 if on else 0))

    def stats(self) -> dict:
        s = GeerStats()
        check(self._lib.geer_frame_stats(self.ptr, ctypes.byref(s)))
        return s.as_dict()

    def association_check(self, rays_per_tile: int = 64, max_missing: int = 16, hit_bits_ptr: int = 0) -> dict:
        """GPU ``oracle.association_bruteforce`` (oracle.py:235-281) against this context's last graph.

        Returns brute-force pair, missing pair (0 = sound), kept-Gaussian and entry counts and the
        first ``max_missing`` missing (tile, gid) pairs.  Validation only.
        """
        import numpy as np

        out = np.zeros(4, np.int64)
        miss = np.zeros((max(max_missing, 1), 2), np.int32)
        check(self._lib.geer_association_check(self.ptr, int(rays_per_tile), out.ctypes.data, miss.ctypes.data,
                                                int(max_missing), hit_bits_ptr or None))
        k = int(min(out[1], max_missing))
        return {"brute_pairs": int(out[0]), "missing": int(out[1]), "n_kept": int(out[2]),
                "graph_entries": int(out[3]), "missing_pairs": miss[:k].tolist()}


_default = threading.local()


def default_context(device: int = 0) -> Context:
    """Per-thread, per-device context of the reference-compatible host API.

    A context is not thread-safe (it owns one stream and the state of its last frame), so every host
    thread gets its own: several threads can render concurrently (ctypes releases the GIL).
    """
    ctxs = getattr(_default, "ctxs", None)
    if ctxs is None:
        ctxs = _default.ctxs = {}
    ctx = ctxs.get(device)
    if ctx is None:
        ctx = Context(device)
        ctxs[device] = ctx
    return ctx
