"""CPU oracle for the 3DGEER rendering hot path — TEST INFRASTRUCTURE ONLY.

ctypes front-end of ``geer_oracle.c``, an fp64 C restatement of the reference
``raygauss`` path (``/root/reference/pkg/src/raygauss``):

* :func:`build_grid`          — ``association.build_grid`` (association.py:301-332)
                                 + world ray directions (renderer.py:76-77)
* :func:`build_render_graph`  — ``association.build_render_graph`` (association.py:391-476)
* :func:`render`              — ``renderer.render`` (renderer.py:123-176)
* :func:`render_backward`     — ``renderer.render_backward`` (renderer.py:234-333)

Arguments are duck-typed like the reference dataclasses (``GaussianScene``,
``Camera``, ``RenderConfig``), so both the reference's objects and the
product's mirrors work.  Parity of this restatement with the reference is
pinned by ``tests/golden`` (fixtures produced by the unmodified reference,
``tests/golden/make_golden.py``) and checked by ``tests/test_oracle_golden.py``.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline legs may
import this module.  The product never does.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libgeer_oracle.so")

MODEL_IDS = {"pinhole": 0, "kb": 1, "beap": 2}


class GeoCamera(ctypes.Structure):
    _fields_ = [
        ("width", ctypes.c_int32),
        ("height", ctypes.c_int32),
        ("model", ctypes.c_int32),
        ("pad_", ctypes.c_int32),
        ("rotation", ctypes.c_double * 9),
        ("translation", ctypes.c_double * 3),
        ("fov_x", ctypes.c_double),
        ("fov_y", ctypes.c_double),
        ("fx", ctypes.c_double),
        ("fy", ctypes.c_double),
        ("cx", ctypes.c_double),
        ("cy", ctypes.c_double),
        ("k", ctypes.c_double * 4),
    ]


class GeoConfig(ctypes.Structure):
    _fields_ = [
        ("lam", ctypes.c_double),
        ("background", ctypes.c_double * 3),
        ("tile_px", ctypes.c_int32),
        ("support_cutoff", ctypes.c_int32),
        ("threads", ctypes.c_int32),
        ("pad_", ctypes.c_int32),
    ]


def build_oracle() -> str:
    """Compile the C restatement (make in oracle/); returns the .so path."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


_lib = None


def _load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        build_oracle()
    lib = ctypes.CDLL(_LIB_PATH)
    P = ctypes.c_void_p
    i64 = ctypes.c_int64
    lib.geo_grid.argtypes = [P, ctypes.c_int, ctypes.c_int, ctypes.c_int, P, P, P, P]
    lib.geo_grid.restype = ctypes.c_int
    lib.geo_graph.argtypes = [i64, P, P, P, P, P, ctypes.c_double, ctypes.c_int, ctypes.c_int, P, P,
                              P, P, P, P, P, P, P, P, ctypes.c_char_p, ctypes.c_int]
    lib.geo_graph.restype = ctypes.c_int
    lib.geo_forward.argtypes = [i64, ctypes.c_int, P, P, P, P, P, P, P, P, P, i64, P, P, P, P, P, P]
    lib.geo_forward.restype = ctypes.c_int
    lib.geo_backward.argtypes = [i64, ctypes.c_int, P, P, P, P, P, P, P, P, P, i64, P, P, P, P, P, P, P, P]
    lib.geo_backward.restype = ctypes.c_int
    lib.geo_free.argtypes = [P]
    lib.geo_num_threads.restype = ctypes.c_int
    _lib = lib
    return lib


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def _f64(a, shape=None):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if shape is not None:
        a = a.reshape(shape)
    return a


def camera_struct(camera) -> GeoCamera:
    c = GeoCamera()
    c.width = int(camera.width)
    c.height = int(camera.height)
    c.model = MODEL_IDS[camera.model]
    c.rotation[:] = [float(v) for v in np.asarray(camera.rotation, dtype=np.float64).ravel()]
    c.translation[:] = [float(v) for v in np.asarray(camera.translation, dtype=np.float64).ravel()]
    nanv = float("nan")
    c.fov_x = float(camera.fov_x) if camera.fov_x is not None else nanv
    c.fov_y = float(camera.fov_y) if camera.fov_y is not None else nanv
    c.fx = float(camera.fx) if camera.fx is not None else nanv
    c.fy = float(camera.fy) if camera.fy is not None else nanv
    c.cx = float(camera.cx) if camera.cx is not None else nanv
    c.cy = float(camera.cy) if camera.cy is not None else nanv
    c.k[:] = [float(v) for v in np.asarray(camera.k, dtype=np.float64).ravel()]
    return c


def config_struct(config, threads=None) -> GeoConfig:
    g = GeoConfig()
    g.lam = float(getattr(config, "lam", 3.0))
    g.background[:] = [float(v) for v in np.asarray(getattr(config, "background", np.zeros(3)), dtype=np.float64).reshape(3)]
    g.tile_px = int(getattr(config, "tile_px", 16))
    g.support_cutoff = 1 if getattr(config, "support_cutoff", True) else 0
    g.threads = int(threads if threads is not None else 0)
    return g


@dataclass
class OracleGrid:
    n_x: int
    n_y: int
    mirror_edges_x: np.ndarray
    mirror_edges_y: np.ndarray
    pixel_tile: np.ndarray  # (H, W) int64
    dirs_world: np.ndarray  # (H, W, 3) float64

    @property
    def n_tiles(self) -> int:
        return self.n_x * self.n_y


@dataclass
class OracleGraph:
    grid: OracleGrid
    order: np.ndarray
    entry_tile: np.ndarray
    ranges: np.ndarray
    mu_c: np.ndarray
    depth: np.ndarray
    keep: np.ndarray
    clamped: np.ndarray


class OracleValueError(ValueError):
    pass


def build_grid(camera, tile_px: int = 16) -> OracleGrid:
    """association.py:301-332 (+ renderer.py:76-77 world directions)."""
    lib = _load()
    w, h = int(camera.width), int(camera.height)
    n_x = max(1, -(-w // tile_px))
    n_y = max(1, -(-h // tile_px))
    dirs = np.empty((h, w, 3), dtype=np.float64)
    ex = np.empty(n_x + 1, dtype=np.float64)
    ey = np.empty(n_y + 1, dtype=np.float64)
    pt = np.empty((h, w), dtype=np.int64)
    cam = camera_struct(camera)
    rc = lib.geo_grid(ctypes.byref(cam), tile_px, n_x, n_y, _ptr(dirs), _ptr(ex), _ptr(ey), _ptr(pt))
    if rc:
        raise MemoryError("oracle build_grid failed")
    return OracleGrid(n_x, n_y, ex, ey, pt, dirs)


def _scene_arrays(scene):
    means = _f64(scene.means).reshape(-1, 3)
    n = len(means)
    log_scales = _f64(scene.log_scales).reshape(n, 3)
    quats = _f64(scene.quats).reshape(n, 4)
    logits = _f64(scene.opacity_logits).reshape(n)
    sh = _f64(scene.sh)
    sh = sh.reshape(n, -1, 3) if n else sh.reshape(0, sh.shape[1] if sh.ndim == 3 else 1, 3)
    return means, log_scales, quats, logits, np.ascontiguousarray(sh)


def build_render_graph(scene, camera, lam: float = 3.0, tile_px: int = 16, grid: OracleGrid | None = None) -> OracleGraph:
    """association.py:391-476."""
    lib = _load()
    grid = grid or build_grid(camera, tile_px)
    means, log_scales, quats, logits, _ = _scene_arrays(scene)
    n = len(means)
    mu_c = np.empty((n, 3))
    depth = np.empty(n)
    keep = np.empty(n, dtype=np.uint8)
    clamped = np.empty(n, dtype=np.uint8)
    ranges = np.empty(grid.n_tiles + 1, dtype=np.int64)
    order_p = ctypes.c_void_p()
    tile_p = ctypes.c_void_p()
    n_ent = ctypes.c_int64()
    err = ctypes.create_string_buffer(256)
    cam = camera_struct(camera)
    rc = lib.geo_graph(n, _ptr(means), _ptr(log_scales), _ptr(quats), _ptr(logits), ctypes.byref(cam), float(lam),
                       grid.n_x, grid.n_y, _ptr(grid.mirror_edges_x), _ptr(grid.mirror_edges_y), _ptr(mu_c),
                       _ptr(depth), _ptr(keep), _ptr(clamped), ctypes.byref(order_p), ctypes.byref(tile_p),
                       ctypes.byref(n_ent), _ptr(ranges), err, 256)
    if rc:
        raise OracleValueError(err.value.decode())
    e = n_ent.value
    order = np.ctypeslib.as_array(ctypes.cast(order_p, ctypes.POINTER(ctypes.c_int64)), shape=(max(e, 1),))[:e].copy()
    tiles = np.ctypeslib.as_array(ctypes.cast(tile_p, ctypes.POINTER(ctypes.c_int64)), shape=(max(e, 1),))[:e].copy()
    lib.geo_free(order_p)
    lib.geo_free(tile_p)
    return OracleGraph(grid, order, tiles, ranges, mu_c, depth, keep.astype(bool), clamped.astype(bool))


@dataclass
class OracleFrame:
    color: np.ndarray
    remaining: np.ndarray
    count: np.ndarray
    n_eval: np.ndarray
    graph: OracleGraph | None


def render(scene, camera, config=None, threads=None, graph: OracleGraph | None = None) -> OracleFrame:
    """renderer.py:123-176 (fp64); also returns the per-pixel alive-entry count."""
    lib = _load()
    lam = float(getattr(config, "lam", 3.0)) if config is not None else 3.0
    tile_px = int(getattr(config, "tile_px", 16)) if config is not None else 16
    cfg = config_struct(config if config is not None else object(), threads)
    h, w = int(camera.height), int(camera.width)
    means, log_scales, quats, logits, sh = _scene_arrays(scene)
    n = len(means)
    if n == 0:
        bg = np.asarray(cfg.background[:], dtype=np.float64)
        return OracleFrame(np.broadcast_to(bg, (h, w, 3)).copy(), np.ones((h, w)), np.zeros((h, w), np.int64),
                           np.zeros((h, w), np.int64), None)
    graph = graph or build_render_graph(scene, camera, lam, tile_px)
    color = np.empty((h, w, 3))
    rem = np.empty((h, w))
    cnt = np.empty((h, w), dtype=np.int64)
    ne = np.empty((h, w), dtype=np.int64)
    cam = camera_struct(camera)
    order = np.ascontiguousarray(graph.order, dtype=np.int64)
    rc = lib.geo_forward(n, sh.shape[1], _ptr(means), _ptr(log_scales), _ptr(quats), _ptr(logits), _ptr(sh),
                         ctypes.byref(cam), ctypes.byref(cfg), _ptr(graph.grid.dirs_world), _ptr(graph.grid.pixel_tile),
                         graph.grid.n_tiles, _ptr(order), _ptr(graph.ranges), _ptr(color), _ptr(rem), _ptr(cnt), _ptr(ne))
    if rc:
        raise MemoryError("oracle render failed")
    return OracleFrame(color, rem, cnt, ne, graph)


@dataclass
class OracleGrads:
    dmeans: np.ndarray
    dlog_scales: np.ndarray
    dquats: np.ndarray
    dopacities: np.ndarray
    dsh: np.ndarray


def render_backward(scene, camera, dl_dimage, config=None, threads=None, graph: OracleGraph | None = None) -> OracleGrads:
    """renderer.py:234-333 (fp64, fixed tile-order reduction)."""
    lib = _load()
    lam = float(getattr(config, "lam", 3.0)) if config is not None else 3.0
    tile_px = int(getattr(config, "tile_px", 16)) if config is not None else 16
    cfg = config_struct(config if config is not None else object(), threads)
    means, log_scales, quats, logits, sh = _scene_arrays(scene)
    n = len(means)
    B = sh.shape[1]
    out = OracleGrads(np.zeros((n, 3)), np.zeros((n, 3)), np.zeros((n, 4)), np.zeros(n), np.zeros((n, B, 3)))
    if n == 0:
        return out
    graph = graph or build_render_graph(scene, camera, lam, tile_px)
    dl = _f64(dl_dimage).reshape(int(camera.height), int(camera.width), 3)
    cam = camera_struct(camera)
    order = np.ascontiguousarray(graph.order, dtype=np.int64)
    rc = lib.geo_backward(n, B, _ptr(means), _ptr(log_scales), _ptr(quats), _ptr(logits), _ptr(sh),
                          ctypes.byref(cam), ctypes.byref(cfg), _ptr(graph.grid.dirs_world), _ptr(graph.grid.pixel_tile),
                          graph.grid.n_tiles, _ptr(order), _ptr(graph.ranges), _ptr(dl), _ptr(out.dmeans),
                          _ptr(out.dlog_scales), _ptr(out.dquats), _ptr(out.dopacities), _ptr(out.dsh))
    if rc:
        raise MemoryError("oracle render_backward failed")
    return out


def num_threads() -> int:
    return int(_load().geo_num_threads())


def set_num_threads(n: int) -> None:
    """OpenMP threads of the oracle from now on (torchrun exports OMP_NUM_THREADS=1)."""
    lib = _load()
    lib.geo_set_num_threads.argtypes = [ctypes.c_int]
    lib.geo_set_num_threads(int(n))


def _rotations(quats: np.ndarray) -> np.ndarray:
    """scene.py:17-32: unit quaternion (r, i, j, k) -> rotation matrix."""
    q = quats / np.linalg.norm(quats, axis=1, keepdims=True)
    r, i, j, k = q[:, 0], q[:, 1], q[:, 2], q[:, 3]
    return np.stack([1 - 2 * (j * j + k * k), 2 * (i * j - r * k), 2 * (i * k + r * j),
                     2 * (i * j + r * k), 1 - 2 * (i * i + k * k), 2 * (j * k - r * i),
                     2 * (i * k - r * j), 2 * (j * k + r * i), 1 - 2 * (i * i + j * j)], axis=1).reshape(-1, 3, 3)


def association_bruteforce(scene, camera, lam: float = 3.0, rays_per_tile: int = 64, tile_px: int = 16,
                           graph: OracleGraph | None = None) -> np.ndarray:
    """oracle.py:235-281 ``association_bruteforce`` as an (n_tiles, ceil(n/32)) uint32 bitmap.

    Tile t holds kept Gaussian g iff min kappa over side x side rays at the centres of a regular
    bipolar-angle grid between the tile's mirror edges is <= lam^2 (side = max(8, ceil(sqrt(rays)))).
    The keep mask and the mirror edges come from this oracle's own build_render_graph.
    """
    graph = graph or build_render_graph(scene, camera, lam, tile_px)
    grid = graph.grid
    means, log_scales, quats, _, _ = _scene_arrays(scene)
    n = len(means)
    words = (n + 31) // 32
    bits = np.zeros((grid.n_tiles, words), np.uint32)
    kept = np.nonzero(graph.keep)[0]
    if len(kept) == 0:
        return bits
    whit = _rotations(quats[kept]).transpose(0, 2, 1) / np.exp(log_scales[kept])[:, :, None]  # scene.py:72-75
    rot = np.asarray(camera.rotation, np.float64)
    origin = -rot.T @ np.asarray(camera.translation, np.float64)  # camera.py:72-74
    o_u = np.einsum("nij,nj->ni", whit, origin[None, :] - means[kept])
    side = max(8, int(np.ceil(np.sqrt(rays_per_tile))))
    frac = (np.arange(side) + 0.5) / side
    for tile in range(grid.n_tiles):
        iy, ix = divmod(tile, grid.n_x)
        t0, t1 = 2.0 * np.arctan(grid.mirror_edges_x[ix]), 2.0 * np.arctan(grid.mirror_edges_x[ix + 1])
        p0, p1 = 2.0 * np.arctan(grid.mirror_edges_y[iy]), 2.0 * np.arctan(grid.mirror_edges_y[iy + 1])
        tt, pp = np.meshgrid(t0 + (t1 - t0) * frac, p0 + (p1 - p0) * frac)
        st, ct, sp, cp = np.sin(tt), np.cos(tt), np.sin(pp), np.cos(pp)  # camera.py:141-155
        d = np.stack([st * cp, ct * sp, ct * cp], axis=-1).reshape(-1, 3)
        d = (d / np.linalg.norm(d, axis=1, keepdims=True)) @ rot
        d_u = np.einsum("nij,rj->nri", whit, d)
        m = np.cross(o_u[:, None, :], d_u)
        hit = kept[(((m * m).sum(-1) / (d_u * d_u).sum(-1)).min(axis=1) <= lam * lam)]
        np.bitwise_or.at(bits[tile], hit >> 5, (np.uint32(1) << (hit & 31).astype(np.uint32)))
    return bits
