"""Parity checks shared by the GPU tests (tolerances from SURVEY §8c / BASELINE north_star)."""

from __future__ import annotations

import numpy as np

IMAGE_ATOL = 1e-4  # max abs on RGB and alpha (north_star: "max abs 1e-4 on images")
GRAD_REL = 1e-3  # per element: |g - g_ref| <= 1e-3 |g_ref| + 1e-4 max|g_ref| (north_star "rel 1e-3")
GRAD_FLOOR = 1e-4
GRAD_KEYS = ("dmeans", "dlog_scales", "dquats", "dopacities", "dsh")


def assert_graph_equal(g, order, entry_tile, ranges, keep=None, clamped=None):
    """Association lists bit-exact (no enumerated ties are expected in fp64; any diff fails)."""
    order = np.asarray(order).astype(np.int64)
    ranges = np.asarray(ranges).astype(np.int64)
    np.testing.assert_array_equal(g.ranges, ranges, err_msg="per-tile ranges differ")
    if not np.array_equal(g.order, order):
        bad = np.nonzero(g.order != order)[0] if len(g.order) == len(order) else []
        raise AssertionError(f"order differs: {len(g.order)} vs {len(order)} entries, "
                             f"{len(bad)} positions differ, first at {bad[:5]}")
    if entry_tile is not None:
        np.testing.assert_array_equal(g.entry_tile, np.asarray(entry_tile).astype(np.int64))
    if keep is not None:
        np.testing.assert_array_equal(g.keep, np.asarray(keep).astype(bool))
    if clamped is not None:
        np.testing.assert_array_equal(g.clamped, np.asarray(clamped).astype(bool))


def image_report(color, remaining, count, ref_color, ref_remaining, ref_count):
    dc = np.abs(np.asarray(color, np.float64) - ref_color)
    da = np.abs(np.asarray(remaining, np.float64) - ref_remaining)
    cnt_bad = int((np.asarray(count) != ref_count).sum()) if ref_count is not None else 0
    return {"color_max": float(dc.max()) if dc.size else 0.0, "color_mean": float(dc.mean()) if dc.size else 0.0,
            "color_p9999": float(np.quantile(dc, 0.9999)) if dc.size else 0.0,
            "alpha_max": float(da.max()) if da.size else 0.0, "count_mismatch": cnt_bad}


def assert_image_close(color, remaining, count, ref_color, ref_remaining, ref_count, check_count=True):
    r = image_report(color, remaining, count, ref_color, ref_remaining, ref_count if check_count else None)
    assert r["color_max"] <= IMAGE_ATOL, r
    assert r["alpha_max"] <= IMAGE_ATOL, r
    if check_count:
        assert r["count_mismatch"] == 0, r
    return r


def grad_report(grads, ref: dict, idx=None, keys=GRAD_KEYS):
    out = {}
    for k in keys:
        g = np.asarray(getattr(grads, k) if not isinstance(grads, dict) else grads[k], np.float64)
        if idx is not None:
            g = g[idx]
        r = np.asarray(ref[k], np.float64)
        scale = np.abs(r).max() if r.size else 0.0
        err = np.abs(g - r)
        viol = err > GRAD_REL * np.abs(r) + GRAD_FLOOR * scale
        sig = np.abs(r) > 1e-2 * scale
        worst = float((err[sig] / np.abs(r[sig])).max()) if sig.any() else 0.0
        out[k] = {"violations": int(viol.sum()), "worst_rel_significant": worst, "max_abs": float(err.max()) if err.size else 0.0,
                  "scale": float(scale)}
    return out


def assert_grads_close(grads, ref: dict, idx=None, keys=GRAD_KEYS):
    rep = grad_report(grads, ref, idx, keys)
    for k, v in rep.items():
        assert v["violations"] == 0, (k, v)
    return rep
