"""Seeded synthetic scenes for the five BASELINE.json configs.

This module holds NONE of the method's arithmetic: it only draws images.  It is
the one piece of code shared by the oracle-side tests and the CUDA-side tests
and bench (task rule: "only the seeded input generators serve both").

Recipes follow SURVEY.md Sec. 8(d) "Synthetic inputs" and DESIGN.md "Input
recipe".  The paper's own scenes (Cartosat-1 PAN 2.5 m, AWiFS 12-bit 56 m,
PAPER.md:126) are not available; these stand-ins reproduce their structure:
step edges, disks, thin lines and salt-and-pepper noise (c1), urban-like blocks
and roads on a smooth background (c2, c3), and water bodies / vegetation on
four bands (c4).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class SceneConfig:
    name: str
    width: int
    height: int
    bands: int
    dtype: type
    bit_depth: int
    seed: int
    description: str


CONFIGS = {
    "c1": SceneConfig("c1", 512, 512, 1, np.uint8, 8, 1304,
                      "512x512 uint8 synthetic panchromatic (steps, disks, lines + salt-and-pepper)"),
    "c2": SceneConfig("c2", 4096, 4096, 1, np.uint8, 8, 13042,
                      "4096x4096 uint8 synthetic urban-like panchromatic tile"),
    "c3": SceneConfig("c3", 12000, 12000, 1, np.uint16, 10, 13043,
                      "12000x12000 uint16 (10-bit) Cartosat-1-like PAN scene"),
    "c4": SceneConfig("c4", 8192, 8192, 4, np.uint16, 12, 13044,
                      "4-band 8192x8192 uint16 (12-bit) AWiFS-like multispectral scene"),
    "c5": SceneConfig("c5", 48000, 48000, 1, np.uint16, 10, 13045,
                      "48000x48000 uint16 (10-bit) PAN mosaic of 4x4 c3-generator tiles"),
}


def _disk(img, cx, cy, R, v):
    H, W = img.shape
    y0, y1 = max(0, int(np.floor(cy - R)) - 1), min(H, int(np.ceil(cy + R)) + 2)
    x0, x1 = max(0, int(np.floor(cx - R)) - 1), min(W, int(np.ceil(cx + R)) + 2)
    yy, xx = np.mgrid[y0:y1, x0:x1]
    m = (xx - cx) ** 2 + (yy - cy) ** 2 <= R * R
    img[y0:y1, x0:x1][m] = v


def scene_c1(clean: bool = False, seed: int = 1304, size: int = 512) -> np.ndarray:
    """c1: background 40, two steps, three disks, four lines, 1% salt-and-pepper.

    ``size`` rescales the layout (used for small parity cases); 512 is c1.
    """
    s = size / 512.0
    img = np.full((size, size), 40, np.uint8)
    img[:, int(256 * s):] = 140
    img[int(384 * s):, :int(256 * s)] = 90
    _disk(img, 128 * s, 128 * s, 40 * s, 220)
    _disk(img, 380 * s, 140 * s, 12.5 * s, 10)
    _disk(img, 400 * s, 420 * s, 60 * s, 240)
    img[int(200 * s), int(20 * s):int(236 * s) + 1] = 250
    img[int(200 * s):int(360 * s) + 1, int(300 * s)] = 20
    n = int(216 * s) + 1
    for i in range(n):
        img[int(260 * s) + i, int(20 * s) + i] = 200
    img[int(300 * s):int(302 * s) + 1, int(270 * s):int(500 * s) + 1] = 0
    if not clean:
        rng = np.random.default_rng(seed)
        u = rng.random(img.shape)
        img[u < 0.005] = 0
        img[(u >= 0.005) & (u < 0.01)] = 255
    return img


def _urban(H, W, seed, scale, n_rect, noise_sigma, maxval, dtype, rows_per_block=1024):
    """Urban-like generator (c2 at scale 1, c3 at scale 4)."""
    rng = np.random.default_rng(seed)
    # 4 random low-frequency cosines, amplitude 10 (x scale), around 100 (x scale)
    kx = rng.uniform(-2 * np.pi / 800, 2 * np.pi / 800, 4)
    ky = rng.uniform(-2 * np.pi / 800, 2 * np.pi / 800, 4)
    ph = rng.uniform(0, 2 * np.pi, 4)
    img = np.empty((H, W), np.float32)
    xs = np.arange(W, dtype=np.float64)
    # cos(kx x + ky y + ph) = cos(kx x) cos(ky y + ph) - sin(kx x) sin(ky y + ph): a rank-8 product
    B = np.concatenate([np.cos(np.outer(kx, xs)), np.sin(np.outer(kx, xs))]).astype(np.float32)
    for y0 in range(0, H, rows_per_block):
        y1 = min(H, y0 + rows_per_block)
        ys = np.arange(y0, y1, dtype=np.float64)
        A = np.concatenate([np.cos(np.outer(ys, ky) + ph), -np.sin(np.outer(ys, ky) + ph)], axis=1)
        img[y0:y1] = np.float32(100.0 * scale) + np.float32(10.0 * scale) * (A.astype(np.float32) @ B)
    # rectangles: sides U{6..48}, value U{130..230} (x scale)
    rw = rng.integers(6, 49, n_rect)
    rh = rng.integers(6, 49, n_rect)
    rx = rng.integers(0, W, n_rect)
    ry = rng.integers(0, H, n_rect)
    rv = rng.integers(130, 231, n_rect) * scale
    for i in range(n_rect):
        img[ry[i]:ry[i] + rh[i], rx[i]:rx[i] + rw[i]] = rv[i]
    # 24 horizontal + 24 vertical roads: width U{4..8}, value U{55..75} (x scale)
    for orient in (0, 1):
        pos = rng.integers(0, H if orient == 0 else W, 24)
        wid = rng.integers(4, 9, 24)
        val = rng.integers(55, 76, 24) * scale
        for p, w, v in zip(pos, wid, val):
            if orient == 0:
                img[p:p + w, :] = v
            else:
                img[:, p:p + w] = v
    # Gaussian noise, then quantise and clip to the bit depth
    out = np.empty((H, W), dtype)
    for y0 in range(0, H, rows_per_block):
        y1 = min(H, y0 + rows_per_block)
        nrng = np.random.default_rng([seed, 1, y0])
        blk = img[y0:y1] + np.float32(noise_sigma) * nrng.standard_normal((y1 - y0, W), dtype=np.float32)
        out[y0:y1] = np.clip(np.rint(blk), 0, maxval).astype(dtype)
    # salt-and-pepper 0.2%
    n_sp = int(round(0.002 * H * W))
    flat = out.reshape(-1)
    idx = rng.integers(0, H * W, n_sp)
    flat[idx[: n_sp // 2]] = 0
    flat[idx[n_sp // 2:]] = maxval
    return out


def scene_c2(seed: int = 13042, size: int = 4096) -> np.ndarray:
    n_rect = int(round(4000 * (size / 4096) ** 2))
    return _urban(size, size, seed, 1, max(n_rect, 1), 3.0, 255, np.uint8)


def scene_c3(seed: int = 13043, size: int = 12000, height: int | None = None) -> np.ndarray:
    H = size if height is None else height
    n_rect = int(round(60000 * (size * H) / (12000 * 12000)))
    return _urban(H, size, seed, 4, max(n_rect, 1), 6.0, 1023, np.uint16)


def scene_c4(seed: int = 13044, size: int = 8192) -> np.ndarray:
    """c4: 4 bands (B2..B5), water ellipses + rivers, vegetation, bare soil; 12-bit."""
    rng = np.random.default_rng(seed)
    H = W = size
    cls = np.full((H, W), 2, np.uint8)  # 0 water, 1 vegetation, 2 bare
    # low-frequency vegetation mask: thresholded sum of cosines
    ys = np.arange(H, dtype=np.float32)[:, None]
    xs = np.arange(W, dtype=np.float32)[None, :]
    f = np.zeros((H, W), np.float32)
    for _ in range(5):
        kx, ky = rng.uniform(-2 * np.pi / 1500, 2 * np.pi / 1500, 2)
        f += np.cos(kx * xs + ky * ys + rng.uniform(0, 2 * np.pi)).astype(np.float32)
    cls[f > 0.5] = 1
    del f
    scale = size / 8192.0
    for _ in range(300):
        cx, cy = rng.uniform(0, W), rng.uniform(0, H)
        a, b = rng.uniform(10, 120) * scale + 2, rng.uniform(10, 120) * scale + 2
        th = rng.uniform(0, np.pi)
        R = max(a, b)
        y0, y1 = max(0, int(cy - R) - 1), min(H, int(cy + R) + 2)
        x0, x1 = max(0, int(cx - R) - 1), min(W, int(cx + R) + 2)
        if y0 >= y1 or x0 >= x1:
            continue
        yy, xx = np.mgrid[y0:y1, x0:x1]
        u = (xx - cx) * np.cos(th) + (yy - cy) * np.sin(th)
        v = -(xx - cx) * np.sin(th) + (yy - cy) * np.cos(th)
        cls[y0:y1, x0:x1][(u / a) ** 2 + (v / b) ** 2 <= 1.0] = 0
    for _ in range(20):  # rivers: meandering polylines of width 3..12
        x, y = rng.uniform(0, W), 0.0
        ang = rng.uniform(np.pi / 3, 2 * np.pi / 3)
        w = rng.uniform(3, 12) * max(scale, 0.25)
        while 0 <= y < H and -W * 0.1 <= x < W * 1.1:
            ang += rng.normal(0, 0.15)
            ang = float(np.clip(ang, 0.2, np.pi - 0.2))
            nx, ny = x + 8 * np.cos(ang), y + 8 * np.sin(ang)
            for t in np.linspace(0, 1, 9):
                px, py = x + t * (nx - x), y + t * (ny - y)
                y0, y1 = max(0, int(py - w)), min(H, int(py + w) + 1)
                x0, x1 = max(0, int(px - w)), min(W, int(px + w) + 1)
                if y0 < y1 and x0 < x1:
                    cls[y0:y1, x0:x1] = 0
            x, y = nx, ny
    means = np.array([[900, 700, 300, 150],      # water   B2..B5
                      [800, 600, 2600, 1400],    # vegetation
                      [1500, 1700, 2000, 2500]], np.float32)  # bare
    out = np.empty((4, H, W), np.uint16)
    for b in range(4):
        nrng = np.random.default_rng([seed, 2, b])
        band = means[cls, b] + nrng.normal(0, 12.0, (H, W)).astype(np.float32)
        out[b] = np.clip(np.rint(band), 0, 4095).astype(np.uint16)
    return out


def scene_c5_tile(i: int, tile: int = 12000) -> np.ndarray:
    """Tile i (0..15) of the c5 4x4 mosaic: c3 generator with seed 13045 + i."""
    return scene_c3(seed=13045 + i, size=tile)


def make(name: str, **kw) -> np.ndarray:
    if name == "c1":
        return scene_c1(**kw)
    if name == "c1_clean":
        return scene_c1(clean=True, **kw)
    if name == "c2":
        return scene_c2(**kw)
    if name == "c3":
        return scene_c3(**kw)
    if name == "c4":
        return scene_c4(**kw)
    raise KeyError(name)


def random_image(rng: np.random.Generator, H: int, W: int, bit_depth: int, kind: str = "mixed"):
    """Small random test images (uniform noise, piecewise-constant blocks or both)."""
    maxv = (1 << bit_depth) - 1
    dtype = np.uint8 if bit_depth <= 8 else np.uint16
    if kind == "uniform":
        return rng.integers(0, maxv + 1, (H, W)).astype(dtype)
    img = np.full((H, W), rng.integers(0, maxv + 1), np.int64)
    for _ in range(max(1, (H * W) // 64)):
        y, x = rng.integers(0, H), rng.integers(0, W)
        h, w = rng.integers(1, max(2, H // 3)), rng.integers(1, max(2, W // 3))
        img[y:y + h, x:x + w] = rng.integers(0, maxv + 1)
    if kind == "mixed":
        m = rng.random((H, W)) < 0.05
        img[m] = rng.integers(0, maxv + 1, int(m.sum()))
    return img.astype(dtype)


def scene_c5_rows(a: int, b: int, out: np.ndarray | None = None, tile: int = 12000, tiles: int = 4) -> np.ndarray:
    """Rows [a, b) of the c5 mosaic (tiles x tiles c3-generator tiles, seeds
    13045 + i, row-major), generating only the tiles those rows cross; written
    into ``out`` ((b - a) x tiles*tile uint16, e.g. pinned host memory) if given."""
    W = tile * tiles
    if out is None:
        out = np.empty((b - a, W), np.uint16)
    for ty in range(a // tile, (b - 1) // tile + 1):
        y0, y1 = max(a, ty * tile), min(b, (ty + 1) * tile)
        for tx in range(tiles):
            t = scene_c5_tile(ty * tiles + tx, tile)
            out[y0 - a:y1 - a, tx * tile:(tx + 1) * tile] = t[y0 - ty * tile:y1 - ty * tile]
    return out
