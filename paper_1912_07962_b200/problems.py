"""Synthetic problem generators for the five BASELINE configurations.

Problem setup is host-side and outside the accelerated path; it follows
the reference's conventions (tomo.py) so the operators are the ones the
reference would build:

* parallel-beam Siddon blocks, one view per block, exact intersection
  lengths (tomo.py:219-301, restated in ``csrc/siddon.cpp``);
* view angles over [0, pi) mapped into the reference's (-90, 90] range by
  theta -> theta - 180 for theta > 90 (tomo.py:158-159): the same rays,
  the detector axis reversed;
* noise scaled so ||eps|| / ||A x_true|| equals the level exactly
  (tomo.py:323-333), Philox-keyed Generators throughout (README.md:142-149).

The phantoms are seeded random ellipses / ellipsoids as BASELINE.json
describes (the reference ships Shepp-Logan tables; the random-ellipse
recipe is documented in DESIGN.md).
"""

from __future__ import annotations

import concurrent.futures as cf
import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import _lib
from .linops import DenseBlockOperator, GeneratedBlockOperator, SparseBlockOperator


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(key=int(seed)))


def scaled_noise(clean: np.ndarray, level: float, rng: np.random.Generator) -> np.ndarray:
    """b = clean + eps with ||eps|| = level ||clean|| (tomo.py:323-333)."""
    if level == 0:
        return clean.copy()
    eps = rng.standard_normal(clean.shape[0])
    eps *= level * np.linalg.norm(clean) / np.linalg.norm(eps)
    return clean + eps


# ---------------------------------------------------------------------------
# configs[0]: dense Gaussian
# ---------------------------------------------------------------------------


def gaussian_dense(m=20000, n=1000, ell=100, seed=1912, noise=0.01, var_scale=1000.0):
    """A ~ N(0, 1/var_scale), x_true ~ N(0, 1), 1% noise; one Philox stream
    drawn in the order A, x_true, eps."""
    g = _rng(seed)
    a = g.standard_normal((m, n)) / np.sqrt(var_scale)
    x_true = g.standard_normal(n)
    clean = a @ x_true
    b = scaled_noise(clean, noise, g)
    return DenseBlockOperator(a, ell, b), b, x_true


# ---------------------------------------------------------------------------
# tomography
# ---------------------------------------------------------------------------


def angles_0_pi(count: int) -> np.ndarray:
    """Equispaced angles over [0, 180) deg, mapped into (-90, 90]."""
    deg = np.arange(count) * (180.0 / count)
    return np.where(deg > 90.0, deg - 180.0, deg)


def siddon2d_block(angle_deg: float, grid: int, rays: int, spacing: float = 1.0):
    """(indptr, indices, data, shape) of one 2D view (tomo.py:259-273)."""
    L = _lib.lib()
    rowptr = np.zeros(rays + 1, dtype=np.int64)
    _lib.check(L.slim_siddon2d_view(float(angle_deg), grid, rays, float(spacing),
                                    _lib.i64ptr(rowptr), None, None))
    nnz = int(rowptr[-1])
    col = np.empty(nnz, dtype=np.int32)
    val = np.empty(nnz, dtype=np.float64)
    _lib.check(L.slim_siddon2d_view(float(angle_deg), grid, rays, float(spacing),
                                    _lib.i64ptr(rowptr), _lib.i32ptr(col), _lib.dptr(val)))
    return rowptr, col, val, (rays, grid * grid)


def siddon3d_block(direction, grid: int, side: int, spacing: float = 1.0):
    """(indptr, indices, data, shape) of one 3D view (tomo.py:285-301)."""
    L = _lib.lib()
    d = np.ascontiguousarray(np.asarray(direction, dtype=float))
    rows = side * side
    rowptr = np.zeros(rows + 1, dtype=np.int64)
    _lib.check(L.slim_siddon3d_view(_lib.dptr(d), grid, side, float(spacing),
                                    _lib.i64ptr(rowptr), None, None))
    nnz = int(rowptr[-1])
    col = np.empty(nnz, dtype=np.int32)
    val = np.empty(nnz, dtype=np.float64)
    _lib.check(L.slim_siddon3d_view(_lib.dptr(d), grid, side, float(spacing),
                                    _lib.i64ptr(rowptr), _lib.i32ptr(col), _lib.dptr(val)))
    return rowptr, col, val, (rows, grid ** 3)


def _pmap(fn, items, threads=None):
    threads = threads or min(32, os.cpu_count() or 1)
    if len(items) <= 1 or threads <= 1:
        return [fn(it) for it in items]
    with cf.ThreadPoolExecutor(max_workers=threads) as pool:
        return list(pool.map(fn, items))


def random_ellipses(grid: int, count: int, seed: int) -> np.ndarray:
    """2D phantom: ``count`` additive ellipses, centres uniform in the image,
    semi-axes U(0.05, 0.4) of the width, intensity U(0.1, 1), angle U(0, pi);
    cell-centre rasterisation (tomo.py:110-120 convention)."""
    g = _rng(seed)
    centers = -1.0 + (np.arange(grid) + 0.5) * (2.0 / grid)
    yy, xx = np.meshgrid(centers, centers, indexing="ij")
    img = np.zeros((grid, grid))
    for _ in range(count):
        x0, y0 = g.uniform(-1.0, 1.0, 2)
        sa, sb = g.uniform(0.05, 0.4, 2) * 2.0
        val = g.uniform(0.1, 1.0)
        ang = g.uniform(0.0, np.pi)
        c, s = np.cos(ang), np.sin(ang)
        u = (xx - x0) * c + (yy - y0) * s
        v = -(xx - x0) * s + (yy - y0) * c
        img[(u / sa) ** 2 + (v / sb) ** 2 <= 1.0] += val
    return img.ravel()


def random_ellipsoids(grid: int, count: int, seed: int) -> np.ndarray:
    """3D phantom: ``count`` additive random ellipsoids (same recipe in 3D)."""
    g = _rng(seed)
    centers = -1.0 + (np.arange(grid) + 0.5) * (2.0 / grid)
    zz, yy, xx = np.meshgrid(centers, centers, centers, indexing="ij")
    vol = np.zeros((grid, grid, grid))
    for _ in range(count):
        c0 = g.uniform(-1.0, 1.0, 3)
        semi = g.uniform(0.05, 0.4, 3) * 2.0
        val = g.uniform(0.1, 1.0)
        q, _ = np.linalg.qr(g.standard_normal((3, 3)))
        pts = np.stack([xx - c0[0], yy - c0[1], zz - c0[2]], axis=-1) @ q
        inside = ((pts / semi) ** 2).sum(axis=-1) <= 1.0
        vol[inside] += val
    return vol.ravel()


@dataclass
class TomoProblem:
    op: SparseBlockOperator
    b: np.ndarray
    x_true: np.ndarray


def _finish_tomo(parts, x_true, noise, seed, dtype):
    blocks = [(ip, ix, d.astype(dtype), shp) for ip, ix, d, shp in parts]
    # clean data from the stored (possibly fp32-rounded) values, fp64 math
    clean = np.concatenate([
        _csr_matvec(ip, ix, d.astype(np.float64), x_true) for ip, ix, d, _ in blocks])
    b = scaled_noise(clean, noise, _rng(seed + 1))
    op = SparseBlockOperator(blocks, b, dtype=dtype)
    return TomoProblem(op, b, x_true)


def _finish_tomo_columns(view_fn, items, split_fn, x_true, noise, seed, dtype, c0, c1,
                         threads=None, chunk=32):
    """Column shard [c0, c1) of a tomography operator, built view by view so a
    rank never holds the whole operator: each view's rows are projected on
    x_true (the same clean data and noise as the unsharded problem, so b is
    bit-identical) and only the shard's columns are kept."""
    from .parallel import slice_csr_columns

    blocks, clean = [], []
    for v0 in range(0, len(items), chunk):
        for part in _pmap(view_fn, items[v0:v0 + chunk], threads):
            for ip, ix, d, shp in split_fn(v0, part):
                d = d.astype(dtype)
                clean.append(_csr_matvec(ip, ix, d.astype(np.float64), x_true))
                blocks.append(slice_csr_columns(ip, ix, d, shp, c0, c1))
    b = scaled_noise(np.concatenate(clean), noise, _rng(seed + 1))
    return TomoProblem(SparseBlockOperator(blocks, b, dtype=dtype), b, x_true)


def _csr_matvec(indptr, indices, data, x):
    import scipy.sparse as sp

    n = x.shape[0]
    return sp.csr_matrix((data, indices, indptr), shape=(indptr.shape[0] - 1, n)) @ x


def tomo2d(grid=256, n_views=180, rays=362, ellipses=10, seed=2, noise=0.01,
           dtype=np.float64, threads=None, col_range=None) -> TomoProblem:
    """configs[1] / configs[2]: one block per view, ell = rays.  ``col_range``
    = (c0, c1): only that column shard is kept (b and x_true stay whole)."""
    angles = angles_0_pi(n_views)
    x_true = random_ellipses(grid, ellipses, seed)
    view = lambda a: siddon2d_block(a, grid, rays)  # noqa: E731
    if col_range is not None:
        return _finish_tomo_columns(view, list(angles), lambda v0, part: [part], x_true, noise,
                                    seed, dtype, *col_range, threads=threads)
    parts = _pmap(view, list(angles), threads)
    return _finish_tomo(parts, x_true, noise, seed, dtype)


def tomo3d_geometry(n_views=180, side=128, sub_rows=2048, seed=4):
    """configs[3] directions (xy-plane over [0, pi)) and the per-view seeded
    ray permutation that defines the sub-blocks (row i of view v is ray
    ray_of_row[v side^2 + i])."""
    theta = np.arange(n_views) * (np.pi / n_views)
    dirs = np.stack([np.cos(theta), np.sin(theta), np.zeros_like(theta)], axis=1)
    rows = side * side
    if rows % sub_rows:
        raise ValueError("detector rows must split evenly into sub-blocks")
    g = _rng(seed + 7)
    ray_of_row = np.concatenate([g.permutation(rows) for _ in range(n_views)]).astype(np.int32)
    return dirs, ray_of_row


def projector_config(cfg_id: int):
    """(geometry, grid, dtype, block_rows, ray_of_row) of a tomography config
    (bench numbering 2..4 = BASELINE configs[1..3]) for the device projector."""
    from .tomo import parallel_2d_geometry, parallel_3d_geometry

    if cfg_id == 2:
        return parallel_2d_geometry(angles_0_pi(180), 362), 256, np.float64, 362, None
    if cfg_id == 3:
        return parallel_2d_geometry(angles_0_pi(720), 1448), 1024, np.float32, 1448, None
    if cfg_id == 4:
        dirs, rmap = tomo3d_geometry(180, 128, 2048, 4)
        return parallel_3d_geometry(dirs, 128), 128, np.float32, 2048, rmap
    raise ValueError(f"config {cfg_id} is not a tomography config")


def _split_view_3d(part, perm, sub_rows):
    """One 3D view's rows in the seeded order, cut into sub_rows-row blocks."""
    ip, ix, d, (nr, nc) = part
    counts = np.diff(ip)[perm]
    starts = ip[:-1][perm]
    out = []
    for s in range(0, nr, sub_rows):
        sel_c = counts[s:s + sub_rows]
        sel_s = starts[s:s + sub_rows]
        nip = np.zeros(sub_rows + 1, dtype=np.int64)
        np.cumsum(sel_c, out=nip[1:])
        gather = np.concatenate([np.arange(a, a + c) for a, c in zip(sel_s, sel_c)]) \
            if sel_c.sum() else np.zeros(0, dtype=np.int64)
        out.append((nip, ix[gather], d[gather], (sub_rows, nc)))
    return out


def tomo3d(grid=128, n_views=180, side=128, sub_rows=2048, ellipsoids=20, seed=4,
           noise=0.01, dtype=np.float32, threads=None, col_range=None) -> TomoProblem:
    """configs[3]: directions in the xy-plane over [0, pi); each view's
    side^2 rays split into side^2 / sub_rows contiguous blocks after a
    seeded per-view row permutation (uniform partition, linops.py:64-72).
    ``col_range`` = (c0, c1): only that column shard is kept."""
    dirs, ray_of_row = tomo3d_geometry(n_views, side, sub_rows, seed)
    rows = side * side
    x_true = random_ellipsoids(grid, ellipsoids, seed)
    view = lambda d: siddon3d_block(d, grid, side)  # noqa: E731
    if col_range is not None:
        return _finish_tomo_columns(view, list(dirs), _Counter3d(ray_of_row, rows, sub_rows),
                                    x_true, noise, seed, dtype, *col_range, threads=threads)
    parts = _pmap(view, list(dirs), threads)
    blocks = []
    for v, part in enumerate(parts):
        blocks += _split_view_3d(part, ray_of_row[v * rows:(v + 1) * rows], sub_rows)
    return _finish_tomo(blocks, x_true, noise, seed, dtype)


class _Counter3d:
    """split_fn for the view-by-view builder: views arrive in order, so the
    view index is a running count."""

    def __init__(self, ray_of_row, rows, sub_rows):
        self.ray_of_row, self.rows, self.sub_rows, self.v = ray_of_row, rows, sub_rows, 0

    def __call__(self, v0, part):
        v = self.v
        self.v += 1
        return _split_view_3d(part, self.ray_of_row[v * self.rows:(v + 1) * self.rows],
                              self.sub_rows)


# ---------------------------------------------------------------------------
# configs[4]: streaming dense LS, A generated by splitmix64, never stored
# ---------------------------------------------------------------------------


def generated_dense(n=65536, m=4194304, ell=256, seed=1912, noise=0.005, device=0):
    """A[i, j] = fp32((2u - 1) / sqrt(n)) from splitmix64(seed ^ (i n + j));
    x_true ~ N(0, 1) (Philox key seed); b = A x_true by the device generator
    (fp64 accumulation) plus Gaussian noise scaled to ``noise`` of ||A x_true||
    (Philox key seed + 1)."""
    op = GeneratedBlockOperator(m, n, ell, seed)
    x_true = _rng(seed).standard_normal(n)
    clean = op.apply_device(x_true, device=device)
    b = scaled_noise(clean, noise, _rng(seed + 1))
    return op.with_rhs(b), b, x_true


# ---------------------------------------------------------------------------
# Shepp-Logan head phantoms for the reference's tomo2d / tomo3d problem kinds
# (tomo.py:100-135): the published 2D table (Shepp & Logan 1974) and the
# contrast-enhanced 3D variant, cell-centre rasterisation on [-1, 1]^d.
# ---------------------------------------------------------------------------

# (x0, y0, semi_a, semi_b, angle_deg, additive intensity)
_SL2D = ((0.0, 0.0, 0.69, 0.92, 0.0, 2.0), (0.0, -0.0184, 0.6624, 0.874, 0.0, -0.98),
         (0.22, 0.0, 0.11, 0.31, -18.0, -0.02), (-0.22, 0.0, 0.16, 0.41, 18.0, -0.02),
         (0.0, 0.35, 0.21, 0.25, 0.0, 0.01), (0.0, 0.1, 0.046, 0.046, 0.0, 0.01),
         (0.0, -0.1, 0.046, 0.046, 0.0, 0.01), (-0.08, -0.605, 0.046, 0.023, 0.0, 0.01),
         (0.0, -0.605, 0.023, 0.023, 0.0, 0.01), (0.06, -0.605, 0.023, 0.046, 0.0, 0.01))
# (intensity, semi_a, semi_b, semi_c, x0, y0, z0, phi, theta, psi), z-x-z Euler degrees
_SL3D = ((1.0, 0.69, 0.92, 0.81, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0),
         (-0.8, 0.6624, 0.874, 0.78, 0.0, -0.0184, 0.0, 0.0, 0.0, 0.0),
         (-0.2, 0.11, 0.31, 0.22, 0.22, 0.0, 0.0, -18.0, 0.0, 10.0),
         (-0.2, 0.16, 0.41, 0.28, -0.22, 0.0, 0.0, 18.0, 0.0, 10.0),
         (0.1, 0.21, 0.25, 0.41, 0.0, 0.35, -0.15, 0.0, 0.0, 0.0),
         (0.1, 0.046, 0.046, 0.05, 0.0, 0.1, 0.25, 0.0, 0.0, 0.0),
         (0.1, 0.046, 0.046, 0.05, 0.0, -0.1, 0.25, 0.0, 0.0, 0.0),
         (0.1, 0.046, 0.023, 0.05, -0.08, -0.605, 0.0, 0.0, 0.0, 0.0),
         (0.1, 0.023, 0.023, 0.02, 0.0, -0.605, 0.0, 0.0, 0.0, 0.0),
         (0.1, 0.023, 0.046, 0.02, 0.06, -0.605, 0.0, 0.0, 0.0, 0.0))


def shepp_logan_2d(n: int) -> np.ndarray:
    centers = -1.0 + (np.arange(n) + 0.5) * (2.0 / n)
    yy, xx = np.meshgrid(centers, centers, indexing="ij")
    img = np.zeros((n, n))
    for x0, y0, sa, sb, ang, value in _SL2D:
        c, s = np.cos(np.radians(ang)), np.sin(np.radians(ang))
        u = (xx - x0) * c + (yy - y0) * s
        v = -(xx - x0) * s + (yy - y0) * c
        img[(u / sa) ** 2 + (v / sb) ** 2 <= 1.0] += value
    img[np.abs(img) < 1e-15] = 0.0
    return img.ravel()


def _euler_zxz(phi, theta, psi):
    cphi, sphi = np.cos(np.radians(phi)), np.sin(np.radians(phi))
    cth, sth = np.cos(np.radians(theta)), np.sin(np.radians(theta))
    cpsi, spsi = np.cos(np.radians(psi)), np.sin(np.radians(psi))
    return np.array([
        [cpsi * cphi - cth * sphi * spsi, cpsi * sphi + cth * cphi * spsi, spsi * sth],
        [-spsi * cphi - cth * sphi * cpsi, -spsi * sphi + cth * cphi * cpsi, cpsi * sth],
        [sth * sphi, -sth * cphi, cth]])


def shepp_logan_3d(n: int) -> np.ndarray:
    centers = -1.0 + (np.arange(n) + 0.5) * (2.0 / n)
    zz, yy, xx = np.meshgrid(centers, centers, centers, indexing="ij")
    vol = np.zeros((n, n, n))
    pts = np.stack([xx.ravel(), yy.ravel(), zz.ravel()])
    for value, sa, sb, sc, x0, y0, z0, phi, theta, psi in _SL3D:
        local = _euler_zxz(phi, theta, psi) @ (pts - np.array([[x0], [y0], [z0]]))
        inside = (local[0] / sa) ** 2 + (local[1] / sb) ** 2 + (local[2] / sc) ** 2 <= 1.0
        vol.ravel()[inside] += value
    vol[np.abs(vol) < 1e-15] = 0.0
    return vol.ravel()
