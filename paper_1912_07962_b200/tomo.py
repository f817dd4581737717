"""Parallel-beam projection operators (reference ``tomo.py``), with the CSR
blocks traced on the GPU.

``build_projector(geom, n)`` keeps the reference signature (tomo.py:304-320)
and returns the same row-block operator: one block per view, Siddon
intersection lengths. With ``device=`` the blocks are traced by the device
projector (``slim_build_projector``, csrc/siddon.cu) straight into HBM when
the solver first needs them, bit-identical to the host restatement
(csrc/siddon.cpp, itself a restatement of tomo.py:219-301), so the matrix
never exists on the host. Host-side block access (``csr_block`` /
``fetch_block``, used by the CPU oracle) traces the same rows on the host.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .linops import DeviceOperator, RowBlockOperator, SampleBlock, SparseBlockOperator

TOMO3D_MAX_N = 64  # reference guard for host-built 3D projectors (tomo.py:304-320)


def _checked_views(mode: str, angles, directions):
    """Validated view parameters of a geometry (same rules and messages as
    tomo.py:153-178): 2D angles in (-90, 90] degrees, 3D unit directions."""
    if mode == "parallel_2d":
        if angles is None or len(angles) == 0:
            raise ValueError("2D geometry needs at least one angle")
        ang = np.asarray(angles, dtype=float)
        if ((ang <= -90.0) | (ang > 90.0)).any():
            raise ValueError("view angles must lie in (-90, 90] degrees")
        return ang, directions
    if mode == "parallel_3d":
        if directions is None or len(directions) == 0:
            raise ValueError("3D geometry needs at least one direction")
        dirs = np.asarray(directions, dtype=float)
        if dirs.ndim != 2 or dirs.shape[1] != 3:
            raise ValueError("directions must be (n_views, 3)")
        if (np.abs(np.sqrt((dirs * dirs).sum(axis=1)) - 1.0) > 1e-12).any():
            raise ValueError("directions must be unit vectors (1e-12)")
        return angles, dirs
    raise ValueError(f"unknown geometry mode {mode!r}")


@dataclass(frozen=True)
class ProjectionGeometry:
    """Parallel-beam acquisition (reference schema, tomo.py:139-182): 2D views
    by angle, 3D views by direction; ``rays_per_view`` is the 2D ray count or
    the 3D detector side (a 3D view then has rays_per_view**2 rows)."""

    mode: str
    angles: np.ndarray | None = None
    directions: np.ndarray | None = None
    rays_per_view: int = 0
    detector_spacing: float = 1.0

    def __post_init__(self):
        ang, dirs = _checked_views(self.mode, self.angles, self.directions)
        object.__setattr__(self, "angles", ang)
        object.__setattr__(self, "directions", dirs)
        if self.rays_per_view < 1:
            raise ValueError("rays_per_view must be >= 1")
        if not self.detector_spacing > 0:
            raise ValueError("detector_spacing must be > 0")

    @property
    def n_views(self) -> int:
        views = self.angles if self.mode == "parallel_2d" else self.directions
        return len(views)


def parallel_2d_geometry(angles_deg, rays_per_view: int,
                         detector_spacing: float = 1.0) -> ProjectionGeometry:
    """Geometry of 2D views at ``angles_deg`` (tomo.py:185-193)."""
    return ProjectionGeometry("parallel_2d", np.asarray(angles_deg, dtype=float), None,
                              rays_per_view, detector_spacing)


def parallel_3d_geometry(directions, detector_side: int,
                         detector_spacing: float = 1.0) -> ProjectionGeometry:
    """Geometry of 3D views along unit ``directions`` (tomo.py:196-204)."""
    return ProjectionGeometry("parallel_3d", None, np.asarray(directions, dtype=float),
                              detector_side, detector_spacing)


def _host_view(geom: ProjectionGeometry, n: int, v: int):
    from .problems import siddon2d_block, siddon3d_block

    if geom.mode == "parallel_2d":
        return siddon2d_block(geom.angles[v], n, geom.rays_per_view, geom.detector_spacing)
    return siddon3d_block(geom.directions[v], n, geom.rays_per_view, geom.detector_spacing)


class ProjectorOperator(RowBlockOperator):
    """Row-block projector whose blocks are traced on the device.

    Rows are the views' rays in view order; within view ``v`` row ``i`` is
    ray ``ray_of_row[v * rows_per_view + i]`` (identity by default), and
    blocks are ``block_rows`` consecutive rows (default: one view).
    """

    access_mode = "random_access"

    def __init__(self, geom: ProjectionGeometry, n: int, *, dtype=np.float64,
                 block_rows: int | None = None, ray_of_row=None, b=None):
        self.geom = geom
        self.grid = int(n)
        self.dims = 2 if geom.mode == "parallel_2d" else 3
        self.rows_per_view = geom.rays_per_view ** (self.dims - 1)
        self.n_cols = self.grid ** self.dims
        self.n_rows = geom.n_views * self.rows_per_view
        self.block_rows = int(block_rows or self.rows_per_view)
        if self.n_rows % self.block_rows:
            raise ValueError(f"{self.n_rows} rows do not split into blocks of {self.block_rows}")
        self.n_blocks = self.n_rows // self.block_rows
        self.dtype = np.dtype(dtype)
        if self.dtype not in (np.float32, np.float64):
            raise ValueError("dtype must be float32 or float64")
        if ray_of_row is not None:
            ray_of_row = np.ascontiguousarray(ray_of_row, dtype=np.int32)
            if ray_of_row.shape != (self.n_rows,):
                raise ValueError(f"ray_of_row must have {self.n_rows} entries")
            if ray_of_row.min() < 0 or ray_of_row.max() >= self.rows_per_view:
                raise ValueError("ray_of_row entries out of range")
        self.ray_of_row = ray_of_row
        self._proj = {"ctx": {}, "views": {}}  # shared by with_rhs copies
        self._b = None
        if b is not None:
            self._bind_rhs(b)

    def _bind_rhs(self, b):
        b = np.ascontiguousarray(np.asarray(b, dtype=float))
        if b.shape != (self.n_rows,):
            raise ValueError(f"b has shape {b.shape}, expected ({self.n_rows},)")
        self._b = b

    def with_rhs(self, b) -> "ProjectorOperator":
        op = ProjectorOperator.__new__(ProjectorOperator)
        op.__dict__.update({k: v for k, v in self.__dict__.items() if not k.startswith("_slim")})
        op._b = None
        op._bind_rhs(b)
        return op

    def has_rhs(self) -> bool:
        return self._b is not None

    @property
    def rhs(self) -> np.ndarray:
        if self._b is None:
            raise ValueError("operator has no right-hand side bound")
        return self._b

    # ---- host access (CPU oracle): the same rows traced on the host ----
    def _view(self, v: int):
        views = self._proj["views"]
        if v not in views:
            views[v] = _host_view(self.geom, self.grid, v)
        return views[v]

    def csr_block(self, i: int):
        self._check_index(i)
        ell = self.block_rows
        rowptr = np.zeros(ell + 1, dtype=np.int64)
        cols, vals = [], []
        for q in range(ell):
            row = (i - 1) * ell + q
            v, j = divmod(row, self.rows_per_view)
            if self.ray_of_row is not None:
                j = int(self.ray_of_row[row])
            ip, ix, d, _ = self._view(v)
            cols.append(ix[ip[j]:ip[j + 1]])
            vals.append(d[ip[j]:ip[j + 1]])
            rowptr[q + 1] = rowptr[q] + (ip[j + 1] - ip[j])
        col = np.concatenate(cols).astype(np.int32)
        val = np.concatenate(vals).astype(self.dtype)
        return rowptr, col, val, (ell, self.n_cols)

    def sparse_block(self, i: int):
        import scipy.sparse as sp

        ip, ix, d, shp = self.csr_block(i)
        return sp.csr_matrix((d.astype(float), ix, ip), shape=shp)

    def fetch_block(self, i: int) -> SampleBlock:
        self._check_index(i)
        if self._b is None:
            raise ValueError("operator has no right-hand side bound; use with_rhs(b)")
        s, e = self.row_range(i)
        return SampleBlock(i, self.sparse_block(i).toarray(), self._b[s:e])

    def to_host(self) -> SparseBlockOperator:
        """The same operator with host-resident blocks (traced on the host)."""
        return SparseBlockOperator([self.csr_block(i) for i in range(1, self.n_blocks + 1)],
                                   self._b, dtype=self.dtype)

    # ---- device ----
    def device_context(self, r: int, device: int = 0) -> DeviceOperator:
        """The operator traced into HBM for memory ``r`` on ``device`` (cached)."""
        key = (int(device), int(r))
        ctxs = self._proj["ctx"]
        dop = ctxs.get(key)
        if dop is None:
            dop = DeviceOperator(n_rows=self.n_rows, n_cols=self.n_cols, ell=self.block_rows, r=r,
                                 layout=_lib.SLIM_CSR_PERBLOCK, dtype=self.dtype, device=device)
            views = (self.geom.angles if self.dims == 2 else self.geom.directions)
            views = np.ascontiguousarray(views, dtype=float)
            rmap = _lib.i32ptr(self.ray_of_row) if self.ray_of_row is not None else None
            dop.call("slim_build_projector", self.dims, self.grid, self.geom.rays_per_view,
                     self.geom.n_views, _lib.dptr(views), C.c_double(self.geom.detector_spacing),
                     rmap)
            dop.call("slim_finalize_operator")
            dop.rhs_id = None
            ctxs[key] = dop
        if self._b is not None and dop.rhs_id is not id(self._b):
            dop.call("slim_set_rhs", _lib.dptr(self._b))
            dop.rhs_id = id(self._b)
            dop.rhs_ref = self._b
        return dop

    def apply_device(self, x, device: int = 0) -> np.ndarray:
        """A x on the device (fp64 accumulation), e.g. for clean data."""
        x = np.ascontiguousarray(np.asarray(x, dtype=float))
        if x.shape != (self.n_cols,):
            raise ValueError(f"x has shape {x.shape}, expected ({self.n_cols},)")
        ctxs = self._proj["ctx"]
        dop = next((d for (dev, _), d in ctxs.items() if dev == int(device)), None)
        if dop is None:
            dop = self.device_context(0, device)
        out = np.empty(self.n_rows)
        dop.call("slim_apply", _lib.dptr(x), _lib.dptr(out))
        return out

    def device_block(self, i: int, device: int = 0):
        """Block ``i`` as traced on the device: (rowptr, col, val)."""
        self._check_index(i)
        ctxs = self._proj["ctx"]
        dop = next((d for (dev, _), d in ctxs.items() if dev == int(device)), None)
        if dop is None:
            dop = self.device_context(0, device)
        rowptr = np.zeros(self.block_rows + 1, dtype=np.int64)
        dop.call("slim_get_csr_block", i, _lib.i64ptr(rowptr), None, None)
        nnz = int(rowptr[-1])
        col = np.empty(nnz, dtype=np.int32)
        val = np.empty(nnz, dtype=self.dtype)
        dop.call("slim_get_csr_block", i, _lib.i64ptr(rowptr), _lib.i32ptr(col), _lib.vptr(val))
        return rowptr, col, val


def build_projector(geom: ProjectionGeometry, n: int, *, device: int | None = None,
                    dtype=np.float64, block_rows: int | None = None, ray_of_row=None):
    """Sparse row-block ray-tracing operator, one block per view (tomo.py:304-320).

    ``device=None`` builds host blocks (the reference's behaviour, same 3D
    size guard); ``device=k`` returns a :class:`ProjectorOperator` traced on
    GPU ``k`` when first used (no 3D size guard: nothing is built on the host).
    """
    if device is None:
        if geom.mode == "parallel_3d" and n > TOMO3D_MAX_N:
            raise ValueError(f"3-D projectors are desk-scale only (n <= {TOMO3D_MAX_N})")
        op = ProjectorOperator(geom, n, dtype=dtype, block_rows=block_rows, ray_of_row=ray_of_row)
        return op.to_host()
    op = ProjectorOperator(geom, n, dtype=dtype, block_rows=block_rows, ray_of_row=ray_of_row)
    op.default_device = int(device)
    return op
