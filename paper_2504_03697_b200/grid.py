"""Device-resident staggered-grid fields (mirror of src/grid.py).

Conventions are the reference's (src/grid.py:1-15): cube of n cells of edge
h, cell (i, j, k) centred at ((i+1/2)h, (j+1/2)h, (k+1/2)h), u/v/w on the
x/y/z-normal faces with extents (n+1,n,n)/(n,n+1,n)/(n,n,n+1), scalars flat
with i fastest.

Storage is B200-first: every field lives in HBM as fp64.  A velocity
component is a physical tensor [k][j][i] whose x-rows are padded to a
multiple of 32 doubles (256 B) so each row starts on a full sector boundary;
``.u`` / ``.v`` / ``.w`` are strided *views* with the reference's logical
[i, j, k] indexing, so ``vel.u[1:n, n-1, :] += g*dt`` means what it means in
the reference.  Scalar fields stay flat and unpadded so ``ScalarField.data``
is exactly the reference's flat vector.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib

ROW_ALIGN = 32  # doubles per 256-byte row alignment


def _device():
    _lib.load_library()
    return torch.device("cuda", torch.cuda.current_device())


def as_device(x, dtype=torch.float64):
    """(tensor on the current CUDA device, came_from_host)."""
    if isinstance(x, torch.Tensor):
        if x.is_cuda and x.dtype == dtype:
            return x, False
        return x.to(device=_device(), dtype=dtype), not x.is_cuda
    a = np.asarray(x, dtype=np.float64 if dtype == torch.float64 else None)
    return torch.as_tensor(np.ascontiguousarray(a), device=_device()).to(dtype), True


def to_host(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy()


@dataclass(frozen=True)
class GridSpec:
    """Cubic grid geometry: ``n`` cells per side, cell edge ``h`` (src/grid.py:22-41).

    ``shape=(nx, ny, nz)`` (extension) describes a box of
    cells instead of the reference's cube; the cube is ``shape=None``.
    """

    n: int
    h: float = 1.0
    shape: tuple | None = None

    def __post_init__(self):
        if self.n < 1:
            raise ValueError(f"grid needs at least one cell per side, got n={self.n}")
        if not self.h > 0:
            raise ValueError(f"cell edge length must be positive, got h={self.h}")
        if self.shape is not None:
            if len(self.shape) != 3 or min(self.shape) < 1:
                raise ValueError(f"shape must be three positive extents, got {self.shape}")
            object.__setattr__(self, "shape", tuple(int(s) for s in self.shape))

    @classmethod
    def box(cls, nx: int, ny: int, nz: int, h: float = 1.0) -> "GridSpec":
        return cls(nx, h, (nx, ny, nz))

    @property
    def dims(self) -> tuple:
        return self.shape if self.shape is not None else (self.n, self.n, self.n)

    @property
    def nx(self) -> int:
        return self.dims[0]

    @property
    def ny(self) -> int:
        return self.dims[1]

    @property
    def nz(self) -> int:
        return self.dims[2]

    @property
    def is_cube(self) -> bool:
        return self.nx == self.ny == self.nz

    @property
    def side_length(self) -> float:
        return self.n * self.h

    @property
    def num_cells(self) -> int:
        return self.nx * self.ny * self.nz


def cell_index(spec: GridSpec, i: int, j: int, k: int) -> int:
    """Flat index of cell (i, j, k); i fastest (src/grid.py:44-48)."""
    n = spec.n
    assert 0 <= i < n and 0 <= j < n and 0 <= k < n, (i, j, k, n)
    return i + n * j + n * n * k


def _extents(spec: GridSpec):
    nx, ny, nz = spec.dims
    return ((nx + 1, ny, nz), (nx, ny + 1, nz), (nx, ny, nz + 1))


def padded_ld(na: int) -> int:
    return ((na + ROW_ALIGN - 1) // ROW_ALIGN) * ROW_ALIGN


class VelocityField:
    """Face-centred velocity components in HBM (src/grid.py:51-71)."""

    def __init__(self, spec: GridSpec, u=None, v=None, w=None):
        self.spec = spec
        dev = _device()
        self._phys = []
        self.ld = []
        views = []
        for comp, (ext, src) in enumerate(zip(_extents(spec), (u, v, w))):
            na, nb, nc = ext
            ld = padded_ld(na)
            phys = torch.zeros((nc, nb, ld), dtype=torch.float64, device=dev)
            view = phys[:, :, :na].permute(2, 1, 0)  # logical [i, j, k]
            if src is not None:
                t, _ = as_device(src)
                if tuple(t.shape) != ext:
                    name = "uvw"[comp]
                    raise ValueError(f"{name} must have shape {ext}, got {tuple(t.shape)}")
                view.copy_(t)
            self._phys.append(phys)
            self.ld.append(ld)
            views.append(view)
        self.u, self.v, self.w = views

    def copy(self) -> "VelocityField":
        return VelocityField(self.spec, self.u, self.v, self.w)

    def components(self):
        return self.u, self.v, self.w

    def ptrs(self):
        return tuple(p.data_ptr() for p in self._phys)

    def copy_from(self, other: "VelocityField") -> None:
        for a, b in zip(self._phys, other._phys):
            a.copy_(b)

    def numpy(self):
        """Host copies in the reference's C-order layout."""
        return tuple(np.ascontiguousarray(to_host(c)) for c in self.components())

    def load_host(self, u, v, w) -> None:
        """Copy reference-layout host arrays into the device field."""
        for view, src in zip(self.components(), (u, v, w)):
            view.copy_(torch.as_tensor(np.asarray(src)))


class ScalarField:
    """Cell-centred values, flat with i fastest, in HBM (src/grid.py:74-94)."""

    def __init__(self, spec: GridSpec, data=None):
        self.spec = spec
        if data is None:
            self.data = torch.zeros(spec.num_cells, dtype=torch.float64, device=_device())
        else:
            t, _ = as_device(data)  # shares a CUDA tensor, like np.asarray
            self.data = t
            if tuple(self.data.shape) != (spec.num_cells,):
                raise ValueError(
                    f"scalar field needs {spec.num_cells} values, got shape {tuple(self.data.shape)}")
            self.data = self.data.contiguous()

    def copy(self) -> "ScalarField":
        return ScalarField(self.spec, self.data.clone())

    def as_3d(self) -> torch.Tensor:
        """View as (nx, ny, nz) with [i, j, k] indexing (no copy)."""
        nx, ny, nz = self.spec.dims
        return self.data.view(nz, ny, nx).permute(2, 1, 0)

    def numpy(self) -> np.ndarray:
        return to_host(self.data)


def sample_velocity(field: VelocityField, point) -> np.ndarray:
    """Trilinear velocity at a point, clamped to each lattice hull (src/grid.py:124-142)."""
    p = np.asarray(point, dtype=np.float64)
    if p.shape != (3,):
        raise ValueError(f"point must have 3 components, got shape {p.shape}")
    if not np.all(np.isfinite(p)):
        raise ValueError(f"non-finite sample point {p!r}")
    if not field.spec.is_cube:
        raise ValueError("sample_velocity is defined on the reference's cube")
    lib = _lib.load_library()
    out = np.empty(3)
    u, v, w = field.ptrs()
    lu, lv, lw = field.ld
    _lib.check(lib.cf_sample_velocity(u, v, w, field.spec.n, lu, lv, lw, field.spec.h, float(p[0]),
                                      float(p[1]), float(p[2]), _lib.np_ptr(out), _lib.stream()),
               "sample_velocity")
    return out


def divergence(field: VelocityField) -> ScalarField:
    """Per-cell divergence (src/grid.py:145-154)."""
    out = ScalarField(field.spec)
    _divergence_into(field, 1.0, out.data)
    return out


def _divergence_into(field: VelocityField, scale: float, out: torch.Tensor, want_max: bool = False):
    lib = _lib.load_library()
    u, v, w = field.ptrs()
    lu, lv, lw = field.ld
    nx, ny, nz = field.spec.dims
    mx = _lib.dbl_out()
    _lib.check(lib.cf_divergence_slab(u, v, w, nx, ny, nz, 0, nz, 0, lu, lv, lw, field.spec.h, float(scale),
                                      out.data_ptr(), _lib.byref(mx) if want_max else None, _lib.stream()),
               "divergence")
    return mx.value if want_max else None
