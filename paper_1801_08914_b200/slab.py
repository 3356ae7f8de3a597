"""Zero-communication z-slab partition of one structured 3D mesh over ranks
(SURVEY.md §8(e)).

Rank r owns the cell layers [z0, z1) of an N0 x N1 x N2 mesh and the H / g rows of
every interior face whose minus cell it owns: the x- and y-faces of its layers
and the z-planes p with p - 1 in [z0, z1).  It hybridizes the sub-mesh of layers
[z0 - 1, z1 + 2) (clipped at the mesh ends) with the global cell sizes, so each
owned row sees both of its cells and all of its columns as interior faces: one
ghost layer below (plane z0 interior), two above (plane z1's plus cell z1 and,
for that cell's top plane z1 + 1 to be an interior column, cell z1 + 1); no
collective is needed.  Multiplier rows are numbered over interior
faces in face order (x-, y-, then z-faces; x fastest, z slowest: mbase in
csrc/kern_pattern.cu, the reference's src/mesh.cpp:75-90), so the owned rows are
one contiguous row range per face axis in both numberings and their CSR column
order is preserved: a rank's share of H is three slices of its sub-mesh values,
placed at three row ranges of the global CSR.  The redundant work is the ghost
layers, 3 / (slab thickness).

Host logic only; the element work runs through Space.hybridize on the rank's
own GPU.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Sequence, Tuple

import numpy as np


def slab_layers(nz: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous split of nz cell layers over world ranks (the first nz % world
    ranks take one layer more)."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    base, extra = divmod(nz, world)
    z0 = rank * base + min(rank, extra)
    return z0, z0 + base + (1 if rank < extra else 0)


def _group_sizes(cells: Sequence[int]) -> Tuple[int, int, int]:
    nx, ny, nz = cells
    return (nx - 1) * ny * nz, nx * (ny - 1) * nz, nx * ny * (nz - 1)


def _face_rank(cells, axis: int, x, y, z):
    """Interior-face rank (the multiplier block index) of face (axis, x, y, z)."""
    nx, ny, nz = cells
    g = _group_sizes(cells)
    if axis == 0:
        return (x - 1) + (nx - 1) * (y + ny * z)
    if axis == 1:
        return g[0] + x + nx * ((y - 1) + (ny - 1) * z)
    return g[0] + g[1] + x + nx * (y + ny * (z - 1))


def _face_of_rank(cells, r):
    """Inverse of _face_rank (vectorised): (axis, x, y, z)."""
    nx, ny, nz = cells
    g = _group_sizes(cells)
    r = np.asarray(r, np.int64)
    axis = np.where(r < g[0], 0, np.where(r < g[0] + g[1], 1, 2))
    q = r - np.where(axis == 0, 0, np.where(axis == 1, g[0], g[0] + g[1]))
    wx = np.where(axis == 0, nx - 1, nx)
    wy = np.where(axis == 1, ny - 1, ny)
    x = q % wx + (axis == 0)
    y = (q // wx) % wy + (axis == 1)
    z = q // (wx * wy) + (axis == 2)
    return axis, x, y, z


@dataclass
class SlabPart:
    """One rank's share of the global H / g: rows [global_start, global_start + n)
    for each (global_start, n) in ``ranges``, values in row order."""
    ranges: List[Tuple[int, int]]
    h_values: List[np.ndarray]
    g_values: List[np.ndarray]


class SlabPlan:
    """The slab of ``rank`` out of ``world`` for a 3D mesh of ``cells`` with RT_order."""

    def __init__(self, cells: Sequence[int], order: int, world: int, rank: int,
                 sizes: Sequence[float] | None = None):
        if len(cells) != 3:
            raise ValueError("slab partition: 3D meshes (z-slabs)")
        self.cells = tuple(int(c) for c in cells)
        nx, ny, nz = self.cells
        self.order, self.world, self.rank = order, world, rank
        self.dpf = (order + 1) ** 2
        self.sizes = tuple(sizes) if sizes is not None else tuple(1.0 / c for c in self.cells)
        self.z0, self.z1 = slab_layers(nz, world, rank)
        self.g0, self.g1 = max(self.z0 - 1, 0), min(self.z1 + 2, nz)
        self.sub_cells = (nx, ny, self.g1 - self.g0)
        self.cell_range = (self.g0 * nx * ny, self.g1 * nx * ny)  # sub-mesh cells, global numbering
        self.owned_cells = (self.z0 * nx * ny, self.z1 * nx * ny)
        # owned face blocks per axis: (first local block, first global block, count)
        blocks = []
        if self.z1 > self.z0:
            for axis in (0, 1):
                x0, y0 = (1, 0) if axis == 0 else (0, 1)
                cnt = ((nx - 1) * ny if axis == 0 else nx * (ny - 1)) * (self.z1 - self.z0)
                if cnt > 0:
                    blocks.append((int(_face_rank(self.sub_cells, axis, x0, y0, self.z0 - self.g0)),
                                   int(_face_rank(self.cells, axis, x0, y0, self.z0)), cnt))
            p0, p1 = max(self.z0 + 1, 1), min(self.z1, nz - 1)
            if p1 >= p0:
                blocks.append((int(_face_rank(self.sub_cells, 2, 0, 0, p0 - self.g0)),
                               int(_face_rank(self.cells, 2, 0, 0, p0)), nx * ny * (p1 - p0 + 1)))
        d = self.dpf
        self.row_ranges = [(lb * d, gb * d, c * d) for lb, gb, c in blocks]  # (local row, global row, rows)

    @property
    def owned_rows(self) -> int:
        return sum(n for _, _, n in self.row_ranges)

    def local_to_global_rows(self, rows) -> np.ndarray:
        """Any sub-mesh multiplier row -> its row in the global numbering."""
        rows = np.asarray(rows, np.int64)
        blk, sub = rows // self.dpf, rows % self.dpf
        axis, x, y, z = _face_of_rank(self.sub_cells, blk)
        out = np.empty_like(rows)
        for a in (0, 1, 2):
            sel = axis == a
            out[sel] = _face_rank(self.cells, a, x[sel], y[sel], z[sel] + self.g0)
        return out * self.dpf + sub

    def inputs(self, alpha, beta, f_hat, n: int):
        """The sub-mesh's slices of the global per-cell inputs (n local dofs per cell)."""
        c0, c1 = self.cell_range
        return (np.asarray(alpha)[c0:c1], np.asarray(beta)[c0:c1], np.asarray(f_hat)[c0 * n:c1 * n])

    def extract(self, row_offsets, h_values, g_values) -> SlabPart:
        """This rank's owned rows out of the sub-mesh's H (CSR row offsets + values) and g."""
        ro = np.asarray(row_offsets)
        hv, gv = np.asarray(h_values), np.asarray(g_values)
        return SlabPart([(gs, n) for _, gs, n in self.row_ranges],
                        [hv[ro[ls]:ro[ls + n]].copy() for ls, _, n in self.row_ranges],
                        [gv[ls:ls + n].copy() for ls, _, n in self.row_ranges])


def place(part: SlabPart, row_offsets, h_out: np.ndarray, g_out: np.ndarray) -> None:
    """Write a rank's share into the global H values / g (global CSR row offsets)."""
    ro = np.asarray(row_offsets)
    for (gs, n), hv, gv in zip(part.ranges, part.h_values, part.g_values):
        if hv.size != ro[gs + n] - ro[gs]:
            raise ValueError("slab part does not match the global pattern")
        h_out[ro[gs]:ro[gs + n]] = hv
        g_out[gs:gs + n] = gv


def hybridize_slab(plan: SlabPlan, alpha, beta, f_hat) -> SlabPart:
    """Hybridize the rank's sub-mesh on the current CUDA device and return its share
    (alpha, beta, f_hat: the GLOBAL per-cell inputs, host arrays)."""
    from . import Space
    sp = Space(3, plan.sub_cells, plan.order, sizes=plan.sizes)
    a, b, f = plan.inputs(alpha, beta, f_hat, sp.n)
    op = sp.hybridize(np.ascontiguousarray(a), np.ascontiguousarray(b), np.ascontiguousarray(f))
    hv, gv = op.values()
    ro, _ = sp.pattern("H")
    return plan.extract(ro, hv, gv)
