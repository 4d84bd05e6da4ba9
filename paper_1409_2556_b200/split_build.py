"""One Jacobian time slice split over ranks: one process per GPU,
torch.distributed for the plumbing, NCCL for the one exchange.

The rows of jacobian.cpp:205-246 are independent and each needs the forward field phi_s and
the adjoint field psi_r on the same cells.  So:

  1. the slice's items (sources, then receivers: the lockstep batch of lt_jacobian_slice) are
     split into contiguous ranges, one per rank, and each rank solves its own (lt_split_solve):
     no communication;
  2. the fine grid's planes (z-planes in 3-D, rows in 2-D) are split into slabs, one per rank;
     each rank sends every slab owner the rows of its bases U over that slab plus one halo
     plane on each interior side (lt_split_export) in ONE grouped all-to-all, and the small
     coefficient sets Y (n_items x n_shifts x m) are all-gathered;
  3. each rank assembles the J columns of its slab for every (source, receiver) row
     (lt_jacobian_assemble_slab); rows never need a reduction.  Predictions come from the
     ranks holding the sources (lt_split_predictions) and are all-gathered.

The exchange logic is written once (`split_slice`) over a small backend interface, so the
same partition / packing / all-to-all / unpacking code runs on the device (`DeviceBackend`,
NCCL) and in the CPU test with the oracle standing in for the library (tests/test_multirank.py,
gloo, world size 2).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Tuple

import numpy as np


def partition(n_items: int, world: int) -> List[Tuple[int, int]]:
    """Contiguous item ranges, sizes differing by at most one."""
    base, extra = divmod(n_items, world)
    out, i0 = [], 0
    for r in range(world):
        i1 = i0 + base + (1 if r < extra else 0)
        out.append((i0, i1))
        i0 = i1
    return out


def slabs(n_planes: int, world: int) -> List[Tuple[int, int]]:
    return partition(n_planes, world)


def view(plane0: int, plane1: int, n_planes: int) -> Tuple[int, int]:
    """The slab's planes plus one halo plane on each interior side."""
    return plane0 - (1 if plane0 > 0 else 0), plane1 + (1 if plane1 < n_planes else 0)


@dataclass
class SplitResult:
    jacobian_slab: object      # (pairs, n_blocks * slab_cells) on the backend's device
    predictions: np.ndarray    # (n_src, n_rec), every rank
    plane_range: Tuple[int, int]
    columns: int               # m (padded basis columns)


def split_slice(backend, dist, rank: int, world: int) -> SplitResult:
    """Steps 1-3 for one time slice; `backend` supplies the compute, `dist` the collectives
    (torch.distributed, initialised)."""
    import torch
    n_items, n_planes, plane = backend.n_items, backend.n_planes, backend.plane_cells
    if world > n_items or world > n_planes:
        raise ValueError("split build: more ranks than items or planes")
    parts = partition(n_items, world)
    slab = slabs(n_planes, world)
    i0, i1 = parts[rank]
    part = backend.solve(i0, i1)
    # every part padded to the largest basis
    m = torch.tensor([backend.columns(part)], dtype=torch.int64, device=backend.device)
    dist.all_reduce(m, op=dist.ReduceOp.MAX)
    m = int(m.item())
    # coefficients of all items (small): all-gather of each part's (Y, m_used)
    ns = backend.n_shifts
    Y, mu = backend.coefficients(part, m)  # (items, ns, m) complex, (items, ns) int
    ygather = [None] * world
    dist.all_gather_object(ygather, (Y, mu))
    Y_all = np.concatenate([g[0] for g in ygather], axis=0)
    mu_all = np.concatenate([g[1] for g in ygather], axis=0)
    assert Y_all.shape == (n_items, ns, m)
    # one grouped all-to-all of the slab basis rows: to rank q, planes view(slab q) of my items
    b_mine = i1 - i0
    send_sizes, chunks = [], []
    for q in range(world):
        v0, v1 = view(*slab[q], n_planes)
        buf = backend.export(part, v0, v1, m)          # complex (m, b_mine, cells) as float64 pairs
        chunks.append(buf)
        send_sizes.append(int(buf.numel()))
    send = torch.cat(chunks)
    v0, v1 = view(*slab[rank], n_planes)
    cells = (v1 - v0) * plane
    recv_sizes = [2 * m * (parts[r][1] - parts[r][0]) * cells for r in range(world)]
    recv = torch.empty(sum(recv_sizes), dtype=torch.float64, device=backend.device)
    dist.all_to_all_single(recv, send, recv_sizes, send_sizes)
    # unpack: rank r's block is (m, items of r, cells); items in global order along dim 1
    blocks, off = [], 0
    for r in range(world):
        nb = parts[r][1] - parts[r][0]
        blocks.append(recv[off: off + recv_sizes[r]].view(m, nb, cells, 2))
        off += recv_sizes[r]
    U_slab = torch.cat(blocks, dim=1).contiguous()  # (m, n_items, cells, re/im)
    J = backend.assemble(slab[rank], U_slab, m, Y_all, mu_all)
    # predictions: the parts holding sources compute theirs, everyone gathers
    pred_part = backend.predictions(part)            # (n_sources of this part, n_rec)
    pgather = [None] * world
    dist.all_gather_object(pgather, pred_part)
    pred = np.concatenate([p for p in pgather if p is not None and len(p)], axis=0)
    backend.release(part)
    return SplitResult(J, pred, slab[rank], m)


class DeviceBackend:
    """The library's C ABI on this rank's GPU: lt_split_* and lt_jacobian_assemble_slab."""

    def __init__(self, pencil, experiment, time_index: int):
        import torch
        from . import capi
        self.capi = capi
        self.lib = capi.lib()
        self.pencil = pencil
        self.ex, self._keep = experiment.c()
        self.t = time_index
        g = experiment.grid
        self.n_src, self.n_rec = len(experiment.sources), len(experiment.receivers)
        self.n_items = self.n_src + self.n_rec
        self.n_shifts = experiment.n_quad // 2
        self.n_planes = g.shape[-1] if g.dim == 3 else g.shape[1]
        self.plane_cells = int(np.prod(g.shape[:2])) if g.dim == 3 else g.shape[0]
        self.blocks = 2 if experiment.include_storativity else 1
        self.device = torch.device("cuda", torch.cuda.current_device())

    def solve(self, i0, i1):
        h = C.c_void_p()
        self.capi.check(self.lib.lt_split_solve(self.pencil.handle, C.byref(self.ex), self.t, i0, i1, C.byref(h)))
        return (h, i0, i1)

    def columns(self, part):
        return int(self.lib.lt_split_columns(part[0]))

    def coefficients(self, part, m):
        h, i0, i1 = part
        Y = np.zeros((i1 - i0, self.n_shifts, m), dtype=np.complex128)
        mu = np.zeros((i1 - i0, self.n_shifts), dtype=np.int32)
        self.capi.check(self.lib.lt_split_coefficients(h, m, self.capi.cptr(Y), mu.ctypes.data_as(self.capi.PI)))
        return Y, mu

    def export(self, part, v0, v1, m):
        import torch
        h, i0, i1 = part
        buf = torch.empty(2 * m * (i1 - i0) * (v1 - v0) * self.plane_cells, dtype=torch.float64, device=self.device)
        self.capi.check(self.lib.lt_split_export(h, v0, v1, m, C.c_void_p(buf.data_ptr()), self.capi.LT_MEM_DEVICE))
        return buf

    def assemble(self, slab, U_slab, m, Y_all, mu_all):
        import torch
        p0, p1 = slab
        cells = (p1 - p0) * self.plane_cells
        J = torch.empty((self.n_src * self.n_rec, self.blocks * cells), dtype=torch.float64, device=self.device)
        Y = np.ascontiguousarray(Y_all.astype(np.complex128))
        mu = np.ascontiguousarray(mu_all.astype(np.int32))
        torch.cuda.synchronize()
        self.capi.check(self.lib.lt_jacobian_assemble_slab(
            self.pencil.handle, C.byref(self.ex), self.t, p0, p1, C.c_void_p(U_slab.data_ptr()), m, self.capi.cptr(Y),
            mu.ctypes.data_as(self.capi.PI), self.capi.LT_MEM_DEVICE, C.c_void_p(J.data_ptr())))
        return J

    def predictions(self, part):
        h, i0, i1 = part
        n_loc = max(0, min(i1, self.n_src) - i0)
        out = np.zeros((n_loc, self.n_rec))
        if n_loc:
            self.capi.check(self.lib.lt_split_predictions(h, self.capi.dptr(out)))
        return out

    def release(self, part):
        self.lib.lt_split_destroy(part[0])
