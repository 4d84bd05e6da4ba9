"""N > 1 plumbing on CPU: world_size-2 gloo ranks, replica realisations and the
max-over-ranks timing reduction bench.py uses."""
import os
import socket

import numpy as np
import torch.multiprocessing as mp

from paper_1409_2556_b200 import inputs
from paper_1409_2556_b200.replicas import replica_config


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    import torch.distributed as dist

    from paper_1409_2556_b200.replicas import barrier, max_over_ranks
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = replica_config(inputs.config(0).scaled((16, 16)), rank)
    lk, _ = cfg.fields()
    barrier()
    vals = max_over_ranks([10.0 * (rank + 1), -float(rank)])
    out[rank] = (float(lk.sum()), vals)
    dist.destroy_process_group()


def test_two_rank_gloo_replicas_and_max():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    assert out[0][1] == [20.0, 0.0] and out[1][1] == [20.0, 0.0]
    assert out[0][0] != out[1][0]  # distinct realisations per rank


def test_rank0_replica_is_the_baseline_input():
    cfg = inputs.config(4)
    assert replica_config(cfg, 0).log_kappa == cfg.log_kappa
    r1 = replica_config(cfg, 1)
    assert r1.log_kappa["seed"] != cfg.log_kappa["seed"]
    assert r1.log_storativity["seed"] != cfg.log_storativity["seed"]
    assert np.isclose(r1.log_kappa["var"], cfg.log_kappa["var"])


# ---- the split build of one Jacobian slice, world size 2 over gloo --------
class OracleBackend:
    """split_build's backend interface with the CPU oracle standing in for the library: the
    bases are the shifted solutions themselves (m = n_shifts, Y = identity), so every field the
    slab assembly forms is bit-identical to the one-rank fields."""

    def __init__(self, cfg, t):
        from oracle import fd as ofd
        from oracle import shifted_solver as oss
        from oracle import talbot as otal
        self.cfg, self.t = cfg, t
        lk, ls = cfg.fields()
        self.grid = ofd.Grid(tuple(cfg.shape), cfg.h)
        self.ops = ofd.assemble_fd(self.grid, np.exp(lk), np.exp(ls))
        self.pencil = oss.ShiftedPencil(self.ops.stiffness, self.ops.mass)
        self.contour = otal.build_contour(cfg.n_quad, cfg.times[t])
        self.n_src, self.n_rec = len(cfg.sources), len(cfg.receivers)
        self.n_items = self.n_src + self.n_rec
        self.n_shifts = cfg.n_quad // 2
        self.n_planes = cfg.shape[-1]
        self.plane_cells = int(np.prod(cfg.shape[:-1]))
        self.device = "cpu"

    def solve(self, i0, i1):
        from oracle import fd as ofd
        from oracle import forward as ofw
        from oracle import jacobian as ojac
        solver = ofw.SolverConfig(kind=self.cfg.solver_kind)
        U = []
        for i in range(i0, i1):
            if i < self.n_src:
                b = ofd.point_weights(self.grid, self.cfg.sources[i]).astype(np.complex128)
                U.append(ojac._solve_family_or_throw(self.pencil, b, list(self.contour.nodes), solver, "forward"))
            else:
                e = ofd.point_weights(self.grid, self.cfg.receivers[i - self.n_src])
                U.append(ojac.solve_adjoint_fields(self.pencil, e, self.contour, solver))
        return (i0, i1, U)

    def columns(self, part):
        return self.n_shifts

    def coefficients(self, part, m):
        i0, i1, _ = part
        Y = np.zeros((i1 - i0, self.n_shifts, m), dtype=np.complex128)
        for k in range(self.n_shifts):
            Y[:, k, k] = 1.0
        return Y, np.full((i1 - i0, self.n_shifts), self.n_shifts, dtype=np.int32)

    def export(self, part, v0, v1, m):
        import torch
        i0, i1, U = part
        a0, a1 = v0 * self.plane_cells, v1 * self.plane_cells
        blk = np.zeros((m, i1 - i0, a1 - a0), dtype=np.complex128)
        for b, u in enumerate(U):
            blk[: u.shape[1], b, :] = u[a0:a1, :].T
        return torch.from_numpy(blk.view(np.float64).ravel().copy())

    def assemble(self, slab, U_slab, m, Y_all, mu_all):
        from oracle import fd as ofd
        from oracle import talbot as otal
        from paper_1409_2556_b200.split_build import view
        p0, p1 = slab
        v0, v1 = view(p0, p1, self.n_planes)
        Us = U_slab.numpy().view(np.complex128)[..., 0]  # (m, items, cells)
        a0, a1 = v0 * self.plane_cells, v1 * self.plane_cells
        fields = []
        for b in range(self.n_items):
            f = np.zeros((self.grid.n_cells, self.n_shifts), dtype=np.complex128)  # zero outside the view
            for k in range(self.n_shifts):
                acc = np.zeros(a1 - a0, dtype=np.complex128)
                for j in range(mu_all[b, k]):
                    acc = acc + Y_all[b, k, j] * Us[j, b]
                if b < self.n_src:
                    acc = acc * otal.qhat_step(self.cfg.rates[b], self.contour.nodes[k])
                f[a0:a1, k] = acc
            fields.append(f)
        s0, s1 = p0 * self.plane_cells, p1 * self.plane_cells
        rows = []
        for s in range(self.n_src):
            for r in range(self.n_rec):
                rk, rs = ofd.sensitivity_rows_fd(self.ops, fields[s], fields[self.n_src + r], self.contour.weights,
                                                 self.contour.nodes, True)
                rows.append(np.concatenate([rk[s0:s1], rs[s0:s1]]))
        return np.array(rows)

    def predictions(self, part):
        from oracle import fd as ofd
        from oracle import talbot as otal
        i0, i1, U = part
        out = []
        for i in range(i0, min(i1, self.n_src)):
            phi = U[i - i0] * np.array([otal.qhat_step(self.cfg.rates[i], z) for z in self.contour.nodes])
            out.append([otal.inverse_laplace_sum(self.contour, phi.T @ ofd.point_weights(self.grid, q))
                        for q in self.cfg.receivers])
        return np.array(out).reshape(len(out), self.n_rec)

    def release(self, part):
        pass


def _split_case():
    return inputs.config(4).scaled((8, 6, 7), n_src=3, n_rec=4, n_times=2)


def _split_worker(rank, world, port, out):
    import torch.distributed as dist

    from paper_1409_2556_b200.split_build import split_slice
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    res = split_slice(OracleBackend(_split_case(), 1), dist, rank, world)
    out[rank] = (res.jacobian_slab, res.predictions, res.plane_range, res.columns)
    dist.destroy_process_group()


def test_two_rank_split_jacobian_equals_one_rank_bit_for_bit():
    """§8e: items split over 2 gloo ranks, one grouped all-to-all of the slab basis rows
    (with one halo plane), slab assembly on each rank: the concatenated column slabs equal the
    one-rank Jacobian slice bit for bit, and so do the predictions."""
    from oracle import fd as ofd
    from oracle import forward as ofw
    from oracle import jacobian as ojac
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_split_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    cfg = _split_case()
    lk, ls = cfg.fields()
    grid = ofd.Grid(tuple(cfg.shape), cfg.h)
    ex = ojac.ThtExperiment(grid, cfg.sources, cfg.rates, cfg.receivers, cfg.times, cfg.n_quad,
                            solver=ofw.SolverConfig(kind=cfg.solver_kind), include_storativity=True)
    ref = ojac.ThtForwardModel(ex, ls).jacobian(lk)
    n, pl = grid.n_cells, int(np.prod(cfg.shape[:-1]))
    rows = [ex.measurement_index(s, r, 1) for s in range(len(cfg.sources)) for r in range(len(cfg.receivers))]
    Jref = ref.jacobian[rows]
    got_k = np.zeros((len(rows), n))
    got_s = np.zeros((len(rows), n))
    for rank in range(world):
        J, pred, (p0, p1), m = out[rank]
        c = (p1 - p0) * pl
        got_k[:, p0 * pl: p1 * pl] = J[:, :c]
        got_s[:, p0 * pl: p1 * pl] = J[:, c:]
        assert np.array_equal(pred.ravel(), ref.predictions[rows])
    assert out[0][2][1] == out[1][2][0] and out[0][2][0] == 0 and out[1][2][1] == cfg.shape[-1]
    assert np.array_equal(got_k, Jref[:, :n]) and np.array_equal(got_s, Jref[:, n:])


def test_split_partition_and_halo():
    from paper_1409_2556_b200.split_build import partition, view
    assert partition(80, 3) == [(0, 27), (27, 54), (54, 80)]
    assert partition(5, 8)[-1] == (5, 5) and sum(b - a for a, b in partition(5, 8)) == 5
    assert view(0, 64, 128) == (0, 65) and view(64, 128, 128) == (63, 128) and view(0, 128, 128) == (0, 128)
