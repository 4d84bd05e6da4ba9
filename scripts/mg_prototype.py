"""Design prototype (not product, not oracle): NumPy model of the device inner
solver — cell-centred geometric multigrid V-cycle (red-black Gauss-Seidel,
multilinear prolongation, R = P^T, rediscretised coarse faces) as the
preconditioner of COCG for (K + tau M) u = v.  Used to choose the level /
smoother / tolerance parameters before writing the CUDA version.
"""
from __future__ import annotations

import sys
import time

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

sys.path.insert(0, ".")
from oracle import fd as fdmod  # noqa: E402
from oracle.talbot import build_contour  # noqa: E402
from oracle.shifted_solver import select_preconditioner_shifts  # noqa: E402
from paper_1409_2556_b200 import inputs  # noqa: E402


class Level:
    def __init__(self, shape, faces, mass):
        self.shape = shape  # numpy array shape (z,y,x)
        self.faces = faces  # list per numpy axis: face arrays with n+1 along axis
        self.mass = mass

    def diagK(self):
        d = np.zeros(self.shape)
        for ax, T in enumerate(self.faces):
            n = self.shape[ax]
            d += np.take(T, range(0, n), axis=ax) + np.take(T, range(1, n + 1), axis=ax)
        return d

    def offsum(self, u):
        s = np.zeros(self.shape, dtype=u.dtype)
        for ax, T in enumerate(self.faces):
            n = self.shape[ax]
            Tin = np.take(T, range(1, n), axis=ax)
            a = [slice(None)] * len(self.shape)
            b = [slice(None)] * len(self.shape)
            a[ax] = slice(0, n - 1)
            b[ax] = slice(1, n)
            s[tuple(a)] += Tin * u[tuple(b)]
            s[tuple(b)] += Tin * u[tuple(a)]
        return s

    def apply(self, tau, u):
        return (self.diagK() + tau * self.mass) * u - self.offsum(u)


def coarsen(lev):
    nd = len(lev.shape)
    agg = [2 if (n % 2 == 0 and n >= 4) else 1 for n in lev.shape]
    cshape = tuple(n // a for n, a in zip(lev.shape, agg))
    # mass: sum over aggregates
    m = lev.mass
    for ax in range(nd):
        if agg[ax] == 2:
            m = np.take(m, range(0, m.shape[ax], 2), axis=ax) + np.take(m, range(1, m.shape[ax], 2), axis=ax)
    faces = []
    for ax, T in enumerate(lev.faces):
        # pick faces at coarse-face positions along ax, sum over the transverse aggregate
        if agg[ax] == 2:
            Tc = np.take(T, range(0, T.shape[ax], 2), axis=ax) / 2.0
        else:
            Tc = T.copy()
        for ax2 in range(nd):
            if ax2 != ax and agg[ax2] == 2:
                Tc = np.take(Tc, range(0, Tc.shape[ax2], 2), axis=ax2) + np.take(Tc, range(1, Tc.shape[ax2], 2), axis=ax2)
        faces.append(Tc)
    return Level(cshape, faces, m), agg


def p1d(nc, agg):
    if agg == 1:
        return sp.identity(nc, format="csr")
    nf = 2 * nc
    rows, cols, vals = [], [], []
    for I in range(nc):
        f0, f1 = 2 * I, 2 * I + 1
        rows += [f0, f1]; cols += [I, I]; vals += [0.75, 0.75]
        if I - 1 >= 0:
            rows.append(f0); cols.append(I - 1); vals.append(0.25)
        else:
            rows.append(f0); cols.append(I); vals.append(-0.25)
        if I + 1 < nc:
            rows.append(f1); cols.append(I + 1); vals.append(0.25)
        else:
            rows.append(f1); cols.append(I); vals.append(-0.25)
    return sp.csr_matrix((vals, (rows, cols)), shape=(nf, nc))


def prolongator(cshape, agg):
    P = None
    for ax in range(len(cshape)):  # numpy axes (z, y, x): kron with x last
        p = p1d(cshape[ax], agg[ax])
        P = p if P is None else sp.kron(P, p, format="csr")
    return P


def to_csr(lev, tau):
    n = int(np.prod(lev.shape))
    idx = np.arange(n).reshape(lev.shape)
    rows, cols, vals = [idx.ravel()], [idx.ravel()], [(lev.diagK() + tau * lev.mass).ravel()]
    for ax, T in enumerate(lev.faces):
        nn = lev.shape[ax]
        Tin = np.take(T, range(1, nn), axis=ax).ravel()
        a = np.take(idx, range(0, nn - 1), axis=ax).ravel()
        b = np.take(idx, range(1, nn), axis=ax).ravel()
        rows += [a, b]; cols += [b, a]; vals += [-Tin, -Tin]
    return sp.csr_matrix((np.concatenate(vals).astype(complex), (np.concatenate(rows), np.concatenate(cols))), shape=(n, n))


class MG:
    def __init__(self, fine, max_coarse=512, nu=1):
        self.levels = [fine]
        self.aggs = []
        self.P = []
        self.nu = nu
        while int(np.prod(self.levels[-1].shape)) > max_coarse:
            c, agg = coarsen(self.levels[-1])
            if all(a == 1 for a in agg):
                break
            self.levels.append(c)
            self.aggs.append(agg)
            self.P.append(prolongator(c.shape, agg))
        self.colors = []
        for lev in self.levels:
            grids = np.indices(lev.shape).sum(axis=0)
            self.colors.append([(grids % 2 == 0), (grids % 2 == 1)])

    def set_tau(self, tau):
        self.tau = tau
        self.diag = [lev.diagK() + tau * lev.mass for lev in self.levels]
        self.coarse_lu = spla.splu(to_csr(self.levels[-1], tau).tocsc())

    def smooth(self, l, u, f, order):
        lev = self.levels[l]
        for c in order:
            mask = self.colors[l][c]
            s = lev.offsum(u)
            u = np.where(mask, (f + s) / self.diag[l], u)
        return u

    def vcycle(self, l, f):
        lev = self.levels[l]
        if l == len(self.levels) - 1:
            return self.coarse_lu.solve(f.ravel()).reshape(lev.shape)
        u = np.zeros(lev.shape, dtype=complex)
        for _ in range(self.nu):
            u = self.smooth(l, u, f, [0, 1])
        r = f - lev.apply(self.tau, u)
        rc = (self.P[l].T @ r.ravel()).reshape(self.levels[l + 1].shape)
        ec = self.vcycle(l + 1, rc)
        u = u + (self.P[l] @ ec.ravel()).reshape(lev.shape)
        for _ in range(self.nu):
            u = self.smooth(l, u, f, [1, 0])
        return u


def cocg(mg, tau, b, tol=1e-12, maxit=100):
    lev = mg.levels[0]
    x = np.zeros(lev.shape, dtype=complex)
    r = b.copy()
    bn = np.linalg.norm(b)
    z = mg.vcycle(0, r)
    p = z.copy()
    rho = np.sum(r * z)
    hist = []
    for it in range(maxit):
        q = lev.apply(tau, p)
        alpha = rho / np.sum(p * q)
        x += alpha * p
        r -= alpha * q
        rel = np.linalg.norm(r) / bn
        hist.append(rel)
        if rel <= tol:
            break
        z = mg.vcycle(0, r)
        rho_new = np.sum(r * z)
        p = z + (rho_new / rho) * p
        rho = rho_new
    return x, hist


def run(cfg, shape, nu=1):
    c = cfg.scaled(shape)
    lk, ls = c.fields()
    grid = fdmod.Grid(c.shape, c.h)
    kappa = np.exp(lk).reshape(grid.array_shape())
    S = np.exp(ls).reshape(grid.array_shape())
    faces_phys = fdmod.face_transmissibilities(grid, kappa)  # per physical dir
    nd = grid.dim
    faces = [None] * nd
    for d in range(nd):
        faces[nd - 1 - d] = faces_phys[d]
    fine = Level(grid.array_shape(), faces, S * grid.h ** nd)
    mg = MG(fine, nu=nu)
    ops = fdmod.assemble_fd(grid, kappa, S)
    contour = build_contour(c.n_quad, c.times[0])
    sched = select_preconditioner_shifts(list(contour.nodes))
    b = fdmod.point_weights(grid, c.sources[0]).reshape(grid.array_shape()).astype(complex)
    for tau in sched.taus:
        mg.set_tau(tau)
        t0 = time.time()
        x, hist = cocg(mg, tau, b)
        A = (ops.stiffness + tau * ops.mass).tocsc()
        xd = spla.spsolve(A, b.ravel())
        err = np.linalg.norm(x.ravel() - xd) / np.linalg.norm(xd)
        print(f"{c.name} levels={[l.shape for l in mg.levels]} tau={tau:.3g} its={len(hist)} "
              f"final={hist[-1]:.2e} err_vs_direct={err:.2e} rates={[f'{h:.1e}' for h in hist[:6]]} "
              f"t={time.time()-t0:.1f}s")
        # smooth RHS (second Krylov vector analogue)
        b2 = (ops.mass @ xd).reshape(grid.array_shape())
        b2 = b2 / np.linalg.norm(b2)
        x2, hist2 = cocg(mg, tau, b2)
        xd2 = spla.spsolve(A, b2.ravel())
        err2 = np.linalg.norm(x2.ravel() - xd2) / np.linalg.norm(xd2)
        print(f"   smooth rhs: its={len(hist2)} final={hist2[-1]:.2e} err={err2:.2e}")


if __name__ == "__main__":
    nu = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    run(inputs.config(0), (100, 100), nu)
    run(inputs.config(2), (128, 128), nu)
    run(inputs.config(1), (256, 256), nu)
    run(inputs.config(4), (32, 32, 32), nu)
    run(inputs.config(3), (64, 64, 32), nu)
