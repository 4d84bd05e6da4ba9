"""The drop-in boundary on the device: the sparse-matrix pencil
ShiftedPencil(K, M) (shifted_solver.hpp:90), the direct mode (shifted_solver.cpp:324-332),
the kept FlexibleBasisState and residual_estimate (hpp:63-74, cpp:334-343), the non-convergence
paths (ConvergenceError, LT_ERR_NOT_CONVERGED) and more than 256 shifts per item; the C++
mirror (include/laptomo/laptomo.hpp) end to end.  All against the CPU oracle."""
from __future__ import annotations

import subprocess
from pathlib import Path

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from oracle import fd as ofd
from oracle import fem
from oracle import forward as ofw
from oracle import shifted_solver as oss
from oracle import talbot as otal
from paper_1409_2556_b200 import capi
from paper_1409_2556_b200 import laptomo as L

from .helpers import fd_case, rel

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _schedule(shifts):
    s = oss.select_preconditioner_shifts(shifts)
    return s, L.PreconditionerSchedule(s.taus, s.pattern)


@pytest.mark.parametrize("index,shape", [(0, (40, 30)), (4, (16, 12, 10)), (4, (64, 32, 8))])
def test_csr_pencil_fd_matches_grid_pencil_and_oracle(index, shape):
    cfg, lk, ls, grid, ops = fd_case(index, shape)
    pg = L.ShiftedPencil(L.Grid(tuple(cfg.shape), cfg.h), lk, ls)
    pc = L.ShiftedPencil.from_csr(L.Grid(tuple(cfg.shape), cfg.h), ops.stiffness, ops.mass)
    assert pc.rows() == grid.n_cells and pc.parameters() == 0
    rng = np.random.default_rng(4)
    x = rng.standard_normal(grid.n_cells) + 1j * rng.standard_normal(grid.n_cells)
    z = -0.4 + 0.3j
    assert rel(pc.apply(z, x), ops.stiffness @ x + z * (ops.mass @ x)) <= 1e-14
    assert rel(pc.apply(z, x), pg.apply(z, x)) <= 1e-14
    contour = otal.build_contour(cfg.n_quad, cfg.times[0])
    shifts = list(contour.nodes)
    sched, gs = _schedule(shifts)
    tau = sched.taus[0]
    u = pc.factorization(tau).solve(x)
    ref = spla.splu((ops.stiffness + tau * ops.mass).tocsc(), permc_spec="COLAMD").solve(x)
    assert rel(u, ref) <= 1e-10
    b = ofd.point_weights(grid, tuple(0.45 * m * cfg.h for m in cfg.shape)).astype(np.complex128)
    got = L.solve_shifted_flexible(pc, b, shifts, gs)
    oref = oss.solve_shifted_flexible(oss.ShiftedPencil(ops.stiffness, ops.mass), b, shifts, sched)
    assert got.all_converged and got.iterations == oref.iterations
    for k in range(len(shifts)):
        assert rel(got.solutions[:, k], oref.solutions[:, k]) <= 1e-8


def test_csr_pencil_p1_reference_assembly():
    """The reference's own assembled pair (assembly.cpp:69-113) through ShiftedPencil(K, M)."""
    rng = np.random.default_rng(5)
    mesh = fem.build_mesh(41, 100.0)
    lk = np.log(1e-4) + 1.2 * rng.standard_normal(mesh.n_elements())
    ls = np.log(1e-5) + 0.2 * rng.standard_normal(mesh.n_elements())
    ops = fem.assemble(mesh, np.exp(lk), np.exp(ls))
    pc = L.ShiftedPencil.from_csr(L.build_mesh(41, 100.0), ops.stiffness, ops.mass)
    pg = L.ShiftedPencil(L.build_mesh(41, 100.0), lk, ls)
    x = rng.standard_normal(ops.n_free()) + 1j * rng.standard_normal(ops.n_free())
    z = 0.01 - 0.02j
    assert rel(pc.apply(z, x), ops.stiffness @ x + z * (ops.mass @ x)) <= 1e-14
    assert rel(pc.apply_mass(x), ops.mass @ x) <= 1e-14
    assert rel(pc.apply(z, x), pg.apply(z, x)) <= 1e-13
    c = otal.build_contour(40, 300.0)
    shifts = list(c.nodes)
    sched, gs = _schedule(shifts)
    b = ops.restrict_to_free(fem.point_source(mesh, 50.0, 50.0)).astype(complex)
    got = L.solve_shifted_flexible(pc, b, shifts, gs)
    oref = oss.solve_shifted_flexible(oss.ShiftedPencil(ops.stiffness, ops.mass), b, shifts, sched)
    assert got.all_converged and abs(got.iterations - oref.iterations) <= 1
    direct = oss.solve_shifted_direct(oss.ShiftedPencil(ops.stiffness, ops.mass), b, shifts)
    for k in range(len(shifts)):
        assert rel(got.solutions[:, k], direct[:, k]) <= 1e-8


def test_csr_pencil_rejects_foreign_pattern():
    cfg, lk, ls, grid, ops = fd_case(0, (20, 20))
    g = L.Grid(tuple(cfg.shape), cfg.h)
    K = ops.stiffness.tolil()
    K[0, 7] = -1e-9  # off the 5-point stencil
    with pytest.raises(ValueError, match="stencil"):
        L.ShiftedPencil.from_csr(g, K.tocsr(), ops.mass)
    K = ops.stiffness.tolil()
    K[0, 1] = K[0, 1] * 1.5  # asymmetric
    with pytest.raises(ValueError, match="symmetric"):
        L.ShiftedPencil.from_csr(g, K.tocsr(), ops.mass)
    with pytest.raises(ValueError, match="diagonal"):
        L.ShiftedPencil.from_csr(g, ops.stiffness, ops.mass + sp.eye(grid.n_cells, k=1) * 1e-3)
    with pytest.raises(ValueError, match="rows"):
        L.ShiftedPencil.from_csr(L.Grid((21, 20), cfg.h), ops.stiffness, ops.mass)
    pc = L.ShiftedPencil.from_csr(g, ops.stiffness, ops.mass)
    ex = L.ThtExperiment(g, cfg.sources, cfg.rates, cfg.receivers[:2], cfg.times[:1], cfg.n_quad)
    exc, keep = ex.c()
    J = np.zeros((2, grid.n_cells))
    with pytest.raises(ValueError, match="parameter fields"):
        capi.check(capi.lib().lt_jacobian(pc.handle, capi.C.byref(exc), capi.dptr(J), None))


def test_direct_mode_matches_oracle_direct():
    cfg, lk, ls, grid, ops = fd_case(2, (48, 40))
    p = L.ShiftedPencil(L.Grid(tuple(cfg.shape), cfg.h), lk, ls)
    contour = otal.build_contour(cfg.n_quad, cfg.times[2])
    shifts = list(contour.nodes)
    b = np.stack([ofd.point_weights(grid, q) for q in cfg.sources[:3]]).astype(np.complex128)
    got = L.solve_shifted_direct(p, b, shifts)
    opencil = oss.ShiftedPencil(ops.stiffness, ops.mass)
    for r in range(3):
        ref = oss.solve_shifted_direct(opencil, b[r], shifts)
        for k in range(len(shifts)):
            assert rel(got[r][:, k], ref[:, k]) <= 1e-10
    # SolverConfig(kind=direct) through the forward driver
    prob = L.ForwardProblem(b[0].real, 1e-4, None, cfg.times[:2], cfg.n_quad)
    sol = L.solve_forward(p, prob, L.SolverConfig(kind="direct"))
    oref = ofw.solve_forward(ofw.ForwardProblem(ops.stiffness, ops.mass, b[0].real, 1e-4, None, cfg.times[:2],
                                                cfg.n_quad), ofw.SolverConfig(kind="direct"))
    assert rel(sol.heads, oref.heads) <= 1e-9
    for d in sol.diagnostics:
        assert d.all_converged and max(d.shift_residuals) <= 1e-10


def test_kept_basis_arnoldi_relation_and_residual_estimate():
    """FlexibleBasisState (hpp:63-74): V orthonormal, the flexible Arnoldi relation
    (K + zM) U = V Hbar(z; T) (acceptance 7), and residual_estimate equal to the
    explicit FOM residual."""
    cfg, lk, ls, grid, ops = fd_case(0, (32, 32))
    p = L.ShiftedPencil(L.Grid(tuple(cfg.shape), cfg.h), lk, ls)
    contour = otal.build_contour(cfg.n_quad, cfg.times[1])
    shifts = list(contour.nodes)
    sched, gs = _schedule(shifts)
    b = ofd.point_weights(grid, (0.37, 0.61)).astype(np.complex128)
    res = L.solve_shifted_flexible(p, b, shifts, gs, L.ShiftedSolveOptions(variant="fom", keep_basis=True))
    st = res.basis
    m = st.steps()
    assert m == res.iterations and m >= 2
    assert np.linalg.norm(st.V.conj().T @ st.V - np.eye(m + 1)) <= 1e-8
    A = lambda z: ops.stiffness + z * ops.mass  # noqa: E731
    for z in [shifts[0], shifts[5], 0.3 - 0.1j]:
        lhs = A(z) @ st.U
        rhs = st.V @ st.shifted_hessenberg(z)
        scale = (sp.linalg.norm(ops.stiffness) + abs(z) * sp.linalg.norm(ops.mass)) * np.linalg.norm(st.U)
        assert np.linalg.norm(lhs - rhs) <= 1e-10 * scale
    for k in (0, 7, 15):
        hz = st.shifted_hessenberg(shifts[k])[:m, :m]
        e1 = np.zeros(m, dtype=complex)
        e1[0] = st.beta
        y = np.linalg.solve(hz, e1)
        eta = L.residual_estimate(st, shifts[k], y)
        explicit = np.linalg.norm(b - A(shifts[k]) @ (st.U @ y))
        assert abs(eta - explicit) <= 1e-8 * explicit + 1e-12 * np.linalg.norm(b)  # to the rounding floor
    assert L.residual_estimate(st, st.taus[m - 1], y) == 0.0
    with pytest.raises(ValueError):
        L.residual_estimate(st, shifts[0], y[:-1])


def test_not_converged_paths():
    cfg, lk, ls, grid, ops = fd_case(0, (32, 32))
    p = L.ShiftedPencil(L.Grid(tuple(cfg.shape), cfg.h), lk, ls)
    contour = otal.build_contour(cfg.n_quad, cfg.times[0])
    shifts = list(contour.nodes)
    sched, gs = _schedule(shifts)
    b = ofd.point_weights(grid, cfg.sources[0]).astype(np.complex128)
    # run_flexible never throws: best-effort iterates, all_converged false (cpp:255-285)
    res = L.solve_shifted_flexible(p, b, shifts, gs, L.ShiftedSolveOptions(maxit=1))
    ref = oss.solve_shifted_flexible(oss.ShiftedPencil(ops.stiffness, ops.mass), b, shifts, sched,
                                     oss.ShiftedSolveOptions(maxit=1))
    assert not res.all_converged and res.unconverged() == ref.unconverged()
    for k in res.unconverged():
        assert rel(res.solutions[:, k], ref.solutions[:, k]) <= 1e-8
    # the drivers raise ConvergenceError with the shift indices (forward.cpp:68)
    prob = L.ForwardProblem(b.real, 1e-4, None, cfg.times[:1], cfg.n_quad)
    with pytest.raises(capi.ConvergenceError) as e:
        L.solve_forward(p, prob, L.SolverConfig(maxit=1))
    assert e.value.unconverged_shifts == ref.unconverged()
    # a 2-D pencil whose multigrid inner solve cannot reach its floor falls back to the exact
    # banded LU (band.cu): the solve is exact
    p.set_inner_tolerance(1e-12, 1)
    u = p.factorization(sched.taus[0]).solve(np.stack([b, 2 * b]))
    ref = spla.splu((ops.stiffness + sched.taus[0] * ops.mass).tocsc()).solve(b)
    assert rel(u[0], ref) <= 1e-12 and rel(u[1], 2 * ref) <= 1e-12
    # a 3-D pencil has no banded fallback: LT_ERR_NOT_CONVERGED with the right-hand sides
    cfg3, lk3, ls3, grid3, ops3 = fd_case(4, (12, 10, 8))
    p3 = L.ShiftedPencil(L.Grid(tuple(cfg3.shape), cfg3.h), lk3, ls3)
    b3 = ofd.point_weights(grid3, (0.5, 0.4, 0.3)).astype(np.complex128)
    p3.set_inner_tolerance(1e-12, 1)
    with pytest.raises(capi.ConvergenceError) as e:
        p3.factorization(sched.taus[0]).solve(np.stack([b3, 2 * b3]))
    assert e.value.unconverged_shifts == [0, 1]
    with pytest.raises(capi.ConvergenceError):
        L.solve_shifted_direct(p3, b3, shifts[:2])
    # ... and inside FGMRES-Sh the failed preconditioner is a FactorizationError
    with pytest.raises(capi.FactorizationError):
        L.solve_shifted_flexible(p3, b3, shifts, gs)


@pytest.mark.parametrize("mesh_n", [41, 101])
def test_banded_exact_shift_and_invert_for_indefinite_2d_shifts(mesh_n):
    """Strongly indefinite shifts (the paper's t = 1 min on the 100 m square, Re tau = -0.83)
    defeat the multigrid V-cycle; 2-D pencils take the exact banded LU instead (band.cu), cached
    by tau, identical to the reference's sparse LU (factorization.cpp:14-33)."""
    rng = np.random.default_rng(mesh_n)
    mesh = fem.build_mesh(mesh_n, 100.0)
    lk = np.log(1e-4) + 1.3 * rng.standard_normal(mesh.n_elements())
    ls = np.full(mesh.n_elements(), np.log(1e-5))
    ops = fem.assemble(mesh, np.exp(lk), np.exp(ls))
    p = L.ShiftedPencil(L.build_mesh(mesh_n, 100.0), lk, ls)
    tau = -0.8312938858819381 + 0.5401183169684252j
    v = rng.standard_normal((3, ops.n_free())) + 1j * rng.standard_normal((3, ops.n_free()))
    A = (ops.stiffness + tau * ops.mass).tocsc()
    lu = spla.splu(A, permc_spec="COLAMD")
    u = p.factorization(tau).solve(v)
    for r in range(3):
        assert rel(u[r], lu.solve(v[r])) <= 1e-10
    ua = p.factorization(tau).solve_adjoint(v[0])
    assert rel(ua, spla.splu((ops.stiffness + np.conj(tau) * ops.mass).tocsc()).solve(v[0])) <= 1e-10


def test_pooled_forty_times_over_256_shifts_per_item():
    """solve_forward_batch with 40 times x 10 shifts = 400 pooled shifts per item (more than
    one 256-shift window of the fused verification kernel)."""
    cfg, lk, ls, grid, ops = fd_case(0, (40, 40))
    p = L.ShiftedPencil(L.Grid(tuple(cfg.shape), cfg.h), lk, ls)
    times = list(np.linspace(2400.0, 3600.0, 40))
    b = ofd.point_weights(grid, (0.5, 0.5))
    prob = L.ForwardProblem(b, 1e-4, None, times, 20)
    got = L.solve_forward_batch(p, prob)
    ref = ofw.solve_forward_batch(ofw.ForwardProblem(ops.stiffness, ops.mass, b, 1e-4, None, times, 20))
    assert rel(got.heads, ref.heads) <= 1e-8
    assert got.diagnostics[0].iterations == ref.diagnostics[0].iterations
    assert len(got.diagnostics[0].shift_residuals) == 10
    assert all(d.all_converged for d in got.diagnostics)


def test_cpp_mirror_on_device(tmp_path):
    """include/laptomo/laptomo.hpp end to end on the device (examples/cpp_mirror_device_check.cpp):
    field and (K, M) pencils, flexible and direct solves, the kept basis and residual_estimate,
    solve_forward and the ConvergenceError path, against the oracle."""
    cfg, lk, ls, grid, ops = fd_case(0, (48, 40))
    src = ofd.point_weights(grid, cfg.sources[0])
    time = cfg.times[1]
    n = grid.n_cells
    K, M = sp.csr_matrix(ops.stiffness), sp.csr_matrix(ops.mass)
    inp, out = tmp_path / "in.bin", tmp_path / "out.bin"
    with open(inp, "wb") as f:
        np.array(cfg.shape, dtype=np.int32).tofile(f)
        np.array([cfg.h]).tofile(f)
        lk.astype(np.float64).tofile(f)
        ls.astype(np.float64).tofile(f)
        for A in (K, M):
            np.array([A.nnz], dtype=np.int64).tofile(f)
            A.indptr.astype(np.int64).tofile(f)
            A.indices.astype(np.int64).tofile(f)
            A.data.astype(np.float64).tofile(f)
        src.astype(np.float64).tofile(f)
        np.array([time]).tofile(f)
    exe = tmp_path / "check"
    libdir = ROOT / "paper_1409_2556_b200" / "_lib"
    subprocess.run(["g++", "-std=c++17", "-O2", f"-I{ROOT / 'include'}", str(ROOT / "examples" / "cpp_mirror_device_check.cpp"),
                    f"-L{libdir}", "-llaptomo_gpu", f"-Wl,-rpath,{libdir}", "-o", str(exe)], check=True)
    run = subprocess.run([str(exe), str(inp), str(out)], check=True, capture_output=True, text=True)
    assert run.stdout.startswith("ok")
    raw = np.fromfile(out, dtype=np.float64)
    nh = 16
    cplx = raw[: 2 * n * (2 * nh + 3)].view(np.complex128)
    x_field = cplx[: n * nh].reshape(nh, n).T
    x_csr = cplx[n * nh: 2 * n * nh].reshape(nh, n).T
    x_dir = cplx[2 * n * nh:].reshape(3, n).T
    rest = raw[2 * n * (2 * nh + 3):]
    eta, heads, tail = rest[: 2 * nh].reshape(nh, 2), rest[2 * nh: 2 * nh + n], rest[2 * nh + n:]
    contour = otal.build_contour(32, time)
    shifts = list(contour.nodes)
    sched = oss.select_preconditioner_shifts(shifts)
    opencil = oss.ShiftedPencil(ops.stiffness, ops.mass)
    oref = oss.solve_shifted_flexible(opencil, src.astype(complex), shifts, sched)
    direct = oss.solve_shifted_direct(opencil, src.astype(complex), shifts[:3])
    for k in range(nh):
        assert rel(x_field[:, k], oref.solutions[:, k]) <= 1e-8
        assert rel(x_csr[:, k], oref.solutions[:, k]) <= 1e-8
    assert rel(x_dir, direct) <= 1e-10
    # |eta| equals the explicit FOM residual (to its rounding floor ~1e-12 ||b||)
    assert np.all(np.abs(eta[:, 0] - eta[:, 1]) <= 1e-7 * eta[:, 1] + 1e-12 * np.linalg.norm(src))
    fref = ofw.solve_forward(ofw.ForwardProblem(ops.stiffness, ops.mass, src, 1e-4, None, [time], 32))
    assert rel(heads, fref.heads[:, 0]) <= 1e-8
    assert tail[0] >= 1 and tail[1] >= 2
