"""Oracle pinning against the reference's own tests that exist for the operator
definition: tests/test_mesh.cpp:12-115 and tests/test_assembly.cpp:84-193
(restated in Python on the oracle's P1 mesh/assembly)."""
import math

import numpy as np
import pytest
import scipy.sparse.linalg as spla

from oracle import fem


def test_smallest_structured_grid():  # test_mesh.cpp:12-17
    m = fem.build_mesh(2, 1.0)
    assert m.n_nodes() == 4 and m.n_elements() == 2 and len(m.dirichlet_nodes) == 4


def test_reference_benchmark_grid():  # test_mesh.cpp:19-24
    m = fem.build_mesh(101, 100.0)
    assert m.n_nodes() == 10201 and m.n_elements() == 20000
    assert len(m.dirichlet_nodes) == 4 * 101 - 4


def test_areas_tessellate():  # test_mesh.cpp:26-35
    m = fem.build_mesh(3, 1.0)
    a = fem.element_areas(m)
    assert np.all(a > 0) and abs(a.sum() - 1.0) <= 1e-14


def test_dirichlet_nodes_are_boundary():  # test_mesh.cpp:37-46
    m = fem.build_mesh(5, 2.0)
    x, y = m.nodes[:, 0], m.nodes[:, 1]
    on = (x == 0) | (y == 0) | (x == 2.0) | (y == 2.0)
    assert set(np.flatnonzero(on)) == set(m.dirichlet_nodes)


def test_invalid_mesh_arguments():  # test_mesh.cpp:48-51
    with pytest.raises(ValueError):
        fem.build_mesh(1, 1.0)
    with pytest.raises(ValueError):
        fem.build_mesh(3, 0.0)


def test_point_on_node_is_unit_vector():  # test_mesh.cpp:53-66
    m = fem.build_mesh(5, 4.0)
    w = fem.point_source(m, 2.0, 3.0)
    nz = np.flatnonzero(w)
    assert len(nz) == 1 and np.allclose(m.nodes[nz[0]], [2.0, 3.0]) and w[nz[0]] == pytest.approx(1.0)


def test_centroid_equal_weights():  # test_mesh.cpp:68-81
    m = fem.build_mesh(4, 3.0)
    c = fem.element_centroids(m)[5]
    w = fem.point_source(m, c[0], c[1])
    nz = np.flatnonzero(w)
    assert len(nz) == 3 and np.allclose(w[nz], 1 / 3, rtol=1e-12) and abs(w.sum() - 1) <= 1e-14


def test_partition_of_unity_and_linear_completeness():  # test_mesh.cpp:83-101
    m = fem.build_mesh(7, 10.0)
    for x in (0.37, 5.0, 9.99):
        for y in (0.01, 4.2, 8.88):
            w = fem.point_source(m, x, y)
            assert w.min() >= 0 and abs(w.sum() - 1) <= 1e-13 and np.count_nonzero(w) <= 3
            assert abs(w @ m.nodes[:, 0] - x) <= 1e-12 * max(1, x)
            assert abs(w @ m.nodes[:, 1] - y) <= 1e-12 * max(1, y)


def test_centre_source_hits_centre_node():  # test_mesh.cpp:103-109
    m = fem.build_mesh(101, 100.0)
    w = fem.point_source(m, 50.0, 50.0)
    assert np.count_nonzero(w) == 1 and w[50 * 101 + 50] == pytest.approx(1.0)


def test_point_outside_rejected():  # test_mesh.cpp:111-115
    m = fem.build_mesh(4, 1.0)
    with pytest.raises(ValueError):
        fem.point_source(m, -0.1, 0.5)
    with pytest.raises(ValueError):
        fem.point_source(m, 0.5, 1.2)


def test_zero_row_sums():  # test_assembly.cpp:84-91
    m = fem.build_mesh(6, 2.5)
    K, _ = fem.assemble_full(m, np.ones(m.n_elements()), np.full(m.n_elements(), 1e-5))
    assert np.max(np.abs(K.toarray().sum(axis=1))) <= 1e-12


def test_mass_conserves_storativity():  # test_assembly.cpp:93-100
    m = fem.build_mesh(5, 3.0)
    _, M = fem.assemble_full(m, np.ones(m.n_elements()), np.full(m.n_elements(), 2.5e-4))
    assert M.toarray().sum() == pytest.approx(2.5e-4 * 9.0, rel=1e-12)


def _stiffness_quadrature_oracle(mesh, i, j):
    """Independent element integration (test_assembly.cpp:17-80): basis through
    barycentric coordinates, central-difference gradients, midpoint rule on a uniform
    sub-triangulation."""
    total = 0.0
    sub = 4
    step = 1e-6 * mesh.side_length
    for e, el in enumerate(mesh.elements):
        li = [v for v in range(3) if el[v] == i]
        lj = [v for v in range(3) if el[v] == j]
        if not li or not lj:
            continue
        p0, p1, p2 = (mesh.nodes[el[v]] for v in range(3))
        Amat = np.column_stack([p1 - p0, p2 - p0])
        Ainv = np.linalg.inv(Amat)
        area = fem.element_areas(mesh)[e]

        def basis(which, x):
            l12 = Ainv @ (x - p0)
            return [1 - l12[0] - l12[1], l12[0], l12[1]][which]

        def grad(which, x):
            g = np.zeros(2)
            for d in range(2):
                xp, xm = x.copy(), x.copy()
                xp[d] += step
                xm[d] -= step
                g[d] = (basis(which, xp) - basis(which, xm)) / (2 * step)
            return g

        s3 = 3.0 * sub
        pts = []
        for a in range(sub):
            for b in range(sub - a):
                pts.append(((3 * a + 1) / s3, (3 * b + 1) / s3))
                if a + b <= sub - 2:
                    pts.append(((3 * a + 2) / s3, (3 * b + 2) / s3))
        for b1, b2 in pts:
            x = p0 + b1 * (p1 - p0) + b2 * (p2 - p0)
            total += area / sub ** 2 * grad(li[0], x) @ grad(lj[0], x)
    return total


def test_stiffness_matches_quadrature_oracle():  # test_assembly.cpp:102-113
    m = fem.build_mesh(2, 1.0)
    K, _ = fem.assemble_full(m, np.ones(2), np.ones(2))
    Kd = K.toarray()
    for i in range(4):
        for j in range(4):
            assert Kd[i, j] == pytest.approx(_stiffness_quadrature_oracle(m, i, j), rel=1e-10, abs=1e-10)


def test_symmetric_and_definite():  # test_assembly.cpp:115-137
    m = fem.build_mesh(7, 4.0)
    e = np.arange(m.n_elements())
    ops = fem.assemble(m, 1e-4 * np.exp(np.sin(0.7 * e)), 1e-5 * (1 + 0.3 * np.cos(1.3 * e)))
    K, M = ops.stiffness.toarray(), ops.mass.toarray()
    assert np.max(np.abs(K - K.T)) <= 1e-12 * np.max(np.abs(K))
    assert np.max(np.abs(M - M.T)) <= 1e-12 * np.max(np.abs(M))
    assert np.linalg.eigvalsh(K).min() > 0 and np.linalg.eigvalsh(M).min() > 0


def test_patch_test():  # test_assembly.cpp:139-146
    m = fem.build_mesh(9, 5.0)
    K, _ = fem.assemble_full(m, np.full(m.n_elements(), 3.7), np.ones(m.n_elements()))
    kv = K @ np.ones(m.n_nodes())
    assert np.max(np.abs(kv)) <= 1e-12 * np.max(np.abs(K.toarray()))


def test_field_preconditions():  # test_assembly.cpp:148-155
    m = fem.build_mesh(3, 1.0)
    k = np.ones(m.n_elements())
    s = np.ones(m.n_elements())
    with pytest.raises(ValueError):
        fem.assemble(m, k[:3], s)
    k[2] = 0.0
    with pytest.raises(ValueError):
        fem.assemble(m, k, s)


def test_manufactured_second_order():  # test_assembly.cpp:157-193
    def err(n):
        m = fem.build_mesh(n, 1.0)
        ops = fem.assemble(m, np.ones(m.n_elements()), np.ones(m.n_elements()))
        c = fem.element_centroids(m)
        f = 2 * math.pi ** 2 * np.sin(math.pi * c[:, 0]) * np.sin(math.pi * c[:, 1])
        share = f * fem.element_areas(m) / 3
        load = np.zeros(m.n_nodes())
        for v in range(3):
            np.add.at(load, m.elements[:, v], share)
        phi = spla.spsolve(ops.stiffness.tocsc(), ops.restrict_to_free(load))
        xy = m.nodes[ops.free_nodes]
        e = phi - np.sin(math.pi * xy[:, 0]) * np.sin(math.pi * xy[:, 1])
        return math.sqrt(e @ (ops.mass @ e))

    e21, e41, e81 = err(21), err(41), err(81)
    assert math.log2(e21 / e41) >= 1.8 and math.log2(e41 / e81) >= 1.8
