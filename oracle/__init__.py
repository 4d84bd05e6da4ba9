"""CPU oracle: a NumPy/SciPy restatement of the laptomo reference hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package
(`paper_1409_2556_b200/`) imports this package.  Only `tests/`,
`__graft_entry__.smoke()` and the `cpu_baseline` / `--impl reference` legs of
`bench.py` may import it, and only as the checker / the reported CPU baseline.

Why a restatement: the reference (`/root/reference/proj`, C++20) needs Eigen
3.4 (`CMakeLists.txt:22`, `find_package(Eigen3 3.4 REQUIRED)`), which is not
present in this image or on the GPU box, so it cannot be compiled here.
Each function cites the reference file:line it follows.  Eigen's
`SparseLU<COLAMD>` (`src/factorization.cpp:14-33`) is replaced by SuperLU with
COLAMD ordering (`scipy.sparse.linalg.splu(permc_spec="COLAMD")`), the same
supernodal-LU family; Eigen `HouseholderQR` / `PartialPivLU` small solves
(`src/shifted_solver.cpp:36-65`) by LAPACK zgeqrf / zgetrf through NumPy.

Pinning: the reference ships no golden vectors for this path (its hot-path
test files are absent, `tests/CMakeLists.txt:6-10`).  The oracle is pinned by
(a) the reference's own tests that do exist (`tests/test_mesh.cpp`,
`tests/test_assembly.cpp`), restated in `tests/test_oracle_fem.py`, and
(b) every known-answer example the reference SPEC gives for this path
(`SPEC.md:185-187, 255-290, 334-342, 397-421`), restated in
`tests/test_oracle_*.py`.  No reference binary can be run, so at the Eigen
boundary parity is pinned by these KATs only ("Oracle").
"""
