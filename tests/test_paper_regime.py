"""The reference SPEC's paper-regime known answers for FGMRES-Sh (
acceptance 3-6) on the oracle: iteration counts in the paper's regime (§4; 100 m square,
P1 on build_mesh(101, 100), variance 1.6, t = 5 min, N_z = 40, tol 1e-10).  The committed counts
(tests/golden/paper_regime.json, scripts/paper_regime.py) are checked against the acceptance
bands, and the cheap cases are re-run here; tests/test_gpu_paper_regime.py holds the device to
the same counts."""
import json
from pathlib import Path

import pytest

G = json.loads((Path(__file__).resolve().parent / "golden" / "paper_regime.json").read_text())
PAPER_SINGLE, PAPER_FLEXIBLE = 126, 53  # Table 1, random field, variance 1.6


def check_bands(d):
    single, flexible = d["random_n101_t300"]
    # acceptance 3: flexible <= 0.75 single, both within [0.5x, 1.5x] of the paper's (126, 53)
    assert flexible <= 0.75 * single
    assert 0.5 * PAPER_SINGLE <= single <= 1.5 * PAPER_SINGLE
    assert 0.5 * PAPER_FLEXIBLE <= flexible <= 1.5 * PAPER_FLEXIBLE
    # acceptance 4: iterations(t = 20 min) < iterations(t = 1 min), both solvers, both fields
    for field in ("random", "franke"):
        for k in (0, 1):
            assert d[f"{field}_n101_t1200"][k] < d[f"{field}_n101_t60"][k]
    # acceptance 5: flexible counts on Franke variance 1.6 over n = 41, 101, 201 within 20%
    f = [d[f"franke_n{n}_t300"][1] for n in (41, 101, 201)]
    assert max(f) <= 1.2 * min(f)
    # acceptance 6: 40 pooled times in [40, 60] min: at most 45 iterations (paper: 27) and at
    # most 1.5x the single-time t = 50 min count
    assert d["random_pooled40"] <= 45
    assert d["random_pooled40"] <= 1.5 * d["random_n101_t3000"][1]


def test_committed_oracle_counts_meet_the_acceptance_bands():
    check_bands(G)


@pytest.mark.parametrize("case", ["franke_n41_t300", "random_n101_t300"])
def test_oracle_reproduces_the_committed_counts(case):
    import sys
    sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "scripts"))
    import paper_regime as PR
    field, n, t = case.split("_")
    assert list(PR.counts(field, float(t[1:]), int(n[1:]))) == G[case]
