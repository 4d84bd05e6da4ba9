"""profiles/traffic.json from ncu --set full summaries (scripts/ncu_summary.py --json): the DRAM
bytes (dram__bytes_read.sum + dram__bytes_write.sum) of one launch of each profiled kernel, keyed
by the library's profile names (the names bench.py's kernel_breakdown uses), so that bench.py
can fill `roofline.traffic` for whichever kernel dominates a run.

  python scripts/make_traffic.py profiles/r2_ncu_inner_v1.json profiles/r2_ncu_outer_v1.json

The captures are of BASELINE configs[4] (128^3, 80 items): scripts/perf_inner.py 4 80 for the
inner-solve kernels and scripts/perf_jac.py 128 1 for the outer / Jacobian kernels.  Kernels
that run on several multigrid levels are told apart by their traffic (a 128^3 launch moves
8x the bytes of a 64^3 one); the median over the captured launches of a name is kept.
"""
import json
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]

# ncu kernel name prefix -> profile name (or a function of the launch's DRAM bytes)
N128 = 128 ** 3 * 80  # cell-items of the finest level at configs[4]


def level(prefix, bytes_per_cell_item_min, coarse=None):
    def f(d):
        return f"{prefix}:l0" if d["traffic_bytes"] > bytes_per_cell_item_min * N128 else f"{coarse or prefix}:l1"
    return f


RULES = [
    ("mg_rb_kernel<0", level("mg_smooth", 2.0, "mg_smooth_coarse")),
    ("mg_rb_kernel<1", level("mg_residual", 4.0)),
    ("prolong_tma_kernel", level("mg_prolong", 3.0)),
    ("restrict_tma_kernel", level("mg_restrict", 1.5)),
    ("apply_tma2_kernel", "cocg_apply:operator"),
    ("pupdate_kernel", "cocg_vec:pupdate"),
    ("axpy_norm_kernel", "cocg_vec:axpy_norm"),
    ("copy_norm_kernel", "cocg_vec:copy_norm"),
    ("bottom_vcycle_kernel", "mg_bottom:fused"),
    ("mid_sweeps_kernel", "mg_smooth_coarse:l2"),
    ("rbpair_zm_kernel", "mg_smooth_coarse:l2"),
    ("residual_pair_zm_kernel", "mg_residual:l2"),
    ("jacobian_mma4_kernel", "jacobian"),
    ("expand_cm2_kernel", "expand"),
    ("verify_residual", "fgmres_verify:verify_residual"),
    ("mass_multidot", "fgmres_orth:mass_multidot"),
    ("gs_update", "fgmres_orth:gs_update"),
    ("multidot", "fgmres_orth:multidot"),
]


def main():
    per = {}
    for path in sys.argv[1:]:
        for d in json.load(open(path)):
            if "traffic_bytes" not in d:
                continue
            name = d["kernel"].replace("lt::", "").replace("(anonymous namespace)::", "")
            for prefix, rule in RULES:
                if name.startswith(prefix):
                    key = rule(d) if callable(rule) else rule
                    per.setdefault(key, []).append(d["traffic_bytes"])
                    break
    out = {k: statistics.median(v) for k, v in sorted(per.items())}
    json.dump(out, open(ROOT / "profiles" / "traffic.json", "w"), indent=1)
    for k, v in out.items():
        print(f"{k:32s} {v / 1e9:9.3f} GB per launch ({len(per[k])} launches)")


if __name__ == "__main__":
    main()
