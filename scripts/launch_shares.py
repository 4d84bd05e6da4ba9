"""Per-kernel shares of an ncu launch list (gpu__time_duration.sum per launch, CSV).

  python scripts/launch_shares.py gpurun_out/TAG_launches.csv profiles/r1_launch_shares_vN.json
"""
import collections
import csv
import json
import re
import sys


def main(src, dst):
    rows = list(csv.reader(open(src)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "us": 1e-3, "ms": 1.0}
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        try:
            v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-6)
        except ValueError:
            continue
        name = re.sub(r"\(.*", "", r[ki]).replace("void ", "").replace("(anonymous namespace)::", "")
        name = re.sub(r"^.*::", "", name) if "<" not in name else re.sub(r"^[^<]*::", "", name.split("<")[0]) + "<" + name.split("<", 1)[1]
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(a[1] for a in agg.values())
    out = {"source": f"{src} (ncu gpu__time_duration.sum, --clock-control none, the launches after a 10000-launch "
                     "warm-up skip; cold, serialised)",
           "total_ms": round(tot, 1), "launches": sum(a[0] for a in agg.values()),
           "shares": {k: {"launches": c, "ms": round(t, 2), "share": round(t / tot, 4)}
                      for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])}}
    json.dump(out, open(dst, "w"), indent=1)
    for k, v in list(out["shares"].items())[:12]:
        print(f"{v['share'] * 100:5.1f}% {v['ms']:9.2f} ms {v['launches']:6d}  {k}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
