"""Summarise ncu --set full reports (.ncu-rep) into one line per kernel: duration, DRAM
traffic, achieved bandwidth, SM/DRAM throughput, occupancy, registers, top stall reasons.

  python scripts/ncu_summary.py gpurun_out/r1v3_full_*.ncu-rep [--json profiles/traffic.json]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "time_us": "gpu__time_duration.sum",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "dram_pct": "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "occ_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "l2_hit": "lts__t_sector_hit_rate.pct",
    "fp64_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "issue_pct": "sm__inst_issued.avg.pct_of_peak_sustained_active",
    "l2_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1_pct": "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
    "mem_pct": "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "l2_sectors": "lts__t_sectors.sum",
    "l2_sectors_tex": "lts__t_sectors_srcunit_tex.sum",
    "smem_wavefronts": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "sm_cycles": "sm__cycles_elapsed.max",
    "tensor_pct": "sm__inst_executed_pipe_tensor.avg.pct_of_peak_sustained_active",
    "lsu_pct": "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smem_bytes": "launch__shared_mem_per_block_dynamic",
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-3, "us": 1, "ms": 1e3,
        "usecond": 1, "nsecond": 1e-3, "msecond": 1e3}


def summarise(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    res = []
    for v in rows[2:]:
        d = {"kernel": v[h.index("Kernel Name")].split("(")[0].replace("void ", "").replace("unnamed>::", "")}
        for k, m in KEYS.items():
            if m in h:
                i = h.index(m)
                try:
                    x = float(v[i].replace(",", ""))
                except ValueError:
                    continue
                d[k] = x * UNIT.get(u[i], 1) if k in ("time_us", "dram_read", "dram_write") else x
        stalls = {}
        for i, name in enumerate(h):
            if name.startswith("smsp__average_warps_issue_stalled_") and name.endswith("_per_issue_active.ratio"):
                try:
                    stalls[name[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = float(v[i])
                except ValueError:
                    pass
        d["top_stalls"] = sorted(stalls.items(), key=lambda kv: -kv[1])[:4]
        if "dram_read" in d and "time_us" in d:
            d["traffic_bytes"] = d["dram_read"] + d["dram_write"]
            d["dram_GBps"] = d["traffic_bytes"] / (d["time_us"] * 1e-6) / 1e9
        res.append(d)
    return res


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    js = sys.argv[sys.argv.index("--json") + 1] if "--json" in sys.argv else None
    if js:
        args = [a for a in args if a != js]
    allr = []
    for p in args:
        for d in summarise(p):
            allr.append(d)
            print(json.dumps({k: (round(x, 3) if isinstance(x, float) else x) for k, x in d.items()}))
    if js:
        json.dump(allr, open(js, "w"), indent=1)
