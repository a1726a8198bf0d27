"""Summarise ncu captures for profiles/ (run here, on the CPU box).

    python tools/ncu_summary.py --rep gpurun_out/prof.ncu-rep --launches gpurun_out/launches.csv \
        --cells 4194304 --out profiles/r1_v1.md

Per kernel: duration, DRAM bytes (read+write), algorithmic bytes
(64 B per cell per sweep), pipe utilisation, issue/occupancy and the top stall
reasons.  From the launch list: per-kernel launch count, mean duration and
share of device time.
"""
import argparse
import csv
import io
import json
import subprocess

KEYS = {
    "duration_us": "gpu__time_duration.sum",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "alu_pipe_pct": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "fma_pipe_pct": "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "sm__instruction_throughput.avg.pct_of_peak_sustained_active",
    "warps_active": "sm__warps_active.avg.per_cycle_active",
    "regs": "launch__registers_per_thread",
    "inst_executed": "smsp__inst_executed.sum",
    "sm_clock_hz": "smsp__cycles_elapsed.avg.per_second",
    "l1_hit_pct": "l1tex__t_sector_hit_rate.pct",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "l2_read_sectors_from_sm": "lts__t_sectors_srcunit_tex_op_read.sum",
}
UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1,
         "msecond": 1e3, "ns": 1e-3, "us": 1, "ms": 1e3, "s": 1e6,
         "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def num(v):
    return float(str(v).replace(",", ""))


def kernel_metrics(rep, cells):
    hdr, units, rows = raw_rows(rep)
    out = []
    for r in rows:
        m = {"kernel": r[hdr.index("Kernel Name")].split("(")[0].split("::")[-1]}
        for key, name in KEYS.items():
            if name in hdr:
                i = hdr.index(name)
                try:
                    m[key] = num(r[i]) * UNITS.get(units[i], 1)
                except ValueError:
                    pass
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((num(r[i]), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        m["top_stalls"] = [(s, round(v, 3)) for v, s in sorted(stalls, reverse=True)[:6]]
        if "dram_read" in m and "dram_write" in m:
            m["dram_bytes"] = m["dram_read"] + m["dram_write"]
        if "l2_read_sectors_from_sm" in m:
            m["l2_read_bytes_from_sm"] = 32 * m["l2_read_sectors_from_sm"]
        if cells and "sweep" in m["kernel"]:
            m["alg_bytes"] = 64 * cells
            m["thread_inst_per_cell"] = m.get("inst_executed", 0) * 32 / cells
        out.append(m)
    return out


def launch_shares(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    acc = {}
    for r in rows[1:]:
        k = r[ki].split("(")[0].split("::")[-1]
        t = num(r[vi]) * UNITS.get(r[ui], 1e-3)  # -> microseconds
        acc.setdefault(k, []).append(t)
    total = sum(sum(v) for v in acc.values())
    return {k: {"launches": len(v), "mean_us": sum(v) / len(v), "share": sum(v) / total}
            for k, v in acc.items()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep")
    ap.add_argument("--launches")
    ap.add_argument("--cells", type=int, default=0)
    ap.add_argument("--out", required=True)
    ap.add_argument("--title", default="")
    a = ap.parse_args()
    res = {}
    if a.rep:
        res["kernels"] = kernel_metrics(a.rep, a.cells)
    if a.launches:
        res["launch_list"] = launch_shares(a.launches)
    lines = [f"# {a.title or a.out}", "", "```json", json.dumps(res, indent=1), "```", ""]
    open(a.out, "w").write("\n".join(lines))
    print("\n".join(lines))


if __name__ == "__main__":
    main()
