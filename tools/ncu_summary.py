"""Key metrics of an `ncu --set full` report, one row per kernel launch, as markdown.

usage: ncu -i report.ncu-rep --page raw --csv > raw.csv; python tools/ncu_summary.py raw.csv
"""
import csv
import sys

METRICS = [
    ("duration us", "gpu__time_duration.sum", 1e-3),
    ("DRAM read MB", "dram__bytes_read.sum", None),
    ("DRAM GB/s", "dram__bytes_read.sum.per_second", None),
    ("DRAM % peak", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", None),
    ("issue active %", "sm__inst_issued.avg.pct_of_peak_sustained_active", None),
    ("warps active %", "sm__warps_active.avg.pct_of_peak_sustained_active", None),
    ("L1 wavefronts smem", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", None),
    ("smem bank conflicts", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", None),
    ("global RED requests", "lts__t_requests_srcunit_tex_op_red.sum", None),
    ("warp instructions", "smsp__inst_executed.sum", None),
    ("registers", "launch__registers_per_thread", None),
]
STALLS = ["long_scoreboard", "short_scoreboard", "wait", "barrier", "not_selected", "selected",
          "math_pipe_throttle", "branch_resolving", "no_instructions", "lg_throttle", "mio_throttle"]


def num(v):
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return None


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    h, units = rows[0], rows[1]
    print("| kernel | " + " | ".join(m[0] for m in METRICS) + " | top stalls (pc samples) |")
    print("|---|" + "---:|" * len(METRICS) + "---|")
    for r in rows[2:]:
        d = dict(zip(h, r))
        name = d.get("Kernel Name", "?").split("(")[0].replace("<unnamed>::", "").replace("void ", "")
        cells = []
        for label, key, scale in METRICS:
            v = num(d.get(key, ""))
            u = units[h.index(key)] if key in h else ""
            if v is None:
                cells.append("-")
                continue
            if key == "gpu__time_duration.sum":
                v = {"nsecond": 1e-3, "ns": 1e-3, "msecond": 1e3, "ms": 1e3}.get(u, 1.0) * v
            if key == "dram__bytes_read.sum":
                v = v / 1e6 if u == "byte" else (v * 1e3 if u == "Gbyte" else v)
            if key == "dram__bytes_read.sum.per_second":
                v = v * 1e3 if u == "Tbyte/s" else v
            cells.append("%.4g" % v)
        st = []
        for s in STALLS:
            v = num(d.get("smsp__pcsamp_warps_issue_stalled_" + s, ""))
            if v:
                st.append((v, s))
        tot = sum(v for v, _ in st) or 1
        top = ", ".join("%s %d%%" % (s, round(100 * v / tot)) for v, s in sorted(st, reverse=True)[:4])
        print("| %s | %s | %s |" % (name, " | ".join(cells), top))


if __name__ == "__main__":
    main()
