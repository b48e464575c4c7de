"""Per-kernel SASS instruction mix of libchp_b200.so (cuobjdump -sass): counts of
the opcodes that show how each kernel does its work -- the streaming loads,
the shared-memory table accesses, global REDs / atomics, the packed 16-bit
compare, the bulk-copy ring -- as a markdown table (static counts in the
binary, not executed counts).

usage: python tools/sass_mix.py [lib.so] > profiles/<round>_sass_mix.md
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1505_00914_b200", "lib", "libchp_b200.so")

COLS = [
    ("LDG.E.NA.LTC256B.128", r"LDG\.E\.NA\.LTC256B\.128"),  # ld_stream: 128-bit, no L1 allocate, 256B L2 prefetch
    ("LDG.128 (other)", r"LDG\.E(?!\.NA\.LTC256B)[^ ]*\.128"),
    ("LDG.64 STRONG.GPU", r"LDG\.E\.64\.STRONG\.GPU"),  # L2-coherent slot reads (ld.cg / relaxed)
    ("LDS", r"\bLDS"),
    ("STS", r"\bSTS"),
    ("ATOMS", r"\bATOMS"),
    ("REDG.E.MIN", r"REDG\.E\.MIN"),
    ("ATOMG", r"\bATOMG"),
    ("VIMNMX.U16x2", r"VIMNMX[^ ]*U16x2"),
    ("VIADDMNMX", r"VIADDMNMX"),
    ("UBLKCP (TMA bulk)", r"UBLKCP"),
    ("SYNCS (mbarrier)", r"\bSYNCS"),
    ("STG", r"\bSTG"),
    ("BAR", r"\bBAR\b|\bBAR\."),
]


def demangle(name):
    try:
        out = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    except Exception:
        out = name
    out = out.replace("(anonymous namespace)::", "")
    return re.sub(r"\(.*", "", out)


def main():
    lib = sys.argv[1] if len(sys.argv) > 1 else LIB
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
    kernels = collections.OrderedDict()
    cur = None
    for line in sass.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = demangle(m.group(1))
            kernels[cur] = collections.Counter()
            continue
        if cur is None or "/*" not in line:
            continue
        ins = line.split("*/", 1)[1] if "*/" in line else line
        ins = ins.split(";")[0]
        if not ins.strip():
            continue
        kernels[cur]["total"] += 1
        for col, rx in COLS:
            if re.search(rx, ins):
                kernels[cur][col] += 1
    print("# SASS instruction mix of libchp_b200.so (static counts per kernel)\n")
    print("Built for sm_100a (`-gencode arch=compute_100a,code=sm_100a`); `cuobjdump -sass`, counted by "
          "`tools/sass_mix.py`. Static instruction counts in the binary, not executed counts.\n")
    print("| kernel | total | " + " | ".join(c for c, _ in COLS) + " |")
    print("|---|---:|" + "---:|" * len(COLS))
    for k, c in sorted(kernels.items()):
        if not c["total"]:
            continue
        print(f"| `{k}` | {c['total']} | " + " | ".join(str(c.get(col, 0)) for col, _ in COLS) + " |")


if __name__ == "__main__":
    main()
