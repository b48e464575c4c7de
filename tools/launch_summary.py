"""Summarise an ncu launch list (--csv --log-file, metrics gpu__time_duration.sum and
dram__bytes_read/write.sum) of `bench.py --steps 1`: the launches of the LAST bench step
(the launches after the previous k_compact up to the last k_compact that follows K1) to
profiles/<round>_launches_config<N>.json, and the K1 DRAM bytes per chp_reduce call to
profiles/k1_traffic_config<N>.json (bench.py reads it into roofline.traffic).

usage: python tools/launch_summary.py <csv> <config> <n> <round>
"""
import collections
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    path, config, n, rnd = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ix = {k: i for i, k in enumerate(h)}
    launches = collections.OrderedDict()
    for r in rows[1:]:
        if r[ix["ID"]] == "ID":
            continue
        key = int(r[ix["ID"]])
        d = launches.setdefault(key, {"kernel": r[ix["Kernel Name"]].split("(")[0].replace("<unnamed>::", "")
                                      .replace("void ", "")})
        d[r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
    # only this repo's kernels (bench.py's pre-timing torch sleep kernel is not part of a step)
    seq = [d for d in launches.values() if d["kernel"].startswith("k_")]
    # the last compaction that directly follows K1 (bench.py's hull leg compacts again)
    last = max(i for i, d in enumerate(seq)
               if d["kernel"].startswith("k_compact") and i > 0 and not seq[i - 1]["kernel"].startswith("k_compact"))
    prev = max((i for i, d in enumerate(seq[:last]) if d["kernel"].startswith("k_compact")), default=-1)
    step = seq[prev + 1:last + 1]
    tot = sum(d.get("gpu__time_duration.sum", 0) for d in step)
    out = []
    for d in step:
        t = d.get("gpu__time_duration.sum", 0)
        b = d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
        e = {"kernel": d["kernel"], "us": round(t / 1e3, 2), "dram_bytes": int(b), "share": round(t / tot, 3)}
        for key, name in (("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct"),
                          ("lts__t_requests_srcunit_tex_op_red.sum", "global_red_requests"),
                          ("lts__t_requests_srcunit_tex_op_atom.sum", "global_atom_requests"),
                          ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum", "smem_atom_wavefronts")):
            if key in d:
                e[name] = round(d[key], 1) if name == "dram_pct" else int(d[key])
        out.append(e)
    k1 = [d for d in out if not d["kernel"].startswith("k_compact")]
    k1_bytes = sum(d["dram_bytes"] for d in k1)
    summary = {
        "config": config, "n": n,
        "source": "ncu --metrics gpu__time_duration.sum, dram__bytes_read/write.sum, dram__throughput pct, "
                  "lts red/atom requests, smem atom wavefronts --clock-control none over bench.py --steps 1 "
                  "(cold, serialised launches: use the shares)",
        "step_launches": out, "step_us_sum": round(tot / 1e3, 1),
        "k1_share": round(sum(d["us"] for d in k1) * 1e3 / tot, 3),
        "k1_dram_bytes_per_call": k1_bytes, "algorithmic_bytes_per_call": 8 * n,
    }
    with open(os.path.join(ROOT, "profiles", f"{rnd}_launches_config{config}.json"), "w") as f:
        json.dump(summary, f, indent=1)
    with open(os.path.join(ROOT, "profiles", f"k1_traffic_config{config}.json"), "w") as f:
        json.dump({"config": config, "round": rnd, "dram_bytes_per_launch": k1_bytes,
                   "what": "sum of dram__bytes_read+write over the launches of one chp_reduce call, "
                           f"from profiles/{rnd}_launches_config{config}.json"}, f, indent=1)
    print(json.dumps(summary)[:400])


if __name__ == "__main__":
    main()
