"""Summarise ncu raw-page CSV exports (tools/gpu/profile_all.sh) into
profiles/: per-kernel metrics JSON, DRAM traffic per stage (read by bench.py
for roofline.traffic) and a markdown table.

    python tools/ncu_summary.py [--tag r01e] gpurun_out/prof_c2_raw.csv gpurun_out/prof_c4_raw.csv
"""
import csv
import json
import os
import re
import sys

M = {
    "duration_ms": ("gpu__time_duration.sum", 1e-3),  # us -> ms (ncu raw reports usecond)
    "regs": ("launch__registers_per_thread", 1),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    "fma_pipe_pct": ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", 1),
    "fp64_pipe_pct": ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 1),
    "dram_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "dram_read_MB": ("dram__bytes_read.sum", None),
    "dram_write_MB": ("dram__bytes_write.sum", None),
    "inst_G": ("smsp__inst_executed.sum", 1e-9),
    "thread_inst_per_inst": ("smsp__thread_inst_executed_per_inst_executed.ratio", 1),
}


def short(name):
    n = re.sub(r"\(.*", "", name).replace("void ", "").replace("hgs::", "").replace("<unnamed>::", "")
    return n.strip()


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": short(r[hdr.index("Kernel Name")])}
        for k, (col, scale) in M.items():
            if col not in hdr:
                continue
            i = hdr.index(col)
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                continue
            u = units[i]
            if scale is None:  # bytes -> MB, unit-aware
                f = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u, 1e-6)
                v *= f
            elif k == "duration_ms":
                v *= {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}.get(u, 1e-3)
            else:
                v *= scale
            d[k] = round(v, 6)
        out.append(d)
    return out


def main():
    args = sys.argv[1:]
    tag = "r01b"
    if args and args[0] == "--tag":
        tag, args = args[1], args[2:]
    allk = []
    for p in args:
        cfg = "c4" if "c4" in os.path.basename(p) else "c2"
        for d in load(p):
            d["config"] = cfg
            allk.append(d)
    # first launch of each (config, kernel)
    seen, uniq = set(), []
    for d in allk:
        key = (d["config"], d["kernel"])
        if key in seen:
            continue
        seen.add(key)
        uniq.append(d)
    os.makedirs("profiles", exist_ok=True)
    json.dump(uniq, open("profiles/ncu_%s_kernels.json" % tag, "w"), indent=1)
    # per-stage DRAM traffic (bytes) of the config-2 kernels, as bench.py names the stages
    stage = {"composite_fwd": ["k_composite_fwd"], "composite_bwd": ["k_composite_bwd"],
             "chain_rule(+touched)": ["k_chain_rule"],
             "depth_keys+sort||preprocess_f64": ["k_depth_keys", "k_sort_plan", "k_onesweep<unsigned long long>",
                                                 "k_rank_scatter", "k_preprocess", "k_tile_counts"],
             "scan": ["k_scan_counts"],
             "binning(dup+tile sort+ranges)": ["k_duplicate", "k_radix_offsets", "k_onesweep<unsigned int>",
                                               "k_tile_ranges"]}
    tr = {"_source": "profiles/ncu_%s_kernels.json (ncu --set full, one launch each, config 2): " % tag +
                     "dram__bytes_read.sum + dram__bytes_write.sum per launch"}
    for st, pref in stage.items():
        b = sum((d.get("dram_read_MB", 0) + d.get("dram_write_MB", 0)) * 1e6 for d in uniq
                if d["config"] == "c2" and any(d["kernel"].startswith(x) for x in pref))
        tr[st] = int(b)
    json.dump(tr, open("profiles/traffic.json", "w"), indent=1)
    cols = ["duration_ms", "regs", "warps_active_pct", "issue_active_pct", "fma_pipe_pct", "fp64_pipe_pct",
            "dram_pct", "dram_read_MB", "dram_write_MB", "inst_G", "thread_inst_per_inst"]
    lines = ["| cfg | kernel | " + " | ".join(cols) + " |", "|" + "---|" * (len(cols) + 2)]
    for d in uniq:
        lines.append("| %s | %s | " % (d["config"], d["kernel"]) +
                     " | ".join(("%.3f" % d[c]) if isinstance(d.get(c), float) else str(d.get(c, "")) for c in cols) + " |")
    open("profiles/ncu_%s_table.md" % tag, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
