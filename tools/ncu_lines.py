"""Per-source-line instruction and stall-sample shares of one kernel from an
ncu report (--import-source on):  python tools/ncu_lines.py REP KERNEL_REGEX [N]"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 45
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kern,
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur, hdr, agg = None, None, {}


def num(x):
    try:
        return int(x.replace(",", ""))
    except ValueError:
        return 0


for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if len(r) > 2 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or not r[0]:
        continue
    ie = num(r[hdr.index("Instructions Executed")])
    sm = num(r[hdr.index("Warp Stall Sampling (All Samples)")])
    agg[(cur, num(r[0]))] = (ie, sm, r[1].strip()[:90])
tot = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
print("total warp instructions", tot, "stall samples", ts)
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print("%-20s %5d %6.2f%% inst %6.2f%% samp  %s" % (k[0], k[1], 100 * v[0] / tot, 100 * v[1] / ts, v[2]))
