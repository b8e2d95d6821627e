"""Summarise an ncu '--page source --csv --print-source sass' export: total
warp instructions, and instruction counts per contiguous address region
(region boundaries at branch targets are approximated by a window size)."""
import csv, sys

def load(p):
    rows = list(csv.reader(open(p)))
    hdr = rows[1]
    ia, isrc, iex, isamp = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    ith = hdr.index("Avg. Threads Executed")
    out = []
    for r in rows[2:]:
        if len(r) <= iex:
            continue
        try:
            out.append((int(r[ia], 16), r[isrc].strip(), int(r[iex]), int(r[isamp]), float(r[ith])))
        except ValueError:
            pass
    return out

if __name__ == "__main__":
    ins = load(sys.argv[1])
    base = ins[0][0]
    tot = sum(x[2] for x in ins)
    samp = sum(x[3] for x in ins)
    print("total warp instr %.3e, samples %d" % (tot, samp))
    thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.002
    for a, s, e, sm, th in ins:
        if e >= thr * tot / 10 or sm >= thr * samp:
            print("%05x %10d %5.1f%% samp %5.2f%% thr %4.1f  %s" % (a - base, e, 100 * e / tot, 100 * sm / max(samp, 1), th, s[:70]))
