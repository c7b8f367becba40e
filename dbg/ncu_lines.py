"""Aggregate an ncu source page (--print-source cuda,sass CSV) by CUDA source line:
share of executed warp instructions and of stall samples per line."""
import csv
import sys


def main(path, top=25):
    rows = list(csv.reader(open(path)))
    cur = hdr = None
    agg = {}
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r[0] == "Function Name":
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r[0].strip().isdigit():
            continue
        d = dict(zip(hdr, r))
        try:
            e = float(d.get("Instructions Executed", "") or 0)
            smp = float(d.get("Warp Stall Sampling (All Samples)", "") or 0)
        except ValueError:
            continue
        key = (cur, int(r[0]))
        a = agg.setdefault(key, [0.0, 0.0, r[1]])
        a[0] += e
        a[1] += smp
    te = sum(v[0] for v in agg.values()) or 1
    ts = sum(v[1] for v in agg.values()) or 1
    print("total warp instructions %.3g, stall samples %.0f" % (te, ts))
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print("%5.1f%% inst %5.1f%% stall  %s:%d  %s" % (100 * v[0] / te, 100 * v[1] / ts, k[0], k[1], v[2].strip()[:80]))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
