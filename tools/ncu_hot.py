"""Summarise an `ncu --page source --csv` dump: hottest SASS lines by warp
stall samples with their top stall reasons (profiling helper)."""
import csv
import sys


def main(path, top=12):
    rows = list(csv.reader(open(path)))
    h = rows[1]
    body = [x for x in rows[2:] if len(x) == len(h) and x[0] != "Address" and x[0] != "Kernel Name"]
    si = h.index("Warp Stall Sampling (All Samples)")
    stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
    tot = sum(float(x[si] or 0) for x in body) or 1.0
    agg = {}
    for x in body:
        for i in stall_cols:
            agg[h[i]] = agg.get(h[i], 0) + float(x[i] or 0)
    print("stalls:", ", ".join(f"{k[6:]}={v / tot * 100:.0f}%" for k, v in
                               sorted(agg.items(), key=lambda kv: -kv[1])[:6]))
    body.sort(key=lambda x: -float(x[si] or 0))
    for x in body[:top]:
        st = sorted(((float(x[i] or 0), h[i][6:]) for i in stall_cols), reverse=True)[:2]
        print(f"{float(x[si]) / tot * 100:5.1f}% {x[0]} {x[1][:70]:70s} {st}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 12)
