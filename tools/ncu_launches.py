"""Launch-list summary (profiling helper): the csv of
`ncu --metrics gpu__time_duration.sum --clock-control none --csv` grouped by
kernel, as markdown rows (launches, mean and total us), first-seen order."""
import csv
import sys


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 14 and r[12] == "gpu__time_duration.sum"]
    agg = {}
    for r in rows:
        name = r[4].replace("void ", "").replace("cnb::", "").split("(")[0][:70]
        v = float(r[14].replace(",", ""))
        us = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}[r[13]] * v
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += us
    print("| kernel | launches | mean us | total us |\n|---|---|---|---|")
    for k, (n, t) in agg.items():
        print(f"| {k} | {n} | {t / n:.1f} | {t:.1f} |")


if __name__ == "__main__":
    main(sys.argv[1])
