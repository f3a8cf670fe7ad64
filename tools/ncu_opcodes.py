"""Tallies executed SASS instructions by opcode for every kernel of an ncu
report (the source page's per-instruction "Instructions Executed" column):
the evidence of warp-ballot / popc / match / redux use in the bitmap work.
    python tools/ncu_opcodes.py report.ncu-rep > profiles/<name>.md"""
import csv
import io
import re
import subprocess
import sys

FAMILIES = ["VOTE", "POPC", "REDUX", "MATCH", "SHFL", "FLO", "ATOM", "ATOMG", "RED", "LDG", "STG", "LDS", "STS",
            "BAR", "NANOSLEEP"]


def kernels(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    ki, ti = h.index("Kernel Name"), h.index("gpu__time_duration.sum")
    return [(r[ki], r[ti]) for r in rows[2:]]


def main(rep):
    ks = kernels(rep)
    print(f"# SASS opcode mix per kernel ({rep.split('/')[-1]})\n")
    print("warp instructions executed, by opcode family (one launch each)\n")
    print("| kernel | us | " + " | ".join(FAMILIES) + " | total |")
    print("|---" * (len(FAMILIES) + 3) + "|")
    for i, (name, us) in enumerate(ks):
        out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                              "--launch-skip", str(i), "--launch-count", "1"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        hdr = next(r for r in rows if "Instructions Executed" in r)
        si, ei = hdr.index("Source"), hdr.index("Instructions Executed")
        tally, total = {f: 0 for f in FAMILIES}, 0
        start = rows.index(hdr) + 1
        for r in rows[start:]:
            if len(r) <= ei or not r[ei].isdigit():
                continue
            n = int(r[ei])
            total += n
            op = re.sub(r"^@!?U?P\w+\s+", "", r[si].strip()).split(" ")[0].split(".")[0]
            if op in tally:
                tally[op] += n
        short = re.sub(r"\(.*", "", name).replace("void ", "")
        print(f"| {short} | {float(us):.1f} | " + " | ".join(str(tally[f]) for f in FAMILIES) + f" | {total} |")


if __name__ == "__main__":
    main(sys.argv[1])
