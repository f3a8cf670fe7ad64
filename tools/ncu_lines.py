"""Per-CUDA-source-line warp stall samples from
`ncu -i rep --page source --csv --print-source cuda,sass -k <kernel> -c 1`
(profiling helper): hottest source lines and their SASS lines' top stall reasons."""
import csv
import sys


def main(path, top=25):
    rows = list(csv.reader(open(path)))
    cur, hdr, out = None, None, []
    last = None
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if len(r) >= 2 and r[0] == "Line No":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        if r[0].isdigit():
            last = [float(r[4] or 0), cur, int(r[0]), r[1].strip()[:80], {}]
            out.append(last)
        elif last is not None and r[2].startswith("0x"):
            for i, c in enumerate(hdr):
                if c.startswith("stall_") and "Not Issued" not in c:
                    try:
                        last[4][c[6:]] = last[4].get(c[6:], 0) + float(r[i] or 0)
                    except ValueError:
                        pass
    tot = sum(x[0] for x in out) or 1.0
    out.sort(key=lambda x: -x[0])
    for s, f, ln, src, st in out[:top]:
        why = sorted(st.items(), key=lambda kv: -kv[1])[:2]
        print(f"{s / tot * 100:5.1f}% {f}:{ln:<5} {src:80s} {[k for k, v in why if v]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
