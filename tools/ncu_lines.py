"""Top source lines by warp-stall samples from an ncu source-page CSV, with each
line's leading stall reasons (dev helper).

usage: ncu -i rep --page source --csv --print-source sass,cuda > src.csv
       python tools/ncu_lines.py src.csv [top] [file-substring]
"""
import csv
import sys


def main(path, top=40, only=None):
    rows = list(csv.reader(open(path)))
    fname, header, out = "?", None, []
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            header = r
            continue
        if header is None or not r or r[0] in ("", "Function Name"):
            continue
        d = dict(zip(header, r))
        try:
            s = int(d["Warp Stall Sampling (All Samples)"])
        except (KeyError, ValueError):
            continue
        stalls = {}
        for k, v in zip(header, r):
            if k.startswith("stall_") and "(Not Issued)" not in k:
                try:
                    stalls[k[6:]] = int(v)
                except ValueError:
                    pass
        out.append((s, fname, r[0], r[1][:80], d.get("Instructions Executed", ""), stalls))
    tot = sum(o[0] for o in out)
    print(f"total samples {tot}")
    for s, f, ln, src, ins, st in sorted(out, key=lambda o: -o[0]):
        if only and only not in f:
            continue
        top_st = ", ".join(f"{k} {100.0 * v / max(s, 1):.0f}%" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:3] if v)
        print(f"{100.0 * s / tot:5.1f}% {f}:{ln:>5} ins={ins:>10}  {src}\n        [{top_st}]")
        top -= 1
        if top == 0:
            break


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40, sys.argv[3] if len(sys.argv) > 3 else None)
