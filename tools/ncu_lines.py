"""Top source lines by warp-stall samples from an ncu source-page CSV (dev helper).

usage: ncu -i rep --page source --csv --print-source sass,cuda > src.csv
       python tools/ncu_lines.py src.csv [top]
"""
import csv
import sys


def main(path, top=40):
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
        stalls = {k: v for k, v in zip(header, r) if k.startswith("stall_") or "Stall" in k and "(" not in k}
        out.append((s, fname, r[0], r[1][:90], d.get("Instructions Executed", ""), stalls))
    tot = sum(o[0] for o in out)
    print(f"total samples {tot}")
    for s, f, ln, src, ins, _ in sorted(out, key=lambda o: -o[0])[:top]:
        print(f"{100.0 * s / tot:5.1f}% {f}:{ln:>5} ins={ins:>10}  {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
