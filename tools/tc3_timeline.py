"""Summarise the tc3 timeline marks of CTA 0 (stderr of tools/tc_timeline.py c5) (dev helper)."""
import re, sys
txt = open(sys.argv[1]).read()
m = re.findall(r"(\d+):(-?\d+)", txt.split("[timeline]")[-1])
d = {int(k): int(v) for k, v in m}
def g(k): return d.get(k)
for j in range(2):
    row = []
    for kb in range(16):
        b = 1000 + 64 * j + 4 * kb
        w0, w1, h, l = g(b), g(b + 1), g(b + 2), g(b + 3)
        e0, e1 = g(2000 + 64 * j + 2 * kb), g(2001 + 64 * j + 2 * kb)
        f0, f1, f2, f3 = (g(1500 + 64 * j + 4 * kb + i) for i in range(4))
        x0, x1 = g(1700 + 64 * j + 2 * kb), g(1701 + 64 * j + 2 * kb)
        if x0 is not None: row.append(f"   exec L1: {x0}->{x1} ({x1 - x0})")
        row.append(f"kb{kb}: A-wait {w0}->{w1} group landed {h} issued {l} | L0epi {e0}->{e1}")
    print(f"chunk {j}:"); print("\n".join("  " + r for r in row))
    print(f"  D1 commit {g(1200 + j)}, D1 seen by epi {g(3100 + j)}")
    for c in range(8):
        print(f"  L2 c{c}: A2 wait {g(1300 + 16 * j + 2 * c)}->{g(1301 + 16 * j + 2 * c)}  epi pub {g(3001 + 32 * j + 2 * c)}")
print("D2 seen", g(3200))

print("producer groups (step 3, chunk 0): start / waited / issued")
print("\n".join(f"e{e}: start {g(3300 + 3 * e)} waited {g(3301 + 3 * e)} issued {g(3302 + 3 * e)}" for e in range(40)))
