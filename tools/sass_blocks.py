"""Per-basic-block executed-instruction breakdown of an ncu report's SASS
(blocks = runs of instructions with equal execution counts).

    python tools/sass_blocks.py gpurun_out/prof_X.ncu-rep [n]
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
idx = {k: i for i, k in enumerate(h)}
data = rows[2:]


def f(r, k):
    try:
        return float(r[idx[k]])
    except Exception:
        return 0.0


blocks, cur = [], None
for r in data:
    e = f(r, "Instructions Executed")
    src = r[idx["Source"]]
    if cur and abs(cur["e"] - e) < 0.5:
        cur["n"] += 1
        cur["src"].append(src)
    else:
        cur = {"e": e, "n": 1, "start": r[idx["Address"]][-5:], "src": [src]}
        blocks.append(cur)
tot = sum(b["e"] * b["n"] for b in blocks)
print("total executed warp instructions", int(tot))
for b in sorted(blocks, key=lambda b: -b["e"] * b["n"])[:n]:
    ops = {}
    for s in b["src"]:
        t = s.split()
        o = t[1] if t and t[0].startswith("@") else (t[0] if t else "")
        o = o.split(".")[0]
        ops[o] = ops.get(o, 0) + 1
    top = sorted(ops.items(), key=lambda x: -x[1])[:6]
    print(b["start"], f"exec={int(b['e'])} n={b['n']} total={int(b['e'] * b['n'])} "
          f"({b['e'] * b['n'] / tot:.3f})", top)
