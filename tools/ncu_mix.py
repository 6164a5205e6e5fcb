"""Executed-instruction mix of an ncu --set full report of the SpMM kernel, per
nonzero: which SASS opcodes the kernel spends its issue slots on, and where
its stall samples land (DESIGN.md 5.2 item 9 used this to find the per-batch
rematerialization).

    python tools/ncu_mix.py gpurun_out/prof_X.ncu-rep NNZ [n_hot_lines]
"""
import collections
import csv
import subprocess
import sys


def main():
    rep, nnz = sys.argv[1], float(sys.argv[2])
    n_hot = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[1]
    idx = {n: i for i, n in enumerate(h)}
    tot, by, stall = 0.0, collections.Counter(), collections.Counter()
    lines = []
    for r in rows[2:]:
        try:
            n = float(r[idx["Instructions Executed"]])
        except (ValueError, IndexError):
            continue
        src = r[idx["Source"]].strip()
        op = (src.split()[1] if src.startswith("@") else src.split()[0]).split(".")[0]
        st = float(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
        by[op] += n
        stall[op] += st
        tot += n
        lines.append((n, st, src))
    st_tot = sum(stall.values()) or 1.0
    print(f"{rows[0][1][:100]}")
    print(f"warp instructions executed: {tot:.4g} = {tot / nnz:.2f} per nonzero")
    for op, n in by.most_common(24):
        print(f"  {op:12s} {n / nnz:6.2f}/nnz  {100 * n / tot:5.1f}% of instr  {100 * stall[op] / st_tot:5.1f}% of stall samples")
    if n_hot:
        print("hottest lines by stall samples:")
        for n, st, src in sorted(lines, key=lambda x: -x[1])[:n_hot]:
            print(f"  {n / nnz:6.3f}/nnz {int(st):8d}  {src[:90]}")


if __name__ == "__main__":
    main()
