"""Prints the key fields of bench.py JSON lines in the given logs (dev helper)."""
import json
import sys

for f in sys.argv[1:]:
    line = None
    for l in open(f):
        if l.startswith("{"):
            line = json.loads(l)
    if line is None:
        print(f, "NO JSON:", open(f).read()[-400:].replace("\n", " | "))
        continue
    print(f.split("/")[-1].ljust(40), round(line["ms_per_step"], 4), round(line["value"]),
          line.get("kernel_variant"), "panel", line.get("panel_cols"), "nnz", line["config"].get("nnz"))
