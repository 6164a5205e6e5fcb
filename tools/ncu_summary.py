"""Summarizes an ncu --set full report of the SpMM kernel into the text
committed under profiles/ (key throughput metrics, DRAM traffic per launch,
stall reasons, optionally the hottest SASS lines).

    python tools/ncu_summary.py gpurun_out/prof_X.ncu-rep [n_hot_lines]
"""
import csv, sys, subprocess
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = csv.reader(out.splitlines()); h = next(r)
keep = ['Duration','DRAM Throughput','L2 Cache Throughput','L1/TEX Cache Throughput','Compute (SM) Throughput','Issue Slots Busy','L1/TEX Hit Rate','L2 Hit Rate','Executed Instructions','Achieved Active Warps Per SM','Theoretical Active Warps per SM','Registers Per Thread','No Eligible','Eligible Warps Per Scheduler','Warp Cycles Per Issued Instruction','Block Limit Shared Mem','Block Limit Registers']
for row in r:
    d = dict(zip(h, row))
    if d.get('Metric Name') in keep: print(d['Metric Name'].ljust(40), d['Metric Unit'].ljust(16), d['Metric Value'])
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines())); h, u, v = rows[0], rows[1], rows[2]
for i, n in enumerate(h):
    if n in ('dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_sector_hit_rate.pct', 'lts__t_sectors_srcunit_tex_op_read.sum', 'gpu__time_duration.sum'):
        print(n, u[i], v[i])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines())); h = rows[1]; idx = {n: i for i, n in enumerate(h)}; data = rows[2:]
def f(r, n):
    try: return float(r[idx[n]])
    except: return 0.0
stalls = [n for n in h if n.startswith("stall_") and "Not Issued" not in n]
print(sorted(((int(sum(f(r, s) for r in data)), s) for s in stalls), reverse=True)[:8])
if len(sys.argv) > 2:
    top = sorted(data, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:int(sys.argv[2])]
    for r in sorted(top, key=lambda r: int(r[idx["Address"]], 16)):
        ss = {s[6:]: int(f(r, s)) for s in stalls if f(r, s) > 0.15 * f(r, "Warp Stall Sampling (All Samples)")}
        print(r[idx["Address"]][-5:], r[idx["Source"]][:58].ljust(58), int(f(r, "Instructions Executed")), int(f(r, "Warp Stall Sampling (All Samples)")), ss)
