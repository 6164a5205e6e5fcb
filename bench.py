"""bench.py -- GE-SpMM hot path on B200 (BASELINE.json metric:
"SpMM GFLOP/s (2*nnz*N) and achieved HBM GB/s vs roofline at 1/2/4/8 B200").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload config5|config2|config1|config3-N|config4] [--op sum|max|min|mean]
                    [--scaling strong|weak] [--extra config2] [--b-panels P]

Workload (default): BASELINE configs[4], the north-star configuration -- R-MAT
scale 24 (16M rows), 2^30 edges requested (Graph500 a/b/c = .57/.19/.19,
deduplicated: 1.02 B nonzeros) x dense B with N=128, fp32, sum-reduce, on one
GPU at N=1 and row-sharded (strong scaling) at N>1.  Synthetic, seeded,
generated on the GPU with torch ops (workloads.rmat_csr) -- the SAME generator
and seed in both arms, so the reference arm reads the identical matrix
(``input`` carries a fingerprint in both lines).  configs[1] (R-MAT scale 20,
N=64) and configs[3] (R-MAT scale 22, N=128) ride along at N=1 under
``extra`` (kernel, roofline, e2e, each with its own clock record).

A step = one execution of the hot path over the matrix with a cached plan
(one kernel launch per column panel, after a reset of its item counter).
Each timed step is bracketed by CUDA events on the launching stream, with a
2x-L2 buffer written between steps (L2 flushed; the flush is outside the
events).  N>1 (torchrun): each rank owns an nnz-balanced row block; time = max
over ranks.  Kernel-only steps run after B is on every rank; the
broadcast-inclusive legs are reported separately (``broadcast``: B broadcast
alone, broadcast then compute, and the column-panelled broadcast overlapped
with the compute), and the N>1 ``e2e`` starts from pinned host buffers
(root's B, every rank's CSR slab) and ends with every rank's C slab on the
host.

Extra keys: roofline (HBM, algorithmic compulsory bytes U per launch, the
ncu DRAM traffic of the same kernel, and gather_ceiling at N=64), cpu_baseline
(the oracle port on all host cores on a bounded row sample, plus one thread),
e2e (N=1: host buffers through gespmm_csr_spmm_host -- pipelined H2D + device
colind check + plan + kernel + D2H), clocks (NVML samples inside the timed
region; the nvidia-smi record rides along), sustained (the same steps after a
1 s soak at the power cap), c_allgather (N>1: fused peer-store vs NCCL
all-gather of C), gpu_launches.

--impl reference: the reference's own CPU implementation of the path (the
unmodified raceset interpreter running gespmm_alg2.mir, oracle/_ref) on a
bounded row sample of the same matrix, all host threads, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback


def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="config5")
    ap.add_argument("--op", default="sum", choices=["sum", "max", "min", "mean"])
    ap.add_argument("--N", type=int, default=0, help="override the workload's dense width (sweeps)")
    ap.add_argument("--extra", default="config2,config4",
                    help="N=1: comma-separated workloads measured after the headline one (kernel, roofline, "
                         "e2e) and reported under 'extra'; '' = none")
    ap.add_argument("--generator", default="torch", choices=["torch", "native"],
                    help="R-MAT input: torch ops (both arms, identical matrix) or the library's CUDA "
                         "generator (gespmm_rmat_csr)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-clocks", action="store_true")
    ap.add_argument("--no-allgather", action="store_true", help="N > 1: skip the C all-gather timing")
    ap.add_argument("--soak-s", type=float, default=0.0, help="back-to-back launches before the timed steps")
    ap.add_argument("--sustained-s", type=float, default=1.0,
                    help="soak length of the extra 'sustained' leg (0 = skip)")
    ap.add_argument("--variant", default="", help="kernel variant override (testing), e.g. vec1_lpr32_cwm2")
    ap.add_argument("--tile-work", type=int, default=0, help="plan tile size override (tuning); 0 = automatic")
    ap.add_argument("--scaling", default="strong", choices=["weak", "strong"],
                    help="N > 1: strong = the workload's rows split nnz-balanced across ranks (default, "
                         "the north-star run); weak = every rank owns one copy of the workload's rows "
                         "(the job is N row-stacked copies sharing B)")
    ap.add_argument("--b-panels", type=int, default=4,
                    help="N > 1: column panels of the B broadcast overlapped with the compute")
    ap.add_argument("--ref-sample-products", type=int, default=800_000,
                    help="--impl reference: nnz*N products per step (bounds interpreter RAM)")
    return ap.parse_args(argv)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def workload_spec(name):
    if name == "config2":
        return dict(kind="rmat", scale=20, edges=16 * 2**20, N=64, seed=3,
                    desc="R-MAT scale 20 (1M rows), 16M edges requested (dedup), N=64 (BASELINE configs[1])")
    if name == "config4":
        return dict(kind="rmat", scale=22, edges=64 * 2**20, N=128, seed=3,
                    desc="R-MAT scale 22 (4M rows), 64M edges requested (dedup), N=128 (configs[3])")
    if name == "config5":
        return dict(kind="rmat", scale=24, edges=2**30, N=128, seed=3,
                    desc="R-MAT scale 24 (16M rows), 2^30 edges requested (dedup), N=128 (configs[4])")
    if name == "config1":
        return dict(kind="uniform", M=4096, K=4096, density=0.01, N=32, seed=1,
                    desc="uniform 4096x4096, 1% density, N=32 (configs[0])")
    if name.startswith("config3"):
        N = int(name.split("-")[1]) if "-" in name else 64
        return dict(kind="reddit", N=N, seed=5,
                    desc=f"Reddit-like 232,965 rows ~114.6M nnz power-law, N={N} (configs[2])")
    raise SystemExit(f"unknown workload {name}")


def make_workload(spec, device, generator="torch"):
    """R-MAT: generator="torch" builds the matrix and B with torch ops
    (workloads.rmat_csr / dense_torch) -- what BOTH arms use by default, so the
    reference arm reads the identical input and no libgespmm code runs on its
    path; "native" uses the library's CUDA generators (gespmm_rmat_csr:
    Philox keys + CUB sort/unique; a different graph of the same law)."""
    import torch

    from paper_2503_08946_b200 import workloads as W

    native = generator == "native" and device.type == "cuda"
    if spec["kind"] == "rmat" and native:
        csr = W.rmat_csr_gpu(spec["scale"], spec["edges"], seed=spec["seed"], device=device)
    elif spec["kind"] == "rmat":
        csr = W.rmat_csr(spec["scale"], spec["edges"], seed=spec["seed"], device=device)
    elif spec["kind"] == "uniform":
        c = W.uniform_csr(spec["M"], spec["K"], spec["density"], seed=spec["seed"])
        csr = W.Csr(torch.as_tensor(c.rowptr, device=device), torch.as_tensor(c.colind, device=device),
                    torch.as_tensor(c.vals, device=device), c.M, c.K)
    else:
        csr = W.reddit_like_csr(seed=spec["seed"], device=device)
    if native:
        B = W.dense_gpu(csr.K, spec["N"], seed=2, device=device)
    else:
        B = W.dense_torch(csr.K, spec["N"], seed=2, device=device)
    return csr, B


def fingerprint(csr, B):
    """Identity of the input, printed by both arms (same numbers = same matrix)."""
    import torch

    return {"M": int(csr.M), "K": int(csr.K), "nnz": int(csr.nnz), "N": int(B.shape[1]),
            "sum_rowptr": int(csr.rowptr.to(torch.int64).sum()),
            "sum_colind": int(csr.colind.to(torch.int64).sum()),
            "sum_vals": round(float(csr.vals.to(torch.float64).sum()), 6),
            "sum_B": round(float(B.to(torch.float64).sum()), 6)}


def algorithmic_bytes(M, K, N, nnz):
    """compulsory bytes U and no-reuse gather bytes G."""
    U = 4 * (M + 1) + 8 * nnz + 4 * K * N + 4 * M * N
    G = 4 * (M + 1) + 8 * nnz + 4 * nnz * N + 4 * M * N
    return U, G


class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int, enabled: bool = True):
        self.index = index
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")
        if enabled:
            try:
                os.makedirs(os.path.dirname(self.path), exist_ok=True)
                self.f = open(self.path, "w")
                self.proc = subprocess.Popen(
                    ["nvidia-smi", f"--id={index}", f"--query-gpu={self.FIELDS}", "--format=csv",
                     "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
            except Exception:
                self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.close()
        sm, mx, reasons = [], 0.0, set()
        names = ["active", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as f:
            for line in f:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) < 9 or not parts[1].split()[0].isdigit():
                    continue
                sm.append(float(parts[1].split()[0]))
                mx = max(mx, float(parts[2].split()[0]))
                for nm, v in zip(names[1:], parts[5:9]):
                    if v.lower().startswith("active"):
                        reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "window": "nvidia-smi -lms 100"}


class NvmlSampler:
    """SM clock / throttle reasons polled in-process (NVML, the library
    nvidia-smi reads) every ~2 ms while running, so a timed region of a few
    tens of milliseconds gets its own samples without a pre-soak."""
    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, index: int, enabled: bool = True):
        import threading

        self.ok = False
        self.sm, self.reasons, self.mx, self.watts, self.limit_w = [], set(), 0.0, [], None
        if not enabled:
            return
        try:
            import pynvml as nv

            nv.nvmlInit()
            self.nv = nv
            self.h = nv.nvmlDeviceGetHandleByIndex(index)
            self.mx = float(nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM))
            try:
                self.limit_w = nv.nvmlDeviceGetEnforcedPowerLimit(self.h) / 1000.0
            except Exception:
                self.limit_w = None
            self.ok = True
        except Exception:
            return
        self.stop_evt = threading.Event()
        self.th = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        nv = self.nv
        while not self.stop_evt.is_set():
            try:
                self.sm.append(float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)))
                try:
                    self.watts.append(nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0)
                except Exception:
                    pass
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, bit in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def start(self):
        if self.ok:
            self.th.start()

    def stop(self, window: str):
        if not self.ok:
            return None
        self.stop_evt.set()
        self.th.join(timeout=2)
        if not self.sm:
            return None
        out = {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": self.mx, "reasons": sorted(self.reasons),
               "samples": len(self.sm), "window": window, "source": "NVML, ~2 ms"}
        if self.watts:  # board power (NVML's own averaging window) against the enforced limit
            out["power_w"] = {"median": statistics.median(self.watts), "max": max(self.watts),
                              "limit": self.limit_w}
        return out


def row_sample(rp, target_nnz):
    """Every s-th row (s chosen so the sample holds ~target_nnz nonzeros): a
    bounded sample that keeps the matrix's degree mix (R-MAT's heavy rows
    are spread over the whole row range, not front-loaded)."""
    import numpy as np

    nnz = int(rp[-1])
    M = rp.shape[0] - 1
    s = max(1, -(-nnz // max(1, target_nnz)))
    rows = np.arange(0, M, s, dtype=np.int64)
    deg = (rp[rows + 1] - rp[rows]).astype(np.int64)
    srp = np.zeros(rows.size + 1, np.int64)
    srp[1:] = np.cumsum(deg)
    starts = rp[rows].astype(np.int64)
    pos = np.repeat(starts - srp[:-1], deg) + np.arange(int(srp[-1]), dtype=np.int64)
    return rows, srp.astype(np.int32), pos, s


def cpu_baseline_port(rp, ci, vv, Bh, N, op, budget_s=10.0, target_nnz=64 << 20):
    """The oracle's fp32 restatement (oracle/gespmm_oracle.c, OpenMP, all host
    threads) on a bounded sample of the same matrix (the whole matrix when it
    has <= target_nnz nonzeros, else every s-th row against the full B),
    repeated for ~budget_s (the contract's 10-30 s of CPU work); best run.
    Plus one host thread on a 2M-nonzero block."""
    import numpy as np

    from oracle import oracle as O

    nth = O.num_threads()
    if int(rp[-1]) > target_nnz:
        rows, srp, pos, s = row_sample(rp, target_nnz)
        sci, svv = ci[pos], vv[pos]
        what = f"every {s}th row ({rows.size} rows, {int(srp[-1])} nnz) of the same matrix x the full B"
    else:
        srp, sci, svv = rp, ci, vv
        what = f"full workload (M={rp.shape[0] - 1}, nnz={int(rp[-1])})"
    best, runs = None, 0
    t_end = time.perf_counter() + budget_s
    while True:
        t0 = time.perf_counter()
        O.spmm_f32(srp, sci, svv, Bh, op, seg_len=256, nthreads=nth)
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
        runs += 1
        if time.perf_counter() > t_end or runs >= 400:
            break
    gflops = 2.0 * int(srp[-1]) * N / best / 1e9
    r1 = min(srp.shape[0] - 1, int(np.searchsorted(srp, min(int(srp[-1]), 2_000_000))) + 1)
    p1 = int(srp[r1])
    t0 = time.perf_counter()
    O.spmm_f32(srp[:r1 + 1], sci[:p1], svv[:p1], Bh, op, seg_len=256, nthreads=1)
    dt1 = time.perf_counter() - t0
    return {"value": round(gflops, 3), "unit": "GFLOP/s", "cores": nth, "kind": "port",
            "sample": f"{what}, N={N}, {op}; best of {runs} runs in ~{budget_s:.0f} s; "
                      f"oracle/gespmm_oracle.c fp32 twin, OpenMP {nth} threads",
            "single_thread": {"value": round(2.0 * p1 * N / dt1 / 1e9, 3), "unit": "GFLOP/s", "cores": 1,
                              "sample": f"first {r1} rows ({p1} nnz) of that sample, one run"}}


def time_allgather(plan, vals, B, C, bounds, rank, world, op, stream, dev, reps=5):
    """Device time (max over ranks) of compute + C all-gather, fused vs NCCL."""
    import torch
    import torch.distributed as dist

    from paper_2503_08946_b200.spmm import ipc_close, ipc_handle, ipc_open

    M = int(bounds[-1])
    a, b = int(bounds[rank]), int(bounds[rank + 1])
    N = B.shape[1]
    full_f = torch.empty((M, N), dtype=torch.float32, device=dev)
    full_n = torch.empty((M, N), dtype=torch.float32, device=dev)
    h, off = ipc_handle(full_f)
    allh = [None] * world
    dist.all_gather_object(allh, (h, off))
    opened, peers = [], []
    for w, (hw, ow) in enumerate(allh):
        if w != rank:
            base = ipc_open(hw)
            opened.append(base)
            peers.append(base + ow)

    def fused():
        plan.execute_peers(vals, B, full_f[a:b], peers, a, reduce=op, stream=stream)

    def nccl():
        plan.execute(vals, B, op, out=full_n[a:b], stream=stream)
        for w in range(world):
            lo, hi = int(bounds[w]), int(bounds[w + 1])
            if hi > lo:
                dist.broadcast(full_n[lo:hi], src=w)

    t_f = timed_region(fused, stream, dev, world, reps)
    t_n = timed_region(nccl, stream, dev, world, reps)
    same = bool(torch.equal(full_f, full_n))
    for base in opened:
        ipc_close(base)
    del full_f, full_n
    return {"fused_peer_stores_ms": t_f, "nccl_broadcasts_ms": t_n, "identical": same,
            "bytes_per_rank": int((b - a) * N * 4 * (world - 1)),
            "what": "compute + full C on every rank; fused = kernel epilogue stores into every "
                    "rank's full C over NVLink (CUDA IPC), nccl = execute then one broadcast per slab owner"}


def timed_region(fn, stream, dev, world, reps=5, before=None):
    """Mean device time of fn() over reps (after one untimed run), CUDA events
    on `stream`, barrier + synchronize on both sides, max over ranks."""
    import torch
    import torch.distributed as dist

    ts = []
    for _ in range(reps + 1):
        if before is not None:
            before()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ts.append(e0.elapsed_time(e1))
    t = torch.tensor([sum(ts[1:]) / reps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_reference(args):
    """Reference arm: the unmodified reference interpreter (oracle/_ref) on
    the identical matrix (same torch generator and seed as our arm)."""
    import numpy as np
    import torch

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return 0
    from oracle import oracle as O

    spec = workload_spec(args.workload)
    if args.N > 0:
        spec["N"] = args.N
    if not O.ref_available():
        print(json.dumps({"impl": "reference",
                          "unavailable": "oracle/_ref/libgespmm_ref.so not built (reference tree absent at build time)"}))
        return 0
    dev = torch.device("cuda:0") if torch.cuda.is_available() else torch.device("cpu")
    csr, B = make_workload(spec, dev, "torch")
    fp = fingerprint(csr, B)
    N = spec["N"]
    rp = csr.rowptr.cpu().numpy().astype(np.int64)
    ci = csr.colind.cpu().numpy()
    vv = csr.vals.cpu().numpy()
    Bh = np.ascontiguousarray(B.cpu().numpy())
    del csr, B
    nth = os.cpu_count() or 1
    target_nnz = max(1, args.ref_sample_products // N)
    M = rp.shape[0] - 1
    deg = np.diff(rp)
    # the interpreter runs one instance per host thread; a row longer than
    # target/threads would leave the other threads idle (and a 10^5-nonzero row
    # takes the interpreter minutes), so the sample draws from rows up to `cap`
    cap = max(1, target_nnz // nth)

    def sample(i):
        """Rows drawn uniformly at random (seeded per step) until ~target_nnz
        nonzeros; rows longer than cap are skipped (recorded in the line)."""
        order = np.random.default_rng(1000 + i).permutation(M)
        d = deg[order]
        ok = order[(d > 0) & (d <= cap)]
        csum = np.cumsum(deg[ok])
        rows = np.sort(ok[: int(np.searchsorted(csum, target_nnz)) + 1])
        srp = np.zeros(rows.size + 1, np.int64)
        srp[1:] = np.cumsum(deg[rows])
        idx = np.concatenate([np.arange(rp[r], rp[r + 1]) for r in rows])
        return srp.astype(np.int32), ci[idx], vv[idx], rows.size

    def step(i):
        srp, sci, svv, nrows = sample(i)
        _, secs, nlog = O.ref_spmm_csr(srp, sci, svv, Bh, nthreads=nth, want_c=False)
        return int(srp[-1]), secs, nlog, nrows

    for i in range(args.warmup):
        step(i)
    tot_nnz, tot_s, tot_rows = 0, 0.0, 0
    for i in range(args.steps):
        n, s, _, rows = step(args.warmup + i)
        tot_nnz += n
        tot_s += s
        tot_rows += rows
    value = 2.0 * tot_nnz * N / tot_s / 1e9
    skipped = deg > cap
    line = {
        "metric": "SpMM GFLOP/s (2*nnz*N)", "value": value, "unit": "GFLOP/s", "impl": "reference",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": tot_s / max(args.steps, 1) * 1e3, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": spec["desc"], "op": "sum", "N": N, "M": M, "nnz": int(rp[-1]),
                   "input": fp, "generator": "torch ops (workloads.rmat_csr), same seed as the GPU arm",
                   "sample": {"nnz_per_step": target_nnz, "row_cap_nnz": cap,
                              "rows_over_cap": int(skipped.sum()),
                              "nnz_in_rows_over_cap": int(deg[skipped].sum())}},
        "cpu_baseline": {"value": value, "unit": "GFLOP/s", "cores": nth, "kind": "reference",
                         "sample": f"per step ~{target_nnz} nnz in {tot_rows / max(args.steps, 1):.0f} "
                                   f"rows drawn at random (seeded; rows > {cap} nnz skipped) from "
                                   f"the same matrix; raceset::run on gespmm_alg2.mir (block 4, "
                                   f"grid rows x N/4), rows split into {nth} parallel instances "
                                   f"(reference SPEC.md:478-479); time = run() calls only"},
        "e2e": {"value": value, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def ncu_record(name, workload, op, world):
    """The committed ncu capture of the same kernel and workload (profiles/):
    DRAM bytes per launch (traffic.json) and the ncu metric summary."""
    if world != 1:
        return None
    try:
        with open(os.path.join(ROOT, "profiles", name)) as f:
            return json.load(f).get(f"{workload}:{op}")
    except Exception:
        return None


def pinned_like(t):
    import torch

    h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    h.copy_(t)
    return h


class Measure:
    """One workload on this rank: build, plan, timed steps and the legs."""

    def __init__(self, args, name, dev, world, rank, local):
        import numpy as np
        import torch
        import torch.distributed as dist

        from paper_2503_08946_b200.spmm import Plan, partition_rows

        self.args, self.name, self.dev, self.world, self.rank = args, name, dev, world, rank
        spec = workload_spec(name)
        if args.N > 0 and name == args.workload:
            spec["N"] = args.N
            spec["desc"] += f" [N overridden to {args.N}]"
        self.spec = spec
        self.N = N = spec["N"]
        csr, B = make_workload(spec, dev, args.generator)
        self.fp = fingerprint(csr, B)
        self.K = K = csr.K
        self.stream = stream = torch.cuda.current_stream(dev)
        self.M_all, self.nnz_all = csr.M, csr.nnz
        if world > 1 and args.scaling == "weak":
            # the job is `world` row-stacked copies of the workload's rows, all
            # gathering from one B; rank r owns rows [rM, (r+1)M)
            self.bounds = np.arange(world + 1, dtype=np.int64) * csr.M
            rowptr, colind, vals = csr.rowptr, csr.colind, csr.vals
            self.M_all, self.nnz_all = csr.M * world, csr.nnz * world
        elif world > 1:
            rp_h = csr.rowptr.cpu().numpy()
            self.bounds = partition_rows(rp_h, world)
            a, b = int(self.bounds[rank]), int(self.bounds[rank + 1])
            p0, p1 = int(rp_h[a]), int(rp_h[b])
            rowptr = (csr.rowptr[a:b + 1] - p0).contiguous()
            colind = csr.colind[p0:p1].clone()  # own 16-byte-aligned storage (a view at p0 is
            vals = csr.vals[p0:p1].clone()      # aligned only when p0 % 4 == 0: 4-byte staging)
            del rp_h
        else:
            self.bounds = None
            rowptr, colind, vals = csr.rowptr, csr.colind, csr.vals
        del csr
        self.B_root = None
        if world > 1:
            if rank == 0:
                self.B_root = B.clone()  # the root's copy survives the broadcast legs
            else:
                B.zero_()  # only the root holds B; the broadcast is the exchange step
            torch.cuda.synchronize()
            dist.barrier()
            self.bcast_ms = timed_region(lambda: dist.broadcast(B, src=0), stream, dev, world, reps=3)
        else:
            self.bcast_ms = 0.0
        self.rowptr, self.colind, self.vals, self.B = rowptr, colind, vals, B
        self.M_loc, self.nnz_loc = rowptr.numel() - 1, colind.numel()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

        def build_plan():
            t0 = time.perf_counter()
            e0.record(stream)
            plan = Plan(rowptr, colind, K)
            e1.record(stream)
            torch.cuda.synchronize()
            return plan, e0.elapsed_time(e1), (time.perf_counter() - t0) * 1e3

        # the first plan of the process also pays one-time costs (lazy module
        # loading of the plan kernels, the stream-ordered pool's first growth);
        # the plan a repeated call builds is the second one
        first, self.plan_first_ms, _ = build_plan()
        first.close()
        self.plan, self.plan_ms, self.plan_wall_ms = build_plan()
        self.info = self.plan.info()
        self.C = torch.empty((self.M_loc, N), dtype=torch.float32, device=dev)
        l2 = torch.cuda.get_device_properties(dev).L2_cache_size
        self.flush = torch.empty(max(2 * l2, 256 << 20) // 4, dtype=torch.float32, device=dev)

    def run_once(self):
        self.plan.execute(self.vals, self.B, self.args.op, out=self.C, stream=self.stream)

    def steps(self, n, warmup):
        import torch
        import torch.distributed as dist

        for _ in range(max(warmup, 3)):
            self.flush.zero_()
            self.run_once()
        torch.cuda.synchronize()
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(n)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(n)]
        if self.world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        for i in range(n):
            self.flush.zero_()  # L2 flush between timed steps (outside the events)
            starts[i].record(self.stream)
            self.run_once()
            ends[i].record(self.stream)
        torch.cuda.synchronize()
        if self.world > 1:
            dist.barrier()
        return [s_.elapsed_time(e_) for s_, e_ in zip(starts, ends)]

    def soak(self, seconds):  # back-to-back launches (sustained load)
        import torch

        t_end = time.perf_counter() + seconds
        while time.perf_counter() < t_end:
            for _ in range(50 if self.N * self.nnz_loc < 1 << 32 else 4):
                self.run_once()
            torch.cuda.synchronize()

    def max_over_ranks(self, ms):
        import torch
        import torch.distributed as dist

        t = torch.tensor([ms], device=self.dev, dtype=torch.float64)
        if self.world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def roofline(self, t_mean):
        U, G = algorithmic_bytes(self.M_loc, self.K, self.N, self.nnz_loc)
        peak, peak_src = peaks()
        achieved = U / (t_mean * 1e-3) / 1e9
        ncu = ncu_record("ncu_metrics.json", self.name, self.args.op, self.world)
        return {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak,
                "traffic": ncu_record("traffic.json", self.name, self.args.op, self.world),
                # the measured side of SURVEY 8(d): ncu DRAM bytes / duration of the
                # same kernel against the same peak (the >= 70 % HBM target)
                "dram_frac_ncu": (ncu["dram_GBs"] / peak) if ncu and ncu.get("dram_GBs") else None,
                "l2_hit_pct_ncu": ncu.get("l2_hit_pct") if ncu else None,
                "bytes_model": f"U = 4(M+1) + 8nnz + 4KN + 4MN = {U} B per launch",
                "peak_source": peak_src, "gather_bytes_G": G, "gather_GBs": G / (t_mean * 1e-3) / 1e9,
                "ncu": ncu}

    def gather_ceiling(self, t_mean):
        """tools/gather_probe.cu replays this matrix's colind as B-row gathers
        at the kernel's memory-level parallelism (8 loads/warp, 32 warps/SM,
        256-nonzero spans) with nothing else: the floor for any kernel
        gathering the same rows in the same order.  N=64."""
        import ctypes

        import torch

        probe = os.path.join(ROOT, "tools", "libgather_probe.so")
        if self.N != 64 or self.world != 1 or not os.path.exists(probe) or os.environ.get("GESPMM_NO_PROBE"):
            return None
        Lp = ctypes.CDLL(probe)
        Lp.gather_probe.restype = ctypes.c_float
        Lp.gather_probe.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
                                    ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                    ctypes.c_void_p, ctypes.c_int64]
        sink = torch.zeros(4, device=self.dev)
        args = (self.B.data_ptr(), self.colind.data_ptr(), self.nnz_loc)
        pms = Lp.gather_probe(*args, 8, 256, 4, 5, sink.data_ptr(), self.flush.data_ptr(), self.flush.numel() * 4)
        pms16 = Lp.gather_probe(*args, 16, 256, 4, 5, sink.data_ptr(), self.flush.data_ptr(),
                                self.flush.numel() * 4)
        if pms <= 0:
            return None
        return {"probe_ms": pms, "kernel_ms": t_mean, "frac": pms / t_mean, "probe_ms_16_in_flight": pms16,
                "what": "gather-only replay of this colind stream, 8 loads/warp x 32 warps/SM "
                        "(tools/gather_probe.cu, best of 5, L2 flushed)"}

    def e2e_single(self, flops, reps):
        """N=1: the public host entry point (gespmm_csr_spmm_host) on pinned
        host buffers, wall clock per call."""
        import torch

        from paper_2503_08946_b200.spmm import csr_spmm_host

        h_rp, h_ci, h_v, h_B = (pinned_like(t) for t in (self.rowptr, self.colind, self.vals, self.B))
        h_C = torch.empty((self.M_loc, self.N), dtype=torch.float32, pin_memory=True)
        csr_spmm_host(h_rp, h_ci, h_v, h_B, self.args.op, out=h_C)  # warm
        et = []
        for _ in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            csr_spmm_host(h_rp, h_ci, h_v, h_B, self.args.op, out=h_C)
            et.append(time.perf_counter() - t0)
        ok = bool(torch.equal(h_C, self.C.cpu()))
        self.host = (h_rp, h_ci, h_v, h_B)
        t = statistics.median(et)
        return {"value": flops / t / 1e9, "unit": "GFLOP/s",
                "h2d_bytes_per_step": int(4 * (self.M_loc + 1) + 8 * self.nnz_loc + 4 * self.K * self.N),
                "d2h_bytes_per_step": int(4 * self.M_loc * self.N),
                "ms_per_step": t * 1e3, "reps": reps, "stat": "median", "equals_device_result": ok,
                "path": "gespmm_csr_spmm_host (pinned host buffers; pipelined: rowptr + B H2D, "
                        "plan, then per item-aligned row chunk, fewest nonzeros first: colind/vals "
                        "H2D -> device colind check -> kernel -> C rows D2H overlapping the next "
                        "chunk; wall clock per call)"}

    def broadcast_legs(self, panels):
        """N>1: the exchange step with the compute -- B broadcast alone,
        broadcast then compute, and the column-panelled broadcast overlapped
        with the compute (sharded.broadcast_B_overlapped); device time on the
        compute stream, max over ranks.  B is re-zeroed on non-root ranks
        before every repetition, so each one really moves B."""
        import torch
        import torch.distributed as dist

        from paper_2503_08946_b200 import sharded as S

        B, st, world, rank = self.B, self.stream, self.world, self.rank
        comm = torch.cuda.Stream(device=self.dev)
        C2 = torch.empty_like(self.C)
        packed = [torch.empty((self.K, c1 - c0), dtype=torch.float32, device=self.dev)
                  for c0, c1 in S.panel_bounds(self.N, panels)]

        def reset():
            if rank != 0:
                B.zero_()
                for t in packed:
                    t.zero_()
            else:
                B.copy_(self.B_root)

        def serial():
            dist.broadcast(B, src=0)
            self.plan.execute(self.vals, B, self.args.op, out=self.C, stream=st)

        def overlapped():
            def panel(p, Bp, c0, c1):
                self.plan.execute(self.vals, Bp, self.args.op, out=C2[:, c0:c1], stream=st)
            S.broadcast_B_overlapped(panel, B, panels, 0, None, cuda_streams=(st, comm), packed=packed)

        t_ser = timed_region(serial, st, self.dev, world, reps=3, before=reset)
        t_ovl = timed_region(overlapped, st, self.dev, world, reps=3, before=reset)
        same = bool(torch.equal(C2, self.C))
        ident = torch.tensor([1 if same else 0], device=self.dev)
        dist.all_reduce(ident, op=dist.ReduceOp.MIN)
        reset()
        dist.broadcast(B, src=0)  # leave B complete on every rank
        torch.cuda.synchronize()
        del C2, packed
        return {"b_broadcast_ms": self.bcast_ms, "broadcast_then_compute_ms": t_ser,
                "overlapped_ms": t_ovl, "b_panels": len(S.panel_bounds(self.N, panels)),
                "identical": bool(ident.item()), "b_bytes": int(self.K * self.N * 4),
                "what": "device time on the compute stream, max over ranks; overlapped = B cut into column "
                        "panels, panel p broadcast (NCCL, comm stream) while panel p-1 computes"}

    def e2e_sharded(self, flops, panels, reps):
        """N>1 end to end: pinned host buffers (the root's B, every rank's CSR
        slab) -> H2D -> plan -> column-panelled B broadcast overlapped with the
        compute -> this rank's C slab D2H; wall clock, max over ranks."""
        import torch
        import torch.distributed as dist

        from paper_2503_08946_b200 import sharded as S
        from paper_2503_08946_b200.spmm import Plan

        dev, st = self.dev, self.stream
        h_rp, h_ci, h_v = (pinned_like(t) for t in (self.rowptr, self.colind, self.vals))
        h_B = pinned_like(self.B_root) if self.rank == 0 else None
        h_C = torch.empty((self.M_loc, self.N), dtype=torch.float32, pin_memory=True)
        d_B = torch.zeros((self.K, self.N), dtype=torch.float32, device=dev)
        d_C = torch.empty_like(self.C)
        comm = torch.cuda.Stream(device=dev)
        packed = [torch.empty((self.K, c1 - c0), dtype=torch.float32, device=dev)
                  for c0, c1 in S.panel_bounds(self.N, panels)]

        def call():
            rp, ci, v = (h.to(dev, non_blocking=True) for h in (h_rp, h_ci, h_v))
            if h_B is not None:
                d_B.copy_(h_B, non_blocking=True)
            plan = Plan(rp, ci, self.K)

            def panel(p, Bp, c0, c1):
                plan.execute(v, Bp, self.args.op, out=d_C[:, c0:c1], stream=st)
            S.broadcast_B_overlapped(panel, d_B, panels, 0, None, cuda_streams=(st, comm), packed=packed)
            h_C.copy_(d_C, non_blocking=True)
            torch.cuda.synchronize()
            plan.close()

        call()
        et = []
        for _ in range(reps):
            torch.cuda.synchronize()
            dist.barrier()
            t0 = time.perf_counter()
            call()
            et.append(time.perf_counter() - t0)
        t = self.max_over_ranks(statistics.median(et))
        ok = bool(torch.equal(h_C, self.C.cpu()))
        ident = torch.tensor([1 if ok else 0], device=dev)
        dist.all_reduce(ident, op=dist.ReduceOp.MIN)
        n_pan = len(packed)
        del d_B, d_C, packed
        return {"value": flops / t / 1e9, "unit": "GFLOP/s",
                "h2d_bytes_per_step": int(4 * (self.M_loc + 1) + 8 * self.nnz_loc
                                          + (4 * self.K * self.N if self.rank == 0 else 0)),
                "d2h_bytes_per_step": int(4 * self.M_loc * self.N), "bytes_are": "rank 0's",
                "ms_per_step": t * 1e3, "reps": reps, "stat": "median, max over ranks",
                "equals_device_result": bool(ident.item()), "b_panels": n_pan,
                "path": "pinned host CSR slab per rank + root's B -> H2D -> Plan -> column-panelled NCCL "
                        "B broadcast overlapped with the compute -> C slab D2H; wall clock"}


def measure_extra(args, name, dev):
    """A secondary workload at N=1: kernel steps, roofline, gather ceiling, e2e."""
    import torch

    from paper_2503_08946_b200.spmm import variant_name

    m = Measure(args, name, dev, 1, 0, 0)
    nvml = NvmlSampler(dev.index or 0, enabled=not args.no_clocks)
    nvml.start()
    times = m.steps(args.steps, args.warmup)
    clk = nvml.stop("warm-up + timed steps")
    t = sum(times) / len(times)
    flops = 2.0 * m.nnz_all * m.N
    out = {"workload": m.spec["desc"], "op": args.op, "N": m.N, "nnz": m.nnz_all, "input": m.fp,
           "value": flops / (t * 1e-3) / 1e9, "unit": "GFLOP/s", "ms_per_step": t,
           "step_ms": {"min": min(times), "median": statistics.median(times), "max": max(times)},
           "roofline": m.roofline(t), "gather_ceiling": m.gather_ceiling(t), "clocks": clk,
           "kernel_variant": m.plan.last_variant() or variant_name(m.N, m.B, m.C, args.op)}
    if not args.no_e2e:
        out["e2e"] = m.e2e_single(flops, reps=max(3, min(args.steps, 10)))
    del m
    torch.cuda.empty_cache()
    return out


def main():
    args = parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    from paper_2503_08946_b200.spmm import panel_width, set_variant_override, variant_name

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and rank == 0:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE {world}", file=sys.stderr)
    # GESPMM_BENCH_BACKEND=gloo (testing only): several ranks may share one GPU
    backend = os.environ.get("GESPMM_BENCH_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count()) if backend != "nccl" else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    if args.variant:
        set_variant_override(args.variant)
    if args.tile_work:
        from paper_2503_08946_b200.spmm import set_tile_work_override
        set_tile_work_override(args.tile_work)

    m = Measure(args, args.workload, dev, world, rank, local)
    N, K = m.N, m.K
    clocks = ClockSampler(local, enabled=not args.no_clocks and rank == 0)
    nvml = NvmlSampler(local, enabled=not args.no_clocks and rank == 0)
    m.soak(args.soak_s)
    nvml.start()
    times = m.steps(args.steps, args.warmup)
    clk_nvml = nvml.stop("timed region")
    sustained = None
    if args.sustained_s > 0:
        # the same steps after ~1 s of back-to-back launches (the part reaches
        # its power cap; clocks sampled over soak + steps)
        nvml2 = NvmlSampler(local, enabled=not args.no_clocks and rank == 0)
        nvml2.start()
        m.soak(args.sustained_s)
        times2 = m.steps(args.steps, 0)
        sustained = {"ms_per_step": m.max_over_ranks(sum(times2) / len(times2)), "soak_s": args.sustained_s,
                     "clocks": nvml2.stop(f"{args.sustained_s} s soak + timed steps")}
    clk = clocks.stop()
    if clk is not None:
        clk["window"] = "whole measurement (timed region + sustained leg), nvidia-smi -lms 100"
    if clk_nvml is not None:
        clk_nvml["nvidia_smi"] = clk
        clk = clk_nvml
    t_mean = sum(times) / len(times)
    t_job = m.max_over_ranks(t_mean)  # ms, max over ranks
    pw = panel_width(K, N)
    n_panels = (N + pw - 1) // pw
    flops = 2.0 * m.nnz_all * N
    value = flops / (t_job * 1e-3) / 1e9
    roof = m.roofline(t_mean)
    roof["gather_ceiling"] = m.gather_ceiling(t_mean)

    c_allgather = None
    if world > 1 and not args.no_allgather:
        try:
            c_allgather = time_allgather(m.plan, m.vals, m.B, m.C, m.bounds, rank, world, args.op, m.stream, dev)
        except Exception as ex:  # report, never fail the bench line
            c_allgather = {"error": f"{type(ex).__name__}: {ex}"[:300]}
    broadcast = None
    if world > 1:
        broadcast = m.broadcast_legs(args.b_panels)

    e2e = None
    if not args.no_e2e:
        reps = max(3, min(args.steps, 10))
        e2e = m.e2e_single(flops, reps) if world == 1 else m.e2e_sharded(flops, args.b_panels, reps)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        if getattr(m, "host", None) is not None:
            h_rp, h_ci, h_v, h_B = (t.numpy() for t in m.host)
        else:
            h_rp, h_ci, h_v, h_B = (t.cpu().numpy() for t in (m.rowptr, m.colind, m.vals, m.B))
        cpu = cpu_baseline_port(h_rp, h_ci, h_v, h_B, N, args.op)

    info = m.info
    line = None
    if rank == 0:
        line = {
            "metric": "SpMM GFLOP/s (2*nnz*N)",
            "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_job, "higher_is_better": True,
            "scaling": args.scaling if world > 1 else "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic" + (f" ({world} row-stacked copies of the workload sharing B, one per rank)"
                                   if world > 1 and args.scaling == "weak" else ""),
            "config": {"workload": m.spec["desc"], "op": args.op, "N": N, "M": m.M_all, "K": K,
                       "nnz": m.nnz_all, "input": m.fp,
                       "generator": ("torch ops (workloads.rmat_csr), same seed as the reference arm"
                                     if args.generator == "torch" else "libgespmm gespmm_rmat_csr"),
                       "l2_flush": f"{m.flush.numel() * 4 >> 20} MiB written between timed steps",
                       "parallelism": (f"row-block x{world} ({args.scaling} scaling)" if world > 1
                                       else "single GPU"),
                       "plan": {"n_items": info["n_items"], "n_long_rows": info["n_long_rows"],
                                "n_segments": info["n_segments"], "build_ms": m.plan_ms,
                                "build_wall_ms": m.plan_wall_ms, "first_build_ms": m.plan_first_ms,
                                "what": "device time of a fresh plan (the process's second; the first "
                                        "also pays one-time module loading and pool growth)"},
                       "b_broadcast_ms": m.bcast_ms},
            "hbm_gbs_algorithmic": roof["achieved"],
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": clk,
            "sustained": sustained,
            "broadcast": broadcast,
            "c_allgather": c_allgather,
            "gpu_launches": args.steps * int(info["kernel_launches_per_execute"]) * n_panels,
            "panel_cols": pw,
            "kernel_variant": m.plan.last_variant() or variant_name(N, m.B, m.C, args.op),
            "step_ms": {"min": min(times), "median": statistics.median(times), "max": max(times)},
        }
    del m
    torch.cuda.empty_cache()
    extras = [w.strip("'\" ") for w in args.extra.split(",")] if world == 1 else []
    extras = [w for w in extras if w and w != "none" and w != args.workload]
    if extras and rank == 0:
        line["extra"] = {}
        for w in extras:
            try:
                line["extra"][w] = measure_extra(args, w, dev)
            except (Exception, SystemExit) as ex:  # report, never fail the headline line
                line["extra"][w] = {"error": f"{type(ex).__name__}: {ex}"[:300]}
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
