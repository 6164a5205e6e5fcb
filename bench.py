"""bench.py -- GE-SpMM hot path on B200 (BASELINE.json metric:
"SpMM GFLOP/s (2*nnz*N) and achieved HBM GB/s vs roofline at 1/2/4/8 B200").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload config2|config1|config3-N|config4|config5] [--op sum|max|min|mean]

Workload (default, BASELINE configs[1]): R-MAT scale 20 (1M rows), 16M edges
requested (Graph500 a/b/c = .57/.19/.19, deduplicated), x dense B with N=64,
fp32, sum-reduce.  Synthetic data, seeded; generated on the GPU.

A step = one execution of the hot path over the matrix with a cached plan
(one kernel launch per column panel, after a reset of its item counter).  Each timed step is bracketed by CUDA events on the
launching stream, with a 2x-L2 buffer written between steps (L2 flushed; the
flush is outside the events).  N>1 (torchrun): row-block sharding, each rank
runs its nnz-balanced row block after a one-time NCCL broadcast of B; time =
max over ranks; value = total flops / that time ("strong" scaling).

Extra keys: roofline (HBM, algorithmic compulsory bytes U per launch, the
ncu DRAM traffic of the same kernel, and gather_ceiling: a live gather-only
replay of the same column stream at the kernel's memory-level parallelism;
see DESIGN.md), cpu_baseline (the oracle port on all host cores, ~10 s, plus a
single-thread sample), e2e (host buffers through gespmm_csr_spmm_host:
pipelined H2D + device colind check + plan + kernel + D2H), clocks (NVML
samples inside the timed region; the nvidia-smi record rides along),
sustained (the same steps after a 1 s soak at the power cap), c_allgather
(N > 1: fused peer-store vs NCCL all-gather of C), gpu_launches.

--impl reference: the reference's own CPU implementation of the path (the
unmodified raceset interpreter running gespmm_alg2.mir, oracle/_ref) on a
bounded row sample of the same workload, all host threads, rank 0 only.
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


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="config2")
    ap.add_argument("--op", default="sum", choices=["sum", "max", "min", "mean"])
    ap.add_argument("--N", type=int, default=0, help="override the workload's dense width (sweeps)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-clocks", action="store_true")
    ap.add_argument("--no-allgather", action="store_true", help="N > 1: skip the C all-gather timing")
    ap.add_argument("--soak-s", type=float, default=0.0, help="back-to-back launches before the timed steps")
    ap.add_argument("--sustained-s", type=float, default=1.0,
                    help="soak length of the extra 'sustained' leg (0 = skip)")
    ap.add_argument("--variant", default="", help="kernel variant override (testing), e.g. vec1_lpr32_cwm2")
    ap.add_argument("--tile-work", type=int, default=0, help="plan tile size override (tuning); 0 = automatic")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="N > 1: weak = every rank owns one copy of the workload's rows (the job is N "
                         "row-stacked copies sharing B: per-GPU work fixed); strong = the workload's "
                         "rows split across ranks (nnz-balanced)")
    ap.add_argument("--ref-sample-products", type=int, default=800_000,
                    help="--impl reference: nnz*N products per step (bounds interpreter RAM)")
    return ap.parse_args()


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
                    desc="R-MAT scale 24 (16M rows), 2^30 edges requested (dedup), N=128 (configs[4], one GPU)")
    if name == "config1":
        return dict(kind="uniform", M=4096, K=4096, density=0.01, N=32, seed=1,
                    desc="uniform 4096x4096, 1% density, N=32 (configs[0])")
    if name.startswith("config3"):
        N = int(name.split("-")[1]) if "-" in name else 64
        return dict(kind="reddit", N=N, seed=5,
                    desc=f"Reddit-like 232,965 rows ~114.6M nnz power-law, N={N} (configs[2])")
    raise SystemExit(f"unknown workload {name}")


def make_workload(spec, device, native=True):
    """native=True: the library's CUDA generators (gespmm_rmat_csr /
    gespmm_uniform_fill); the reference arm passes native=False and gets the
    same recursion from torch ops, so no libgespmm code runs on that arm."""
    import numpy as np
    import torch

    from paper_2503_08946_b200 import workloads as W

    native = native and device.type == "cuda"
    if spec["kind"] == "rmat" and native:
        # native CUDA generator (gespmm_rmat_csr: Philox keys, CUB sort + unique)
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
    del np
    return csr, B


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
        self.sm, self.reasons, self.mx = [], set(), 0.0
        if not enabled:
            return
        try:
            import pynvml as nv

            nv.nvmlInit()
            self.nv = nv
            self.h = nv.nvmlDeviceGetHandleByIndex(index)
            self.mx = float(nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM))
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
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": self.mx, "reasons": sorted(self.reasons),
                "samples": len(self.sm), "window": window, "source": "NVML, ~2 ms"}


def cpu_baseline_port(csr, B, N, budget_s=10.0):
    """The oracle's fp32 restatement (oracle/gespmm_oracle.c, OpenMP, all host
    threads) on the full matrix, repeated for ~budget_s (about 10 s of CPU
    work, the contract's bounded sample); best run."""
    import numpy as np

    from oracle import oracle as O

    rp = csr.rowptr.cpu().numpy()
    ci = csr.colind.cpu().numpy()
    vv = csr.vals.cpu().numpy()
    Bh = np.ascontiguousarray(B.cpu().numpy())
    nth = O.num_threads()
    best = None
    t_end = time.perf_counter() + budget_s
    runs = 0
    while True:
        t0 = time.perf_counter()
        O.spmm_f32(rp, ci, vv, Bh, "sum", seg_len=256, nthreads=nth)
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
        runs += 1
        if time.perf_counter() > t_end or runs >= 400:
            break
    gflops = 2.0 * csr.nnz * N / best / 1e9
    # single host thread on a bounded row block (1 thread and nproc threads)
    r1 = min(csr.M, int(np.searchsorted(rp, min(int(rp[-1]), 2_000_000))) + 1)
    rp1 = rp[:r1 + 1]
    p1 = int(rp1[-1])
    t0 = time.perf_counter()
    O.spmm_f32(rp1, ci[:p1], vv[:p1], Bh, "sum", seg_len=256, nthreads=1)
    dt1 = time.perf_counter() - t0
    return {"value": round(gflops, 3), "unit": "GFLOP/s", "cores": nth, "kind": "port",
            "sample": f"full workload (M={csr.M}, nnz={csr.nnz}, N={N}), best of {runs} runs in ~{budget_s:.0f} s, "
                      f"oracle/gespmm_oracle.c fp32 twin, OpenMP {nth} threads",
            "single_thread": {"value": round(2.0 * p1 * N / dt1 / 1e9, 3), "unit": "GFLOP/s", "cores": 1,
                              "sample": f"first {r1} rows ({p1} nnz) of the same matrix, one run"}}


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

    def timed(fn):
        ts = []
        for _ in range(reps + 1):
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            torch.cuda.synchronize()
            dist.barrier()  # every rank's peer stores have landed
            ts.append(e0.elapsed_time(e1))
        t = torch.tensor([sum(ts[1:]) / reps], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def fused():
        plan.execute_peers(vals, B, full_f[a:b], peers, a, reduce=op, stream=stream)

    def nccl():
        plan.execute(vals, B, op, out=full_n[a:b], stream=stream)
        for w in range(world):
            lo, hi = int(bounds[w]), int(bounds[w + 1])
            if hi > lo:
                dist.broadcast(full_n[lo:hi], src=w)

    t_f = timed(fused)
    t_n = timed(nccl)
    same = bool(torch.equal(full_f, full_n))
    for base in opened:
        ipc_close(base)
    return {"fused_peer_stores_ms": t_f, "nccl_broadcasts_ms": t_n, "identical": same,
            "bytes_per_rank": int((b - a) * N * 4 * (world - 1)),
            "what": "compute + full C on every rank; fused = kernel epilogue stores into every "
                    "rank's full C over NVLink (CUDA IPC), nccl = execute then one broadcast per slab owner"}


def run_reference(args):
    """Reference arm: the unmodified reference interpreter (oracle/_ref)."""
    import numpy as np
    import torch

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return 0
    from oracle import oracle as O

    spec = workload_spec(args.workload)
    if not O.ref_available():
        print(json.dumps({"impl": "reference",
                          "unavailable": "oracle/_ref/libgespmm_ref.so not built (reference tree absent at build time)"}))
        return 0
    dev = torch.device("cuda:0") if torch.cuda.is_available() else torch.device("cpu")
    csr, B = make_workload(spec, dev, native=False)
    N = spec["N"]
    rp = csr.rowptr.cpu().numpy().astype(np.int64)
    ci = csr.colind.cpu().numpy()
    vv = csr.vals.cpu().numpy()
    Bh = np.ascontiguousarray(B.cpu().numpy())
    nth = os.cpu_count() or 1
    target_nnz = max(1, args.ref_sample_products // N)
    M = csr.M
    deg = np.diff(rp)
    cap = max(1, target_nnz // nth)  # longer rows would leave host threads idle

    def sample(i):
        """Rows drawn uniformly at random (seeded per step) until ~target_nnz
        nonzeros; rows longer than target/threads are skipped."""
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
    line = {
        "metric": "SpMM GFLOP/s (2*nnz*N)", "value": value, "unit": "GFLOP/s", "impl": "reference",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": tot_s / max(args.steps, 1) * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": spec["desc"], "op": "sum", "N": N, "M": M, "nnz": csr.nnz},
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


def main():
    args = parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2503_08946_b200.spmm import (Plan, csr_spmm_host, partition_rows, set_variant_override,
                                            variant_name)

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

    spec = workload_spec(args.workload)
    if args.N > 0:
        spec["N"] = args.N
        spec["desc"] += f" [N overridden to {args.N}]"
    N = spec["N"]
    if args.variant:
        set_variant_override(args.variant)
    if args.tile_work:
        from paper_2503_08946_b200.spmm import set_tile_work_override
        set_tile_work_override(args.tile_work)
    csr, B = make_workload(spec, dev)
    M_all, K, nnz_all = csr.M, csr.K, csr.nnz
    stream = torch.cuda.current_stream(dev)

    # ---- row-block sharding (world > 1) ----------------------------------
    # weak: the job is `world` row-stacked copies of the workload's rows, all
    # gathering from one B (A_job = [A; A; ...], C_job = [C; C; ...]); rank r
    # owns rows [r*M, (r+1)*M) -- per-GPU work equals the 1-GPU run.
    # strong: the workload's own rows split nnz-balanced across ranks.
    if world > 1 and args.scaling == "weak":
        bounds = np.arange(world + 1, dtype=np.int64) * M_all
        rowptr, colind, vals = csr.rowptr, csr.colind, csr.vals
        M_all, nnz_all = M_all * world, nnz_all * world
        if rank != 0:
            B.zero_()  # only the root holds B; the broadcast is the exchange step
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        dist.broadcast(B, src=0)
        e1.record(stream)
        torch.cuda.synchronize()
        bcast_ms = e0.elapsed_time(e1)
    elif world > 1:
        rp_h = csr.rowptr.cpu().numpy()
        bounds = partition_rows(rp_h, world)
        a, b = int(bounds[rank]), int(bounds[rank + 1])
        p0, p1 = int(rp_h[a]), int(rp_h[b])
        rowptr = (csr.rowptr[a:b + 1] - p0).contiguous()
        colind = csr.colind[p0:p1].contiguous()
        vals = csr.vals[p0:p1].contiguous()
        if rank != 0:
            B.zero_()  # only the root holds B; the broadcast is the exchange step
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        dist.broadcast(B, src=0)
        e1.record(stream)
        torch.cuda.synchronize()
        bcast_ms = e0.elapsed_time(e1)
    else:
        rowptr, colind, vals = csr.rowptr, csr.colind, csr.vals
        bcast_ms = 0.0
    M_loc, nnz_loc = rowptr.numel() - 1, colind.numel()

    # ---- plan (cached across steps; its build is reported separately) ----
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(stream)
    plan = Plan(rowptr, colind, K)
    e1.record(stream)
    torch.cuda.synchronize()
    plan_ms = e0.elapsed_time(e1)
    plan_wall_ms = (time.perf_counter() - t0) * 1e3
    info = plan.info()
    C = torch.empty((M_loc, N), dtype=torch.float32, device=dev)

    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = torch.empty(max(2 * l2, 256 << 20) // 4, dtype=torch.float32, device=dev)

    def run_once():
        plan.execute(vals, B, args.op, out=C, stream=stream)

    for _ in range(max(args.warmup, 3)):
        flush.zero_()
        run_once()
    torch.cuda.synchronize()

    clocks = ClockSampler(local, enabled=not args.no_clocks and rank == 0)
    nvml = NvmlSampler(local, enabled=not args.no_clocks and rank == 0)

    def soak(seconds):  # back-to-back launches (sustained load)
        t_end_soak = time.perf_counter() + seconds
        while time.perf_counter() < t_end_soak:
            for _ in range(50):
                run_once()
            torch.cuda.synchronize()

    def timed_steps():
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        for i in range(args.steps):
            flush.zero_()  # L2 flush between timed steps (outside the events)
            starts[i].record(stream)
            run_once()
            ends[i].record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        return [s_.elapsed_time(e_) for s_, e_ in zip(starts, ends)]

    soak(args.soak_s)
    nvml.start()
    times = timed_steps()
    clk_nvml = nvml.stop("timed region")
    # sustained: the same steps after ~1 s of back-to-back launches (the part
    # reaches its power cap; clocks sampled over soak + steps)
    sustained = None
    if args.sustained_s > 0:
        nvml2 = NvmlSampler(local, enabled=not args.no_clocks and rank == 0)
        nvml2.start()
        soak(args.sustained_s)
        times2 = timed_steps()
        t2 = torch.tensor([sum(times2) / len(times2)], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(t2, op=dist.ReduceOp.MAX)
        sustained = {"ms_per_step": float(t2.item()), "soak_s": args.sustained_s,
                     "clocks": nvml2.stop(f"{args.sustained_s} s soak + timed steps")}
    clk = clocks.stop()
    if clk is not None:
        clk["window"] = "whole measurement (timed region + sustained leg), nvidia-smi -lms 100"
    if clk_nvml is not None:
        clk_nvml["nvidia_smi"] = clk
        clk = clk_nvml
    t_mean = sum(times) / len(times)
    t_max = torch.tensor([t_mean], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    t_job = float(t_max.item())  # ms, max over ranks

    from paper_2503_08946_b200.spmm import panel_width
    pw = panel_width(K, N)
    n_panels = (N + pw - 1) // pw
    flops = 2.0 * nnz_all * N
    value = flops / (t_job * 1e-3) / 1e9
    U, G = algorithmic_bytes(M_loc, K, N, nnz_loc)
    peak, peak_src = peaks()
    achieved = U / (t_mean * 1e-3) / 1e9

    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath) and world == 1:  # ncu bytes of the single-GPU launch
        try:
            with open(tpath) as f:
                traffic = json.load(f).get(f"{args.workload}:{args.op}")
        except Exception:
            traffic = None
    # the >= 70 % HBM target is stated on ncu DRAM throughput, with
    # the L2 sector hit rate beside it -- from the committed capture of the
    # same kernel and workload (never measured under ncu here)
    ncu = None
    npath = os.path.join(ROOT, "profiles", "ncu_metrics.json")
    if os.path.exists(npath) and world == 1:
        try:
            with open(npath) as f:
                ncu = json.load(f).get(f"{args.workload}:{args.op}")
        except Exception:
            ncu = None

    # ---- C all-gather (N > 1): fused peer stores vs NCCL after the compute --
    # The fused path (gespmm_plan_execute_peers) writes every finished C row
    # into every rank's full-C buffer over NVLink from the kernel epilogue
    # (CUDA IPC); the baseline computes the slab, then one NCCL broadcast per
    # slab owner.  Both timed on the device, max over ranks.
    c_allgather = None
    if world > 1 and not args.no_allgather:
        try:
            c_allgather = time_allgather(plan, vals, B, C, bounds, rank, world, args.op, stream, dev)
        except Exception as ex:  # report, never fail the bench line
            c_allgather = {"error": f"{type(ex).__name__}: {ex}"[:300]}

    # ---- live gather ceiling: the same column stream, gathers only ---------
    # tools/gather_probe.cu replays this matrix's colind as B-row gathers at the
    # kernel's memory-level parallelism (8 loads/warp, 32 warps/SM, 256-nonzero
    # spans) with nothing else; its time is the floor for any kernel gathering
    # the same rows in the same order.  N = 64 only.
    gather_ceiling = None
    probe = os.path.join(ROOT, "tools", "libgather_probe.so")
    if N == 64 and world == 1 and os.path.exists(probe) and not os.environ.get("GESPMM_NO_PROBE"):
        import ctypes

        Lp = ctypes.CDLL(probe)
        Lp.gather_probe.restype = ctypes.c_float
        Lp.gather_probe.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
                                    ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                    ctypes.c_void_p, ctypes.c_int64]
        sink = torch.zeros(4, device=dev)
        pms = Lp.gather_probe(B.data_ptr(), colind.data_ptr(), nnz_loc, 8, 256, 4, 5, sink.data_ptr(),
                              flush.data_ptr(), flush.numel() * 4)
        pms16 = Lp.gather_probe(B.data_ptr(), colind.data_ptr(), nnz_loc, 16, 256, 4, 5, sink.data_ptr(),
                                flush.data_ptr(), flush.numel() * 4)
        if pms > 0:
            gather_ceiling = {"probe_ms": pms, "kernel_ms": t_mean, "frac": pms / t_mean,
                              "probe_ms_16_in_flight": pms16,
                              "what": "gather-only replay of this colind stream, 8 loads/warp x 32 warps/SM "
                                      "(tools/gather_probe.cu, best of 5, L2 flushed)"}

    # ---- e2e through the public host API (H2D + validate + plan + kernel + D2H)
    e2e = None
    if not args.no_e2e:
        hp = lambda t: t.cpu().pin_memory()  # noqa: E731
        h_rp, h_ci, h_v, h_B = hp(rowptr), hp(colind), hp(vals), hp(B)
        h_C = torch.empty((M_loc, N), dtype=torch.float32).pin_memory()
        csr_spmm_host(h_rp, h_ci, h_v, h_B, args.op, out=h_C)  # warm
        reps = max(3, min(args.steps, 10))
        et = []
        for _ in range(reps):
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            csr_spmm_host(h_rp, h_ci, h_v, h_B, args.op, out=h_C)
            et.append(time.perf_counter() - t0)
        e2e_t = torch.tensor([sum(et) / len(et)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
        e2e = {"value": flops / float(e2e_t.item()) / 1e9, "unit": "GFLOP/s",
               "h2d_bytes_per_step": int(4 * (M_loc + 1) + 8 * nnz_loc + 4 * K * N),
               "d2h_bytes_per_step": int(4 * M_loc * N),
               "ms_per_step": float(e2e_t.item()) * 1e3,
               "path": "gespmm_csr_spmm_host (pinned host buffers; pipelined: rowptr + B H2D, "
                       "plan, then per item-aligned row chunk, fewest nonzeros first: colind/vals "
                       "H2D -> device colind check -> kernel -> C rows D2H overlapping the next "
                       "chunk; wall clock per call)"}

    # ---- CPU baseline (rank 0, N=1 only) ----------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_port(csr, B, N)

    if rank == 0:
        line = {
            "metric": "SpMM GFLOP/s (2*nnz*N)",
            "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_job, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f32",
            "data": "synthetic" + (f" ({world} row-stacked copies of the workload sharing B, one per rank)"
                                   if world > 1 and args.scaling == "weak" else ""),
            "config": {"workload": spec["desc"], "op": args.op, "N": N, "M": M_all, "K": K,
                       "nnz": nnz_all, "l2_flush": f"{flush.numel() * 4 >> 20} MiB written between timed steps",
                       "parallelism": (f"row-block x{world} ({args.scaling} scaling)" if world > 1
                                       else "single GPU"),
                       "plan": {"n_items": info["n_items"], "n_long_rows": info["n_long_rows"],
                                "n_segments": info["n_segments"], "build_ms": plan_ms,
                                "build_wall_ms": plan_wall_ms},
                       "b_broadcast_ms": bcast_ms},
            "hbm_gbs_algorithmic": achieved,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "bytes_model": f"U = 4(M+1) + 8nnz + 4KN + 4MN = {U} B per launch",
                         "peak_source": peak_src,
                         "gather_bytes_G": G, "gather_GBs": G / (t_mean * 1e-3) / 1e9,
                         "gather_ceiling": gather_ceiling, "ncu": ncu},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": clk,
            "sustained": sustained,
            "c_allgather": c_allgather,
            "gpu_launches": args.steps * int(info["kernel_launches_per_execute"]) * n_panels,
            "panel_cols": pw,
            "kernel_variant": variant_name(N, B, C, args.op),
            "step_ms": {"min": min(times), "median": statistics.median(times), "max": max(times)},
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
