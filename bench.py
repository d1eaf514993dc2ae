"""RGDBEK hot-path benchmark (driver contract: one JSON line from rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C2c] [--impl ours|reference]

A "step" is one RGDBEK iteration (the whole hot path: pass T, column scores +
Philox keys + exact block selection, pass N, z update, row scores + keys +
selection, x update) over the synthetic workload resident in HBM.

  value       iterations/s on the device (CUDA events on the solver's stream,
              max over ranks), inputs resident, K iterations per timed region
  e2e         the same metric through the C ABI from HOST buffers: create()
              (H2D of A and b) + K iterations + get_x (D2H), host clock
  roofline    the dominant kernel (dense pass T / pass N GEMV) timed alone with
              CUDA events: algorithmic bytes / mean launch time vs the measured
              HBM copy peak (MEASURED_PEAKS.json)
  cpu_baseline  the CPU oracle (oracle/, numpy fp64) on a bounded sample
  time_to_tol   device time of rgdbek_solve to ||x - x*||/||x*|| <= 1e-6

--impl reference times the oracle itself (the slow plain program this tier
uses as its reference arm) on the same workload, metric and unit.
"""
import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np

METRIC = "RGDBEK iterations/sec and time-to-1e-6 rel. error; SpMV HBM GB/s vs peak"
UNIT = "iterations/s"

WORKLOADS = {
    "C2c": "dense Gaussian 20000x5000 consistent, seed 0 (BASELINE configs[1])",
    "C2i": "dense Gaussian 20000x5000 noisy-inconsistent (||r|| = 0.1||Ax*||), seed 0 (BASELINE configs[1])",
    "C1": "dense Gaussian 200x50 consistent, seed 0 (BASELINE configs[0])",
    "C3": "2-D Poisson 5-point, 4M unknowns, CSR symmetric (BASELINE configs[2])",
    "C4": "1-D Gaussian Toeplitz blur sigma=r=20 on 1024^2 image + noise (BASELINE configs[3])",
    "C5s": "population-model sliding window 50000x5000, 20 nnz/row, inconsistent (configs[4] scaled)",
    "C5": "population-model sliding window 50M x 5M, 1e9 nnz, inconsistent (BASELINE configs[4], 1 GPU)",
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ---------------------------------------------------------------------------------------
# clocks during the timed region (NVML; nvidia-smi equivalent fields)
# ---------------------------------------------------------------------------------------
class ClockSampler:
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x2: "applications_clocks_setting", 0x1: "gpu_idle", 0x10: "sync_boost"}

    def __init__(self, device=0, period=0.02):
        self.samples, self.reasons, self.ok = [], set(), False
        self.period = period
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # no NVML: report null clocks
            log("clock sampler unavailable:", e)
            self.max_mhz = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------------------------
def make_solver(w, device, stream, row_range=None, nccl_comm=None, A_host=None, b_host=None,
                csr_host=None):
    """The C-ABI solver for workload w (this rank's rows when row_range is given).
    A_host / b_host / csr_host: pinned host copies (the e2e leg)."""
    from paper_2509_19267_b200 import Solver
    from paper_2509_19267_b200.dist import shard_csr
    if w.dense:
        A = w.A if A_host is None else A_host
        b = w.b if b_host is None else b_host
        if row_range is not None:
            A, b = A[row_range[0]:row_range[1]], b[row_range[0]:row_range[1]]
        return Solver(A, b, eta=w.eta, device=device, stream=stream, m=w.shape[0],
                      row_range=row_range, nccl_comm=nccl_comm)
    rp, ci, val = w.csr_arrays() if csr_host is None else csr_host
    b = w.b if b_host is None else b_host
    if row_range is not None:
        rp, ci, val = shard_csr(rp, ci, val, *row_range)
        b = b[row_range[0]:row_range[1]]
    return Solver.from_csr(w.shape[0], w.shape[1], rp, ci, val, b, eta=w.eta,
                           symmetric=w.symmetric and row_range is None, device=device,
                           stream=stream, row_range=row_range, nccl_comm=nccl_comm)


def iteration_bytes(w):
    """Algorithmic bytes of one iteration: both reads of A + 32 B/row + 24 B/col."""
    m, n = w.shape
    a = 8.0 * m * n if w.dense else 12.0 * w.A.nnz + 4.0 * (m + 1)
    a_t = a if (w.dense or w.symmetric) else 12.0 * w.A.nnz + 4.0 * (n + 1)
    return a + a_t + 32.0 * m + 24.0 * n


def time_kernel(s, kernel, reps, torch):
    """Mean launch time (s) of one hot kernel, CUDA events on the solver's stream."""
    st = torch.cuda.ExternalStream(s.stream)
    s.launch_kernel(kernel, 3)                      # warm
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    bytes_per = s.launch_kernel(kernel, reps)
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e-3 / reps, bytes_per


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class OneCore:
    """SURVEY §8(d) oracle timing: one host core — BLAS pools limited to 1 thread
    (threadpoolctl) and the process pinned to one CPU (sched_setaffinity, the
    `taskset -c` equivalent) for the duration; restored on exit."""

    def __enter__(self):
        self.aff = os.sched_getaffinity(0)
        self.cpu = max(self.aff)
        os.sched_setaffinity(0, {self.cpu})
        try:
            from threadpoolctl import threadpool_limits
            self.lim = threadpool_limits(limits=1)
        except Exception:
            self.lim = None
        return self

    def __exit__(self, *a):
        if self.lim is not None:
            self.lim.restore_original_limits()
        os.sched_setaffinity(0, self.aff)

    def threads(self):
        try:
            from threadpoolctl import threadpool_info
            return max([i.get("num_threads", 1) for i in threadpool_info()] or [1])
        except Exception:
            return 1


def cpu_oracle_sample(w, budget_s=15.0, max_iters=None, mode="pinv_free", inner=(1e-13, 200),
                      lazy=0):
    """Oracle iterations/s on a bounded sample (first iterations of the same solve), one core."""
    from oracle import Oracle
    from oracle.lazy import LazyOracle
    o = (LazyOracle(w.A, w.b, w.eta, parts=lazy) if lazy else
         Oracle(w.A, w.b, w.eta, update=mode, inner_tol=inner[0], inner_max=inner[1]))
    with OneCore() as oc:
        threads = oc.threads()
        t0 = time.perf_counter()
        it = 0
        while True:
            o.iterate(0)
            it += 1
            el = time.perf_counter() - t0
            if el >= budget_s or (max_iters and it >= max_iters):
                break
    return it / el, it, el, threads


def load_traffic(workload, kernel):
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get(workload, {}).get(kernel)
    return None


PHASE_NAMES = {1: "passT", 2: "s_v_colkeys", 3: "colsel_L2", 4: "colsel_L3",
               5: "colsel_mask_x", 6: "passN", 7: "stop_z_rowkeys", 8: "rowsel_L2",
               9: "rowsel_L3", 10: "rowsel_mask", 0: "bookkeeping",
               11: "dense_colsums_keys", 12: "dense_flush", 13: "colsel_local_L1",
               14: "colsel_local_L2L3", 15: "rowsel_local"}


def phase_profile(w, local, stream, steps, lazy=0):
    """Per-phase device microseconds per iteration of the persistent kernel (a separate
    handle created with RGDBEK_PHASE_TIMING=1; one thread of CTA 0 reads %globaltimer
    after each grid barrier)."""
    os.environ["RGDBEK_PHASE_TIMING"] = "1"
    try:
        sp = make_solver(w, local, stream)
    finally:
        del os.environ["RGDBEK_PHASE_TIMING"]
    if lazy:
        sp.set_lazy(lazy)
    sp.reset(0)
    sp.step(steps)
    pt = sp.phase_times()
    sp.close()
    return {PHASE_NAMES[i]: round(pt[i] / 1e3 / (steps + 1), 2) for i in PHASE_NAMES}


def sparse_record(args, local, torch, peak, peak_src):
    """The SpMV half of the metric ("SpMV HBM GB/s vs peak"): the C4 workload (BASELINE
    configs[3], 1024^2 Toeplitz blur, 43M nnz, CSR) at full size, same K / W as the
    headline, CUDA events on the solver's stream; iteration-level and in-kernel pass
    roofline fractions (pass bytes = the CSR bytes of A only, 12 nnz + 4 (m+1))."""
    from workloads import by_name
    w = by_name("C4")
    m, n = w.shape
    stream = torch.cuda.current_stream()
    s = make_solver(w, local, stream.cuda_stream)
    s.reset(0)
    s.step(args.warmup)
    s.reset(0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    s.step(args.steps)
    e1.record(stream)
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) * 1e-3
    s.close()
    value = args.steps / t
    b_iter = iteration_bytes(w)
    ach = b_iter * value / 1e9
    ph = phase_profile(w, local, stream.cuda_stream, min(args.steps, 300))
    a_bytes = 12.0 * w.A.nnz + 4.0 * (m + 1)
    passes = {}
    for k in ("passT", "passN"):
        us = ph.get(k) or 0.0
        if us > 0:
            gbs = a_bytes / (us * 1e-6) / 1e9
            passes[k] = {"us_per_iter": us, "achieved": round(gbs, 1), "frac": round(gbs / peak, 4)}
    tr = load_traffic("C4", "k_persistent_per_iter")
    return {"workload": "C4", "description": WORKLOADS["C4"], "m": m, "n": n, "nnz": int(w.A.nnz),
            "value": round(value, 3), "unit": UNIT, "steps": args.steps,
            "ms_per_step": round(1e3 * t / args.steps, 5),
            "roofline": {"bound": "hbm", "kernel": "k_persistent (sparse, TMA-fed CSR tiles)",
                         "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(ach / peak, 4), "iteration_bytes": b_iter,
                         "traffic_per_iter": tr, "traffic_source": "profiles/traffic.json (ncu --set full)",
                         "peak_source": peak_src, "in_kernel_passes": passes},
            "phases_us_per_iter": ph}


def multi_rhs_record(args, local, torch, peak, nr=3):
    """NEXT #2: the C4 blur operator with nr right-hand sides in one solve
    (rgdbek_create_csr_multi).  An iteration advances all nr solves; algorithmic bytes of
    one iteration = both reads of A + nr x (32 B per row + 24 B per column)."""
    from paper_2509_19267_b200 import Solver
    from workloads import by_name
    w = by_name("C4")
    m, n = w.shape
    rng = np.random.default_rng(0)
    B = np.array([w.b] + [w.A @ np.clip(rng.random(n), 0, 1) for _ in range(nr - 1)])
    stream = torch.cuda.current_stream()
    s = Solver.from_scipy_multi(w.A, B, eta=w.eta, stream=stream.cuda_stream)
    s.reset(0)
    s.step(args.warmup)
    s.reset(0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    s.step(args.steps)
    e1.record(stream)
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) * 1e-3
    s.close()
    value = args.steps / t
    a_bytes = 12.0 * w.A.nnz + 4.0 * (m + 1)
    b_iter = 2 * a_bytes + nr * (32.0 * m + 24.0 * n)
    return {"workload": "C4", "nrhs": nr, "value": round(value, 3), "unit": UNIT,
            "rhs_iterations_per_s": round(nr * value, 3), "steps": args.steps,
            "ms_per_step": round(1e3 * t / args.steps, 5),
            "roofline": {"bound": "hbm", "achieved": round(b_iter * value / 1e9, 1), "peak": peak,
                         "unit": "GB/s", "frac": round(b_iter * value / 1e9 / peak, 4),
                         "iteration_bytes": b_iter,
                         "a_bytes_per_rhs_iteration": round(2 * a_bytes / nr, 1)}}


def run_ours(args):
    import torch
    from workloads import by_name
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        log(f"warning: WORLD_SIZE={world} but --gpus {args.gpus}")
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    w = by_name(args.workload)
    if args.eta:
        w.eta = args.eta
    m, n = w.shape
    stream = torch.cuda.current_stream()
    comm, rows = None, None
    use_nccl = args.multi == "nccl"
    if world > 1:
        # row-sharded solve of ONE system (strong scaling): nnz-balanced row blocks.
        # Default: the peer-memory sharded engine (one persistent kernel per GPU, window
        # partials / halos / histograms over NVLink, sharded.cuh); --multi nccl: the NCCL
        # graph engine ([A_p^T z_p | A_p^T xi_p | X_p] allreduce and small collectives)
        from paper_2509_19267_b200.dist import init_nccl_comm, partition_rows
        parts = partition_rows(m if w.dense else w.A.indptr, world)
        rows = parts[rank]
        if use_nccl:
            comm = init_nccl_comm(local)
    s = make_solver(w, local, stream.cuda_stream, rows, comm)
    # Algorithm 2: on one GPU --lazy P logical processes; across peer-sharded GPUs every
    # rank is one process (set before connecting)
    lazy_arg = (1 if args.lazy else 0) if (world > 1 and not use_nccl) else args.lazy
    if world > 1 and not use_nccl:
        if lazy_arg:
            s.set_lazy(1)
        from paper_2509_19267_b200.dist import connect_peers
        connect_peers(s)
    if args.mode == "exact":
        s.set_mode("exact", inner_tol=args.inner_tol, inner_max=args.inner_max)
    if args.lazy and not (world > 1 and not use_nccl):
        s.set_lazy(args.lazy)
    engine, ctas = s.engine_info()
    s.reset(0)
    s.step(args.warmup)                              # W untimed warm-up iterations
    s.reset(0)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        s.step(args.steps)                           # exactly K iterations (+ the stop-test tail)
        e1.record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    t = e0.elapsed_time(e1) * 1e-3
    if dist:
        tt = torch.tensor([t], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt.item())
    value = args.steps / t                           # iterations of the one (sharded) system
    launches = 1 + (1 if engine == 0 else s.launches_per_iteration() * (args.steps + 1))
    npass = s.passes() if engine == 0 else 2 * (args.steps + 1)   # passes over A in the timed call
    a_bytes_exact = s.a_bytes() if args.mode == "exact" else 0.0

    # roofline of the dominant kernel.  Persistent engine: the timed region IS one
    # launch of k_persistent (K iterations); achieved = K * B_iter / event time.
    peak, peak_src = load_peaks()
    b_iter = iteration_bytes(w)
    kernels = {}
    for kid, kname in ((0, "passT"), (1, "passN")):
        dt, bytes_per = time_kernel(s, kid, 20, torch)
        kernels[kname] = {"seconds": dt, "bytes": bytes_per, "gbs": bytes_per / dt / 1e9}
    s.reset(0)
    tr = load_traffic(args.workload, "k_persistent_per_iter")
    if engine == 0 and args.mode == "exact":
        # exact mode: the inner solves make the passes per iteration data-dependent;
        # algorithmic bytes = (passes run) x (bytes of A per pass) + the vector sweeps
        m_, n_ = w.shape
        # bytes of A the launch read (full passes, and the dense x-solve's row-masked
        # passes over A^J only: rgdbek_get_a_bytes) + the vector sweeps
        b_launch = a_bytes_exact + args.steps * (32.0 * m_ + 24.0 * n_)
        ach = b_launch / t / 1e9
        roofline = {"bound": "hbm", "kernel": f"k_persistent_exact ({ctas} CTAs x 1024 threads; "
                                              f"{args.steps} iterations, {npass} passes over A)",
                    "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
                    "frac": round(ach / peak, 4), "traffic": None,
                    "algorithmic_bytes_per_launch": b_launch, "peak_source": peak_src,
                    "passes_per_iteration": round(npass / args.steps, 2)}
    elif engine == 0:
        ach = b_iter * args.steps / t / 1e9 / world
        roofline = {"bound": "hbm", "kernel": f"k_persistent ({ctas} CTAs x 1024 threads; "
                                              f"{args.steps} iterations per launch)",
                    "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
                    "frac": round(ach / peak, 4),
                    "traffic": (tr * (args.steps + 1)) if tr else None,
                    "algorithmic_bytes_per_launch": b_iter * args.steps,
                    "peak_source": peak_src}
    else:
        dom = max(kernels, key=lambda k: kernels[k]["seconds"])
        kd = kernels[dom]
        roofline = {"bound": "hbm", "kernel": dom, "achieved": round(kd["gbs"], 1),
                    "peak": peak, "unit": "GB/s", "frac": round(kd["gbs"] / peak, 4),
                    "traffic": load_traffic(args.workload, dom), "peak_source": peak_src}
    roofline["standalone_kernels"] = {
        k: {"achieved": round(v["gbs"], 1), "frac": round(v["gbs"] / peak, 4),
            "us_per_launch": round(v["seconds"] * 1e6, 2), "algorithmic_bytes": v["bytes"]}
        for k, v in kernels.items()}
    roofline["iteration_bytes"] = b_iter
    roofline["iteration_frac"] = round(b_iter * value / world / 1e9 / peak, 4)

    # time to tolerance (device time of rgdbek_solve, REL_ERR 1e-6)
    ttt = None
    if w.xstar is not None and w.stop == "rel_err" and not args.skip_ttt:
        s.set_stop("rel_err")
        s.set_reference(w.xstar)
        res = s.solve(1e-6, 100000, 0)
        ttt = {"seconds": res["seconds"], "iters": res["iters"], "rel_err": res["rel_err"],
               "outcome": res["outcome"], "tol": 1e-6, "eta": w.eta}
        s.set_stop("rse")
    s.close()

    # e2e through the C ABI from host (pinned) buffers
    e2e = None
    if not args.skip_e2e:
        A_h = torch.from_numpy(np.ascontiguousarray(w.A)).pin_memory() if w.dense else None
        csr_h = None if w.dense else tuple(torch.from_numpy(a).pin_memory() for a in w.csr_arrays())
        b_h = torch.from_numpy(w.b).pin_memory()
        x_h = torch.empty(n, dtype=torch.float64).pin_memory()
        # short runs are repeated (median of 3): one create() is a few ms of host work
        reps = 3 if args.steps / value < 2.0 else 1
        runs = []
        for _ in range(reps):
            if dist:
                dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            s2 = make_solver(w, local, stream.cuda_stream, rows, comm,
                             A_host=A_h if w.dense else None, b_host=b_h, csr_host=csr_h)
            if world > 1 and not use_nccl:
                if lazy_arg:
                    s2.set_lazy(1)
                from paper_2509_19267_b200.dist import connect_peers
                connect_peers(s2)
            if args.mode == "exact":
                s2.set_mode("exact", inner_tol=args.inner_tol, inner_max=args.inner_max)
            if args.lazy and not (world > 1 and not use_nccl):
                s2.set_lazy(args.lazy)
            t1 = time.perf_counter()
            s2.reset(0)
            s2.step(args.steps)
            t2 = time.perf_counter()
            s2.x(out=x_h)
            t3 = time.perf_counter()
            s2.close()
            log(f"e2e: create {1e3 * (t1 - t0):.2f} ms, reset+step {1e3 * (t2 - t1):.2f} ms, "
                f"get_x {1e3 * (t3 - t2):.2f} ms")
            runs.append(t3 - t0)
        t_e2e = sorted(runs)[len(runs) // 2]
        if dist:
            tt = torch.tensor([t_e2e], device="cuda", dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t_e2e = float(tt.item())
        a_bytes = (m * n * 8) if w.dense else (w.A.nnz * 12 + (m + 1) * 8)
        e2e = {"value": round(args.steps / t_e2e, 3), "unit": UNIT,
               "h2d_bytes_per_step": int((a_bytes + 8 * m) / args.steps),
               "d2h_bytes_per_step": int(8 * n / args.steps),
               "reps": reps,
               "note": "create() from pinned host A,b + K iterations + get_x to host; host clock"
                       + ("; median of 3" if reps > 1 else "")}

    # per-phase device time of the persistent kernel (separate instrumented handle)
    phases = None
    if engine == 0 and world == 1 and not args.skip_phases and args.mode == "pinv_free":
        phases = phase_profile(w, local, stream.cuda_stream, min(args.steps, 300), args.lazy)
    sparse = None
    if (world == 1 and not args.skip_sparse and w.dense and args.mode == "pinv_free"
            and not args.lazy):
        sparse = sparse_record(args, local, torch, peak, peak_src)
        sparse["multi_rhs"] = multi_rhs_record(args, local, torch, peak)
    if comm is not None:
        from paper_2509_19267_b200.dist import destroy_nccl_comm
        destroy_nccl_comm(comm)

    out = None
    if rank == 0:
        cpu = None
        if not args.skip_cpu:
            v, it, el, threads = cpu_oracle_sample(w, budget_s=args.cpu_budget, mode=args.mode,
                                                   inner=(args.inner_tol, args.inner_max),
                                                   lazy=args.lazy)
            cpu = {"value": round(v, 4), "unit": UNIT, "cores": threads, "kind": "oracle",
                   "cpu_model": cpu_model(), "host_cores": os.cpu_count(),
                   "sample": f"first {it} iterations of the same {args.workload} solve "
                             f"(seed 0) in {el:.1f} s, numpy/BLAS fp64 incl. the per-iteration "
                             f"RSE matvec; one core (BLAS threads 1, pinned to one CPU)"}
        out = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1e3 * t / args.steps, 5),
            "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.workload, "description": WORKLOADS.get(args.workload),
                       "m": m, "n": n, "nnz": int(w.nnz), "eta": w.eta,
                       "parallelism": (f"rows{world} ({'NCCL graph engine' if use_nccl else 'peer-memory sharded persistent kernel'})"
                                       if world > 1 else "single"),
                       "engine": "persistent" if engine == 0 else "graph",
                       "update": args.mode,
                       "algorithm": ((f"Algorithm 2 across the {world} ranks (lazy averaging)"
                                      if world > 1 and not use_nccl else
                                      f"Algorithm 2, {args.lazy} logical processes (lazy averaging)")
                                     if args.lazy else "Algorithm 1"),
                       "l2": "inputs larger than L2 (A = %.0f MB > 126 MB)" % (
                           (m * n * 8 if w.dense else w.A.nnz * 12) / 1e6)},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "time_to_tol": ttt,
            "gpu_launches": launches, "clocks": clk.summary(),
            "phases_us_per_iter": phases, "sparse": sparse,
        }
        print(json.dumps(out), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return out


def run_reference(args):
    """The oracle (plain numpy fp64 CPU program) on the same workload and metric."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    from workloads import by_name
    from oracle import Oracle
    w = by_name(args.workload)
    o = Oracle(w.A, w.b, w.eta)
    with OneCore() as oc:
        threads = oc.threads()
        for _ in range(min(args.warmup, 3)):
            o.iterate(0)
        o.reset()
        # bounded sample: at most ~budget seconds of timed iterations
        t0 = time.perf_counter()
        it = 0
        while it < args.steps:
            o.iterate(0)
            it += 1
            if time.perf_counter() - t0 > args.cpu_budget and it >= 3:
                break
        el = time.perf_counter() - t0
    v = it / el
    sample = (f"{it} of the requested {args.steps} iterations of the {args.workload} solve "
              f"(seed 0), stopped at the {args.cpu_budget:.0f} s budget" if it < args.steps
              else f"all {it} iterations of the {args.workload} solve (seed 0)")
    out = {"metric": METRIC, "value": round(v, 4), "unit": UNIT, "n_gpus": args.gpus,
           "steps": it, "warmup": args.warmup, "ms_per_step": round(1e3 * el / it, 3),
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic", "impl": "reference",
           "config": {"workload": args.workload, "description": WORKLOADS.get(args.workload),
                      "m": w.shape[0], "n": w.shape[1], "eta": w.eta},
           "cpu_baseline": {"value": round(v, 4), "unit": UNIT, "cores": threads, "kind": "oracle",
                            "cpu_model": cpu_model(), "host_cores": os.cpu_count(),
                            "sample": sample + "; one core (BLAS threads 1, pinned to one CPU)"},
           "e2e": {"value": round(v, 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--workload", default="C2c", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--skip-ttt", action="store_true")
    ap.add_argument("--skip-phases", action="store_true")
    ap.add_argument("--skip-sparse", action="store_true",
                    help="omit the C4 SpMV sub-record of the default (dense) line")
    ap.add_argument("--mode", default="pinv_free", choices=["pinv_free", "exact"],
                    help="exact = Alg. 1's pseudoinverse updates by inner CGLS (NEXT #1)")
    ap.add_argument("--lazy", type=int, default=0,
                    help="the paper's parallel Algorithm 2 with this many logical row "
                         "processes (dense, 1 GPU); 0 = Algorithm 1")
    ap.add_argument("--eta", type=float, default=None, help="override the workload's eta")
    ap.add_argument("--multi", default="peer", choices=["peer", "nccl"],
                    help="multi-GPU engine: peer-memory sharded kernel (default) or NCCL graph engine")
    ap.add_argument("--inner-tol", type=float, default=1e-13)
    ap.add_argument("--inner-max", type=int, default=200)
    args = ap.parse_args()
    if args.warmup < 3:
        log("warmup raised to 3 (timing rule)")
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
