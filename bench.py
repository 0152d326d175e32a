"""NS-RGS benchmark (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl reference]

One "step" = one whole pass of the hot path on the resident synthetic instance of the chosen
BASELINE.json config: spectral initialisation (subspace iteration on the panel A.X kernel +
scaled-NS polar), T NS-RGS iterations (fused A.X + gradient/projection/step + K-step
Newton-Schulz retraction, fused fp64 objective trace) and the alignment metrics.
value = T * K_steps / (max over ranks of the device time of K_steps solves)  [NS-RGS it/s].

--impl reference times the fp64 oracle (oracle/, as it stands) on the host cores on a bounded
sample of the same workload (a panel of nodes' block rows; scaled to whole-problem it/s).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {  # BASELINE.json "configs" (seed 0 everywhere, eta = 1/n)
    "c1": dict(n=100, d=3, sigma=0.5, T=50, K=3),
    "c2": dict(n=2000, d=3, sigma=0.5, T=100, K=5),
    "c3": dict(n=20000, d=5, sigma=0.3 * np.sqrt(20000) / 5, T=100, K=5),
    "c4": dict(n=12000, d=10, sigma=0.2 * np.sqrt(12000) / 10, T=100, K=6),
    "c5": dict(n=40000, d=5, sigma=0.3 * np.sqrt(40000) / 5, T=100, K=5),
}
# Not a BASELINE config: the paper's block size d = 25 (Table 1 :336-363) at a size that
# streams 40 GB, with the paper's protocol T_s = 1 (K = 1) — the tcgen05 wide pass
SIDE_CONFIGS = {"w25": dict(n=4000, d=25, sigma=0.2, T=50, K=1)}
METRIC = "NS-RGS iterations/sec and effective HBM GB/s (% of roofline) at 1/2/4/8 B200"
INIT_TOL, INIT_MAX_SWEEPS = 1e-5, 100


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def _traffic(cfg_name):
    """dram bytes per panel launch from the committed ncu --set full summary, if any."""
    p = os.path.join(ROOT, "profiles", "ncu_full_summary.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        v = j.get(cfg_name, {}).get("dram_bytes_per_launch")
        return float(v) if v else None
    return None


class Clocks:
    """nvidia-smi sampler for the timed region (clocks + throttle reasons)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,power.draw")

    def __init__(self, device):
        self.device, self.rows, self.proc = device, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), "--query-gpu=" + self.Q,
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[2 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def _dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ------------------------------------------------------------------------------------ oracle
def _oracle_worker(cfg, node0, m, warm, passes_fixed, budget_s, barrier, q):
    """One host process of the CPU baseline: oracle.nsrgs.step_rows (Algorithm 2 restricted to a
    panel of m nodes, the oracle's arithmetic unchanged) on its own panel, 1 BLAS thread."""
    from threadpoolctl import threadpool_limits

    from oracle import instance as inst
    from oracle import nsrgs as ons

    with threadpool_limits(limits=1):
        n, d = cfg["n"], cfg["d"]
        Z = inst.ground_truth(0, n, d)
        nodes = np.arange(node0, node0 + m)
        R = inst.measurement_rows(0, Z, cfg["sigma"], nodes)   # fp32-rounded A rows, fp64 (untimed)
        for _ in range(warm):
            ons.step_rows(R, Z, nodes, 1.0 / n, cfg["K"])
        barrier.wait()
        passes, t0 = 0, time.perf_counter()
        while True:
            ons.step_rows(R, Z, nodes, 1.0 / n, cfg["K"])
            passes += 1
            el = time.perf_counter() - t0
            if (passes_fixed and passes >= passes_fixed) or (not passes_fixed and (el >= budget_s or passes >= 100000)):
                break
    q.put((m, passes, el))


def _host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def _oracle_pool(cfg, nodes_per_worker, warm=1, passes_fixed=0, budget_s=10.0, workers=None):
    """The oracle on all host cores: one spawned process per core, each timing step_rows on its
    own panel of nodes (the sample) after a common barrier.  Returns (it/s scaled to the whole
    problem, workers, max seconds per pass, sample description)."""
    import multiprocessing as mp

    n = cfg["n"]
    W = workers or max(1, min(_host_cores(), 64, n // max(1, nodes_per_worker)))
    m = max(1, min(nodes_per_worker, n // W))
    ctx = mp.get_context("spawn")
    barrier, q = ctx.Barrier(W), ctx.Queue()
    procs = [ctx.Process(target=_oracle_worker, args=(cfg, w * m, m, warm, passes_fixed, budget_s, barrier, q))
             for w in range(W)]
    for p in procs:
        p.start()
    res = [q.get() for _ in range(W)]
    for p in procs:
        p.join()
    nodes_per_s = sum(mm * ps / el for mm, ps, el in res)
    per_pass = max(el / ps for _, ps, el in res)
    sample = (f"oracle.nsrgs.step_rows in {W} processes (1 BLAS thread each) x {m} nodes = {W * m} of {n} nodes "
              f"({W * m * cfg['d']} of {n * cfg['d']} A rows, fp64), each on its own panel; "
              f"it/s = (sum over processes of nodes x passes / seconds) / {n}")
    return nodes_per_s / n, W, per_pass, sample


def _oracle_single_thread(cfg, nodes_sample, passes=3):
    """The same sample with the BLAS pool limited to one thread (context figure)."""
    from threadpoolctl import threadpool_limits

    from oracle import instance as inst
    from oracle import nsrgs as ons

    n, d = cfg["n"], cfg["d"]
    Z = inst.ground_truth(0, n, d)
    nodes = np.arange(nodes_sample)
    R = inst.measurement_rows(0, Z, cfg["sigma"], nodes)
    with threadpool_limits(limits=1):
        ons.step_rows(R, Z, nodes, 1.0 / n, cfg["K"])
        t0 = time.perf_counter()
        for _ in range(passes):
            ons.step_rows(R, Z, nodes, 1.0 / n, cfg["K"])
        per = (time.perf_counter() - t0) / passes
    return (nodes_sample / n) / per


def _read_stream_gbs(torch, device, stream, gib=8, reps=5):
    """In-run HBM read-stream ceiling: the library's TMA read probe
    (nsrgs_probe_read_stream: the dense pass's access pattern — one CTA per SM, 32 KB bulk
    copies into a shared-memory ring — with the arithmetic removed) over a buffer far larger
    than L2; best of `reps`, CUDA events on `stream`."""
    from paper_2604_07372_b200 import nsrgs

    buf = torch.ones(gib * (1 << 30) // 4, dtype=torch.float32, device=device)
    torch.cuda.synchronize()
    g = nsrgs.probe_read_stream(buf, stream, reps)
    del buf
    torch.cuda.empty_cache()
    return g


def run_reference(args, cfg, world):
    """--impl reference: the fp64 oracle as it stands, on all host cores (process per core, each
    on its own node panel), `warmup` untimed passes then `steps` timed passes; rank 0 only."""
    _, rank, _ = _dist_env()
    if rank != 0:
        return
    n = cfg["n"]
    value, W, per, sample = _oracle_pool(cfg, args.nodes_per_core, warm=max(1, args.warmup), passes_fixed=args.steps)
    line = {"metric": METRIC, "value": value, "unit": "it/s", "impl": "reference", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": per * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": _config_dict(args, cfg, world),
            "cpu_baseline": {"value": value, "unit": "it/s", "cores": W, "kind": "oracle", "sample": sample,
                             "host_cores": _host_cores(), "blas_threads_per_process": 1},
            "e2e": {"value": value, "unit": "it/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _config_dict(args, cfg, world):
    n, d = cfg["n"], cfg["d"]
    return {"workload": f"{args.config}: n={n} d={d} sigma={cfg['sigma']:.4f} T={cfg['T']} K={cfg['K']} "
                        f"eta=1/n seed=0; step = spectral init (tol {INIT_TOL}) + T NS-RGS iterations "
                        f"(fused objective trace) + alignment metrics",
            "n": n, "d": d, "N": n * d, "A_bytes_total": 4 * (n * d) ** 2, "parallelism": f"row-block x{world}",
            "l2": "inputs larger than L2 (A shard >> 126 MB); no flush needed" if 4 * (n * d) ** 2 / world > 2e8
            else "A shard fits near L2; numbers are L2-assisted (report only)"}


# ------------------------------------------------------------------------------------ GPU arm
def _side_config(nsrgs, torch, make_solver, name, cfg, steps, warmup, barrier, stream, world, local):
    """Whole-solve it/s and the panel pass's roofline for another BASELINE config on the same
    GPUs (spectral init + T iterations + metrics per step, as the headline)."""
    n, d, T, K = cfg["n"], cfg["d"], cfg["T"], cfg["K"]
    s = make_solver(n, d)
    Zd = torch.from_numpy(s.generate(0, cfg["sigma"])).to(f"cuda:{local}")

    def solve():
        sw = s.init_spectral(0, INIT_MAX_SWEEPS, INIT_TOL)
        s.run(T, 1.0 / n, K, trace=True)
        return sw, s.alignment_error(Zd)

    for _ in range(warmup):
        solve()
    s.reset_stats(timing=True)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        sw, met = solve()
    e1.record(stream)
    barrier()
    ms = e0.elapsed_time(e1)
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    st = s.stats()
    s.close()
    N = n * d
    rows_local = N // world
    avg = st["panel_ms_total"] / max(1, st["panel_launches"])
    bytes_launch = 4 * rows_local * N + 4 * N * d + 4 * rows_local * d
    peak = _peaks()[0]
    return {"config": name, "n": n, "d": d, "T": T, "K": K, "sigma": cfg["sigma"], "n_gpus": world,
            "value": T * steps / (ms / 1e3), "unit": "it/s", "ms_per_step": ms / steps, "init_sweeps": sw,
            "avg_pass_ms": avg, "bytes_per_launch": bytes_launch, "achieved_gbs": bytes_launch / (avg / 1e3) / 1e9,
            "frac_of_peak": bytes_launch / (avg / 1e3) / 1e9 / peak,
            "aggregate_gbs": world * bytes_launch / (avg / 1e3) / 1e9, "rel_err": met[0],
            "rel_err_first_order": cfg["sigma"] * np.sqrt((d - 1) / n),
            "kernel": ("wide_tc_kernel (tcgen05 kind::tf32 3xTF32, TMEM operands + accumulators)" if st.get("wide_tc") == 2
                       else "wide_kernel" if d > 10 else "panel_kernel (fused A.X + epilogue)"),
            "x_exchange": (
                ("fused P2P NVLink stores from the epilogue" if st.get("p2p") else "NCCL all-gather")
                if world > 1 else "none (1 GPU)")}


def run_gpu(args, cfg):
    import torch
    import torch.distributed as dist

    from paper_2604_07372_b200 import nsrgs

    world, rank, local = _dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def make_solver(n_, d_):
        """One context per (config, rank); world > 1: a fresh NCCL unique id broadcast from rank 0."""
        nid_ = None
        if world > 1:
            idt = torch.zeros(128, dtype=torch.uint8, device="cuda")
            if rank == 0:
                idt.copy_(torch.frombuffer(bytearray(nsrgs.get_nccl_unique_id()), dtype=torch.uint8))
            dist.broadcast(idt, 0)
            nid_ = bytes(idt.cpu().numpy().tobytes())
        return nsrgs.Solver(n_, d_, nsrgs.F32, rank=rank, world=world, device=local, nccl_id=nid_, stream=stream)

    n, d, T, K = cfg["n"], cfg["d"], cfg["T"], cfg["K"]
    eta = 1.0 / n
    stream = torch.cuda.Stream()
    s = make_solver(n, d)
    Zh = s.generate(0, cfg["sigma"])                     # A shard generated on the device, resident
    if args.symmetric:
        s.set_symmetric(True)
    Zd = torch.from_numpy(Zh).to(f"cuda:{local}")
    Zpin = torch.from_numpy(Zh).pin_memory()
    Xpin = torch.empty((n, d, d), dtype=torch.float32).pin_memory()

    def solve(e2e=False):
        sw = s.init_spectral(0, INIT_MAX_SWEEPS, INIT_TOL)
        tr = s.run(T, eta, K, trace=True)
        if e2e:
            s.get_X(Xpin)                                # D2H of the result (pinned)
            met = s.alignment_error(Zpin.numpy())        # H2D of the ground truth (pinned)
        else:
            met = s.alignment_error(Zd)
        return sw, tr, met

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(k, e2e):
        barrier()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        out = None
        for _ in range(k):
            out = solve(e2e)
        ev1.record(stream)
        barrier()
        ms = ev0.elapsed_time(ev1)
        if world > 1:
            t = torch.tensor([ms], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms, out

    for _ in range(args.warmup):
        solve()
    s.reset_stats(timing=True)
    with Clocks(local) as clk:
        ms, (sweeps, trace, met) = timed(args.steps, e2e=False)
    st = s.stats()
    clocks = clk.summary()
    s.reset_stats(timing=False)
    ms_e2e, _ = timed(args.steps, e2e=True)

    # NS-RGS vs GPM per-iteration cost on the same A pass (the paper's comparison, PAPER.md:313,
    # :327 "approximately 1.7x"; its hardware: MATLAB on an i9-14900HX CPU)
    def per_iter_ms(fn, iters=10):
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn(iters)
        e1.record(stream)
        barrier()
        return e0.elapsed_time(e1) / iters

    # phase split of one solve (device time): spectral init | T iterations | metrics
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    barrier()
    ev[0].record(stream)
    s.init_spectral(0, INIT_MAX_SWEEPS, INIT_TOL)
    ev[1].record(stream)
    s.run(T, eta, K, trace=True)
    ev[2].record(stream)
    s.alignment_error(Zd)
    ev[3].record(stream)
    barrier()
    phases = {"init_ms": ev[0].elapsed_time(ev[1]), "iterations_ms": ev[1].elapsed_time(ev[2]),
              "metrics_ms": ev[2].elapsed_time(ev[3])}
    phases["iterations_per_sec_run_only"] = T / (phases["iterations_ms"] / 1e3)
    s.init_spectral(0, INIT_MAX_SWEEPS, INIT_TOL)
    rgs_ms = per_iter_ms(lambda k: s.run(k, eta, K, trace=False))
    gpm_ms = per_iter_ms(lambda k: s.gpm_run(k, trace=False))

    N = n * d
    rows_local = N // world
    value = T * args.steps / (ms / 1e3)
    e2e_value = T * args.steps / (ms_e2e / 1e3)
    peak, peak_kind = _peaks()
    # A shard + X^t in + X^{t+1} out; the symmetric pass needs only the upper half
    a_bytes = 4 * (N * (N + 1) // 2) if args.symmetric else 4 * rows_local * N
    bytes_launch = a_bytes + 4 * N * d + 4 * rows_local * d
    avg_ms = st["panel_ms_total"] / max(1, st["panel_launches"])
    achieved = bytes_launch / (avg_ms / 1e3) / 1e9
    passes = st["panel_launches"] / args.steps                              # A passes per solve
    eff_gbs = passes * a_bytes * args.steps / (ms / 1e3) / 1e9 * world
    # in-run ceiling right after the headline's measurements (same instance resident, same clocks /
    # power state), before the variants and side configs
    read_peak = _read_stream_gbs(torch, f"cuda:{local}", stream, reps=10) if not args.no_read_probe else None
    # §8(f) row 1 alongside the headline: the symmetric half-storage pass on the same instance
    sym_variant = None
    if world == 1 and d <= 6 and not args.symmetric and not args.no_sym_variant:
        s.set_symmetric(True)
        for _ in range(max(1, args.warmup - 1)):
            solve()
        s.reset_stats(timing=True)
        with Clocks(local) as clk2:
            ms_sym, (_, _, met_sym) = timed(args.steps, e2e=False)
        st2 = s.stats()
        s.set_symmetric(False)
        avg2 = st2["panel_ms_total"] / max(1, st2["panel_launches"])
        a_sym = 4 * (N * (N + 1) // 2)
        sym_variant = {"value": T * args.steps / (ms_sym / 1e3), "unit": "it/s", "ms_per_step": ms_sym / args.steps,
                       "avg_pass_ms": avg2, "a_bytes_per_pass_algorithmic": a_sym,
                       "a_bytes_per_pass_read": st2["a_bytes_per_pass"],
                       "achieved_gbs": (a_sym + 4 * N * d + 4 * rows_local * d) / (avg2 / 1e3) / 1e9,
                       "rel_err": met_sym[0], "clocks": clk2.summary(),
                       "note": "upper-triangle stream, 2 FMA directions per element (FFMA2/issue-bound, not HBM-bound)"}
    # §8(f) row 2 alongside: incomplete observations (p < 1) on block-sparse
    # storage — the same (n, d, sigma, T, K) with each pair observed with probability p,
    # mu = 1/(np); only observed blocks are stored and streamed
    bsr_variant = None
    if world == 1 and args.bsr_p > 0 and not args.no_bsr_variant:
        pb = args.bsr_p
        sb = nsrgs.Solver(n, d, nsrgs.F32, device=local, stream=stream)
        Zb = torch.from_numpy(sb.generate(0, cfg["sigma"], p=pb, storage="bsr")).to(f"cuda:{local}")

        def solve_b():
            sb.init_spectral(0, INIT_MAX_SWEEPS, INIT_TOL)
            sb.run(T, 1.0 / (n * pb), K, trace=True)
            return sb.alignment_error(Zb)

        for _ in range(max(1, args.warmup - 1)):
            solve_b()
        sb.reset_stats(timing=True)
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            met_b = solve_b()
        e1.record(stream)
        barrier()
        ms_b = e0.elapsed_time(e1)
        stb = sb.stats()
        avgb = stb["panel_ms_total"] / max(1, stb["panel_launches"])
        bsr_variant = {"p": pb, "value": T * args.steps / (ms_b / 1e3), "unit": "it/s", "ms_per_step": ms_b / args.steps,
                       "avg_pass_ms": avgb, "stored_bytes_per_pass": stb["a_bytes_per_pass"],
                       "dense_bytes_per_pass": 4 * rows_local * N, "nnzb": stb["bsr_nnzb"],
                       "achieved_gbs": stb["a_bytes_per_pass"] / (avgb / 1e3) / 1e9,
                       "frac_of_peak": stb["a_bytes_per_pass"] / (avgb / 1e3) / 1e9 / _peaks()[0],
                       "rel_err": met_b[0], "rel_err_first_order": cfg["sigma"] * np.sqrt((d - 1) / (n * pb)),
                       "kernel": "bsr_kernel (warp per node row: bulk-copied A chunks, gathered X_j records, "
                                 "fused epilogue)"}
        sb.close()
    s.close()
    # the other dense BASELINE configs on the same GPUs (driver-visible): c4 (d = 10, FMA
    # co-limited) and the largest, c5 (160 GB; the north star's scaling config)
    side = {}
    for name in args.side_configs.split(",") if args.side_configs else []:
        if name == args.config:
            continue
        c = CONFIGS.get(name) or SIDE_CONFIGS[name]
        if c["n"] % world or 4 * (c["n"] * c["d"]) ** 2 / world > 170e9:     # shard must fit one B200's 180 GB
            continue
        side[name] = _side_config(nsrgs, torch, make_solver, name, c, max(1, args.side_steps), 1, barrier,
                                  stream, world, local)
    if read_peak is not None:   # the ceiling is the best the probe reaches in this run: once more at the end
        read_peak = max(read_peak, _read_stream_gbs(torch, f"cuda:{local}", stream, reps=10))
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        v, W, per, sample = _oracle_pool(cfg, args.nodes_per_core, warm=1, budget_s=args.cpu_budget)
        cpu = {"value": v, "unit": "it/s", "cores": W, "kind": "oracle", "sample": sample + f", {args.cpu_budget:.0f} s",
               "host_cores": _host_cores(), "blas_threads_per_process": 1,
               "single_thread_value": _oracle_single_thread(cfg, args.nodes_per_core)}
    traffic = _traffic(args.config)
    line = {
        "metric": METRIC, "value": value, "unit": "it/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (on-device Philox instance, PAPER.md §4.1 model)",
        "config": {**_config_dict(args, cfg, world), "init_sweeps": sweeps,
                   "storage": "symmetric half (upper triangle read)" if args.symmetric else "dense row-major shard",
                   "x_exchange": ("fused P2P NVLink stores from the epilogue" if st.get("p2p") else "NCCL all-gather")
                   if world > 1 else "none (1 GPU)"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "peak_kind": peak_kind,
                     "kernel": ("wide_tc_kernel (tcgen05 kind::tf32 3xTF32, TMEM operands + accumulators, fused epilogue)"
                                if st.get("wide_tc") == 2 else "panel_kernel (fused A.X + epilogue)"),
                     "bytes_per_launch": bytes_launch, "avg_launch_ms": avg_ms,
                     "frac_of_nominal_8TBs": achieved / 8000.0,
                     "read_stream_gbs_in_run": read_peak,
                     "frac_of_read_stream": achieved / read_peak if read_peak else None},
        "effective_gbs": eff_gbs, "a_passes_per_step": passes, "phases": phases,
        "e2e": {"value": e2e_value, "unit": "it/s", "h2d_bytes_per_step": 4 * n * d * d,
                "d2h_bytes_per_step": 4 * n * d * d + 8 * T + 24},
        "gpu_launches": st["kernel_launches"],
        "gpm_comparison": {"ns_rgs_ms_per_iter": rgs_ms, "gpm_ms_per_iter": gpm_ms, "gpm_over_ns_rgs": gpm_ms / rgs_ms,
                           "paper_context": "NS-RGS ~1.7x faster than GPM per solve (synthetic, PAPER.md:327), "
                                            "~2.3x (Lucy, :376) on MATLAB R2023b / Intel i9-14900HX CPU (:295); "
                                            "on B200 both are bound by the same A pass"},
        "clocks": clocks,
        "result": {"rel_err": met[0], "d_F": met[1], "mse": met[2], "F_first": float(trace[0]),
                   "F_last": float(trace[-1]), "ns_region_max": st["ns_region_max"]},
        "launch": {"grid": st["grid"], "threads": st["threads"], "stages": st["stages"],
                   "rows_per_panel": st["rows_per_panel"], "panels": st["panels"],
                   "cut_panels": st["cut_panels"], "smem": st["smem_bytes"]},
    }
    if cpu:
        line["cpu_baseline"] = cpu
    if sym_variant:
        line["symmetric_variant"] = sym_variant
    if bsr_variant:
        line["bsr_variant"] = bsr_variant
    for name, v in side.items():
        line[f"{name}_line"] = v
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _launch_ranks(argv, gpus):
    """--gpus N > 1 without a torchrun environment: start N ranks on this node (one per GPU) with
    torch.distributed.run on 127.0.0.1, or fail with a clear message if fewer GPUs are visible."""
    import socket

    import torch

    ng = torch.cuda.device_count()
    if ng < gpus:
        print(f"bench.py: --gpus {gpus} needs {gpus} visible GPUs on this node, found {ng}; "
              f"nothing was timed", file=sys.stderr, flush=True)
        sys.exit(2)
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *argv]
    sys.exit(subprocess.call(cmd))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3", help="c1..c5 (headline: c3 at every N, strong scaling)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--nodes-per-core", type=int, default=8, help="oracle sample: nodes per host process")
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--symmetric", action="store_true", help="symmetric half-storage pass (d <= 6, 1 GPU)")
    ap.add_argument("--no-sym-variant", action="store_true", help="skip the extra symmetric-variant measurement")
    ap.add_argument("--no-read-probe", action="store_true", help="skip the in-run read-stream peak probe")
    ap.add_argument("--sigma", type=float, default=None, help="noise level override (c2 lists 0.5, 2 and 8)")
    ap.add_argument("--bsr-p", type=float, default=0.5, help="observation probability of the block-sparse variant")
    ap.add_argument("--no-bsr-variant", action="store_true", help="skip the block-sparse (p < 1) variant")
    ap.add_argument("--side-configs", default="c4,c5,w25",
                    help="other dense configs measured on the same GPUs after the headline ('' = none)")
    ap.add_argument("--side-steps", type=int, default=2)
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    if args.sigma is not None:
        cfg["sigma"] = args.sigma
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is not None and int(env_world) != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={env_world}", file=sys.stderr, flush=True)
        sys.exit(2)
    if args.impl == "reference":
        run_reference(args, cfg, int(env_world) if env_world else args.gpus)
        return
    if args.gpus > 1 and env_world is None:
        _launch_ranks(sys.argv[1:], args.gpus)
    run_gpu(args, cfg)


if __name__ == "__main__":
    main()
