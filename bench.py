#!/usr/bin/env python
"""Benchmark of the Whittaker hot path (BASELINE.json metric) on 1..N B200s.

A step = one forward (whit_forward) + one backward (whit_backward) over the
whole per-GPU batch of the 'hetero' workload (BASELINE.json configs[2]:
262,144 series x T = 3,288 daily steps, d = 2, per-date lambda, fp32 I/O,
fp64 arithmetic).  Multi-GPU: one process per GPU (torchrun), each rank
solves its own shard of independent series (weak scaling, no data-path
collective; torch.distributed/NCCL only for the barrier and the max-over-
ranks timing).

Prints ONE JSON line (rank 0).  `--impl reference` times the CPU oracle
(oracle/, test infrastructure) on the host cores instead.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "series fwd+bwd solves/s (T=3288, d=2, per-date λ) and % of HBM peak, 1/2/4/8 GPU"
UNIT = "series/s"
FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="libwhit", choices=["libwhit", "reference"])
    ap.add_argument("--config", default="hetero", choices=["hetero", "homo", "toy", "s2tile"])
    ap.add_argument("--io", default="f32", choices=["f32", "f64"])
    ap.add_argument("--op", default="fwdbwd", choices=["fwdbwd", "train", "variance", "irregular", "table1"],
                    help="fwdbwd: whit_forward + whit_backward (the BASELINE metric); train: whit_forward_mse "
                         "(fused masked-MSE, NEXT-3) + whit_backward; variance: whit_posterior_variance (NEXT-4); "
                         "irregular: whit_forward_times + whit_backward on T = 350 uneven acquisition dates "
                         "(NEXT-2, the paper's Table 1 length); table1: the paper's Table 1 workload -- C = 10 "
                         "bands per pixel on T = 350 uneven dates, d = 2 (whit_forward_times_bands, NEXT-1 x NEXT-2)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=0, help="series in the CPU-oracle sample (0 = auto)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak (default): the config's B series per GPU; strong: B series for the whole job, "
                         "split over the ranks (fwdbwd op)")
    ap.add_argument("--dist-smoke", action="store_true",
                    help="initialise the NCCL process group even at world size 1 (under torchrun) so the "
                         "barrier / all_reduce / all_gather paths of the multi-GPU run execute on one GPU")
    return ap.parse_args()


# ----------------------------------------------------------------------------- helpers
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def shard(rank: int, world: int, B: int, strong: bool = False):
    """Weak scaling (default): B is per rank and rank r owns the global series [r*B, (r+1)*B).
    Strong scaling: B is the job total, split into contiguous ranges of a multiple of 4 series
    (the fp32 row-stride rule), the last rank taking the remainder.  Returns (offset, count)."""
    if not strong:
        return rank * B, B
    per = (B // world) // 4 * 4
    off = rank * per
    return off, (B - off if rank == world - 1 else per)


def dist_is_init() -> bool:
    import torch.distributed as dist
    return dist.is_available() and dist.is_initialized()


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar over the default process group (identity without one)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_checksums(tensors, world: int) -> dict:
    """Exact per-rank checksums: int64 sum of each tensor's bit patterns (order-independent, so equal
    results give equal sums on any device), all-gathered across ranks (NCCL on the GPU, gloo in the
    CPU tests) outside the timed region."""
    import torch
    import torch.distributed as dist
    sums = torch.stack([t.view(torch.int32 if t.element_size() == 4 else torch.int64).sum(dtype=torch.int64)
                        for t in tensors])
    allsums = [sums]
    if dist.is_available() and dist.is_initialized():
        allsums = [torch.empty_like(sums) for _ in range(dist.get_world_size())]
        dist.all_gather(allsums, sums)
    return {"kind": "int64 sum of the output bit patterns (z, grad_y, grad_lambda) per rank",
            "per_rank": [[int(v) for v in a.tolist()] for a in allsums]}


def measured_peak_gbs():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        v = float(json.load(open(p))["hbm_gbs"])
        return v, "measured (MEASURED_PEAKS.json hbm_gbs, copy r+w)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int, period_ms: int = 50):
        self.dev = device_index
        self.period = period_ms
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-i", str(self.dev), f"-lms={self.period}"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=1)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def algorithmic_bytes(B: int, T: int, d: int, esz: int, per_date: bool, K: int = 16, wbits: bool = False):
    """Bytes each launch must move in the R-mode design: inputs read in the
    up sweep and re-read in the down sweep, outputs written once, fp64 checkpoints.
    wbits: W read as 1 bit per date (4-B words, one per 32 dates) instead of an esz plane."""
    C = math.ceil(T / K)
    nfac, nrhs = d + d * (d - 1) // 2, d
    lam_rows = (T - d) if per_date else 0
    wrow = (4 * math.ceil(T / 32) / T) if wbits else esz  # bytes of w per date
    fwd = (2 * ((T + lam_rows) * esz + T * wrow)    # y, w (+ lambda) read twice
           + (T + (T - d)) * esz                    # z, D z written
           + 2 * C * (nfac + nrhs) * 8              # checkpoints written + read
           + (0 if per_date else esz)) * B          # scalar lambda
    bwd = (2 * ((T + lam_rows) * esz + T * wrow)    # g, w (+ lambda) read twice
           + (T - d) * esz                          # D z read
           + T * esz + (lam_rows * esz if per_date else esz)  # grad_y, grad_lambda written
           + C * nrhs * 8 * 2                       # rhs checkpoints written + read
           + C * nfac * 8                           # factor checkpoints read
           + (0 if per_date else esz) + 4) * B      # scalar lambda, info
    minimum_fwd = ((2 * T + lam_rows) * esz + (2 * T - d) * esz) * B   # single read + z + D z
    minimum_bwd = ((2 * T + lam_rows) * esz + (T - d) * esz + (T + lam_rows) * esz) * B
    return fwd, bwd, minimum_fwd, minimum_bwd


def load_profile_traffic():
    """dram bytes/launch from the committed ncu --set full summary (profiles/), if any."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        return json.load(open(p))
    except Exception:
        return None


# ----------------------------------------------------------------------------- CPU oracle legs
def _oracle_one(args):
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    y, w, lam, g, d = args
    from oracle import whittaker as O1
    t = time.perf_counter()
    O1.forward_backward(y, w, lam, d, g)
    return time.perf_counter() - t


def oracle_pool(cores: int):
    import multiprocessing as mp
    os.environ.update({"OMP_NUM_THREADS": "1", "OPENBLAS_NUM_THREADS": "1", "MKL_NUM_THREADS": "1"})
    pool = mp.get_context("spawn").Pool(cores)
    pool.map(_oracle_warm, range(cores))  # import numpy/scipy/oracle in every worker, untimed
    return pool


def _oracle_warm(_):
    import oracle  # noqa: F401
    return 0


def oracle_rate(hin: dict, n: int, d: int, pool):
    """fwd+bwd series/s of the CPU oracle (O1 dense + refinement) over n series on the pool's processes."""
    items = [(hin["y"][i], hin["w"][i], hin["lam"][i], hin["g"][i], d) for i in range(n)]
    t0 = time.perf_counter()
    per = pool.map(_oracle_one, items, chunksize=1)
    wall = time.perf_counter() - t0
    return n / wall, wall, sum(per)


def _banded_one(args):
    """One series, fwd+bwd, with a conventional CPU banded solver (LAPACK pbsv via scipy's
    solveh_banded, fp64): the context baseline beside the oracle; not the oracle, not the product."""
    import numpy as np
    from scipy.linalg import solveh_banded
    y, w, lam, g, d = args
    t = time.perf_counter()
    T = y.shape[0]
    c = np.array([(-1) ** (d - j) * __import__("math").comb(d, j) for j in range(d + 1)], dtype=np.float64)
    lt = np.zeros(T)
    lt[:T - d] = lam if np.ndim(lam) else lam
    ab = np.zeros((d + 1, T))  # upper band storage: ab[d + i - j, col j] = Omega[row i, col j]
    ab[d] = w.copy()
    for i in range(d + 1):  # Omega[r+i, r+j] += lambda_r c_i c_j over the difference rows r
        for j in range(i, d + 1):
            ab[d + i - j, j:j + T - d] += lt[:T - d] * (c[i] * c[j])
    b = np.where(w != 0, w * np.nan_to_num(y), 0.0)
    z = solveh_banded(ab, b)
    u = solveh_banded(ab, g)
    dz = np.convolve(z, c[::-1], "valid")
    du = np.convolve(u, c[::-1], "valid")
    _ybar, _lbar = w * u, -du * dz
    return time.perf_counter() - t


def banded_rate(hin: dict, n: int, d: int, pool):
    items = [(hin["y"][i], hin["w"][i], hin["lam"][i], hin["g"][i], d) for i in range(n)]
    t0 = time.perf_counter()
    pool.map(_banded_one, items, chunksize=max(1, n // (4 * (pool._processes or 1))))
    wall = time.perf_counter() - t0
    return n / wall, wall


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def sample_host_inputs(x: dict, n: int):
    """n series spread over the shard, copied to host (series-major float64)."""
    import numpy as np
    import torch
    B = x["y"].shape[1]
    idx = torch.linspace(0, B - 1, n).long().to(x["y"].device)
    out = {}
    for k in ("y", "w", "lam", "g"):
        v = x[k]
        v = v[:, idx] if v.dim() == 2 else v[idx]
        a = v.double().cpu().numpy()
        out[k] = np.ascontiguousarray(a.T) if a.ndim == 2 else a
    return out


# ----------------------------------------------------------------------------- reference arm
def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    import torch
    import synth
    cfg = synth.CONFIGS[args.config]
    cores = min(host_cores(), 32)
    n = args.cpu_sample or cores
    # the same workload's series (global ids spread over the batch), generated on the host
    ids = torch.linspace(0, cfg.B - 1, n).long()
    x = synth.make_inputs(cfg, device="cpu", dtype=torch.float32 if args.io == "f32" else torch.float64,
                          series_ids=ids)
    hin = sample_host_inputs(x, n)
    pool = oracle_pool(cores)
    for _ in range(args.warmup):
        oracle_rate(hin, min(n, cores), cfg.d, pool)
    rates, walls = [], []
    for _ in range(args.steps):
        r, wall, _cpu = oracle_rate(hin, n, cfg.d, pool)
        rates.append(r)
        walls.append(wall)
    pool.close()
    value = statistics.median(rates)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 0, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": statistics.median(walls) * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.config, "B": cfg.B, "T": cfg.T, "d": cfg.d, "lambda": cfg.lam_mode,
                   "io": args.io, "sample_series_per_step": n},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": f"{n} series of the {args.config} workload per step, O1 dense fp64 + 2 long-double "
                                   f"refinement steps, fwd+bwd, {cores} processes"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- libwhit arm
def run_libwhit(args):
    import torch
    import torch.distributed as dist

    ws_n, rank, local = dist_env()
    if ws_n != args.gpus:
        if ws_n == 1 and args.gpus > 1:
            print(json.dumps({"error": f"--gpus {args.gpus} needs torchrun with {args.gpus} processes"}))
            return 2
    if ws_n > 1 or args.dist_smoke:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local if ws_n > 1 else 0)
    torch.cuda.set_device(dev)
    distributed = dist.is_initialized()

    import paper_2604_00048_b200 as P
    import synth

    if args.config == "s2tile":
        return run_s2tile(args, P, synth, dev, ws_n, rank)
    cfg = synth.CONFIGS[args.config]
    io = torch.float32 if args.io == "f32" else torch.float64
    esz = 4 if io == torch.float32 else 8
    B, T, d = cfg.B, cfg.T, cfg.d
    per_date = cfg.lam_mode == "per_date"
    strong = args.scaling == "strong" and args.op == "fwdbwd"
    B_job = B if strong else ws_n * B
    off, B = shard(rank, ws_n, B, strong)
    x = synth.make_inputs(cfg, B=B, series_offset=off, device=dev, dtype=io)
    y, w, lam, g = x["y"], x["w"], x["lam"], x["g"]
    stream = torch.cuda.current_stream(dev)
    wsp = P.Workspace(d, T, B, io, per_date, device=dev, stream=stream)
    z = torch.empty_like(y)
    gy = torch.empty_like(y)
    gl = torch.empty_like(lam)

    if args.op in ("irregular", "table1"):
        del x, y, w, lam, g, z, gy, gl, wsp
        torch.cuda.empty_cache()
        if args.op == "table1":
            return run_table1(args, P, synth, io, dev, stream, ws_n, rank)
        return run_irregular(args, P, synth, cfg, io, dev, stream, ws_n, rank)
    if args.op != "fwdbwd":
        return run_op(args, P, x, wsp, d, T, B, io, dev, stream, ws_n, rank)

    def step():
        P.whit_forward(y, w, lam, d, T, B, z, wsp)
        P.whit_backward(g, wsp, z, gy, gl)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    nfail = P.whit_failures(wsp)

    K = args.steps
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(K)]
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clk = ClockSampler(dev.index if dev.index is not None else 0)
    if distributed:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clk.start()
    time.sleep(0.15)  # let the sampler attach before the timed region
    t_start.record(stream)
    for i in range(K):
        ev[i][0].record(stream)
        P.whit_forward(y, w, lam, d, T, B, z, wsp)
        ev[i][1].record(stream)
        P.whit_backward(g, wsp, z, gy, gl)
        ev[i][2].record(stream)
    t_end.record(stream)
    torch.cuda.synchronize(dev)
    if distributed:
        dist.barrier()
    clocks = clk.stop()
    total_ms = t_start.elapsed_time(t_end)
    fwd_ms = [e[0].elapsed_time(e[1]) for e in ev]
    bwd_ms = [e[1].elapsed_time(e[2]) for e in ev]
    ms_step = max_over_ranks(total_ms / K, dev)
    value = B_job / (ms_step / 1e3)

    # per-rank checksums of the outputs (exact: int64 sums of the bit patterns, order-independent), gathered
    # over NCCL outside the timed region.  Rank r owns global series [r*B, (r+1)*B) at every N, so rank r's
    # checksum is the same at every world size (results are bitwise independent of placement).
    checksums = gather_checksums((z, gy, gl), ws_n)

    # roofline of the dominant kernel
    fb, bb, mf, mb = algorithmic_bytes(B, T, d, esz, per_date)
    f_avg, b_avg = statistics.mean(fwd_ms), statistics.mean(bwd_ms)
    dom = "whit_backward" if b_avg >= f_avg else "whit_forward"
    dom_ms, dom_bytes, dom_min = (b_avg, bb, mb) if dom == "whit_backward" else (f_avg, fb, mf)
    peak, peak_src = measured_peak_gbs()
    achieved = dom_bytes / (dom_ms / 1e3) / 1e9
    prof = load_profile_traffic() or {}
    traffic = prof.get(dom, {}).get("dram_bytes_per_launch") if isinstance(prof.get(dom), dict) else None
    roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": traffic,
            "kernel": dom, "kernel_ms": round(dom_ms, 4), "algorithmic_bytes": dom_bytes,
            "minimum_bytes": dom_min, "peak_source": peak_src,
            "traffic_source": prof.get("source") if traffic is not None else None,
            "fwd_ms": round(f_avg, 4), "bwd_ms": round(b_avg, 4),
            "step_GBps_algorithmic": round((fb + bb) / (ms_step / 1e3) / 1e9, 1),
            "step_frac_of_min_bytes": round((mf + mb) / (ms_step / 1e3) / 1e9 / peak, 4)}

    # the same step with the binary W bit-packed (whit_forward_wbits), reported beside the headline
    wbits_line = None
    if args.config == "hetero":
        bits = P.whit_pack_mask(w)
        for _ in range(3):
            P.whit_forward_wbits(y, bits, lam, d, T, B, z, wsp)
            P.whit_backward(g, wsp, z, gy, gl)
        torch.cuda.synchronize(dev)
        evb = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(K)]
        t_start.record(stream)
        for i in range(K):
            evb[i][0].record(stream)
            P.whit_forward_wbits(y, bits, lam, d, T, B, z, wsp)
            evb[i][1].record(stream)
            P.whit_backward(g, wsp, z, gy, gl)
            evb[i][2].record(stream)
        t_end.record(stream)
        torch.cuda.synchronize(dev)
        msb = max_over_ranks(t_start.elapsed_time(t_end) / K, dev)
        fbb, bbb, _, _ = algorithmic_bytes(B, T, d, esz, per_date, wbits=True)
        fa = statistics.mean(e[0].elapsed_time(e[1]) for e in evb)
        ba = statistics.mean(e[1].elapsed_time(e[2]) for e in evb)
        domb, dms, dbytes = ("whit_backward", ba, bbb) if ba >= fa else ("whit_forward_wbits", fa, fbb)
        ach = dbytes / (dms / 1e3) / 1e9
        wbits_line = {"value": B_job / (msb / 1e3), "unit": UNIT, "ms_per_step": msb,
                      "w_format": "uint32 bit planes [ceil(T/32)][B] (binary W, P:26), whit_forward_wbits",
                      "gpu_launches": 2 * K,
                      "roofline": {"bound": "hbm", "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
                                   "frac": round(ach / peak, 4), "kernel": domb, "kernel_ms": round(dms, 4),
                                   "algorithmic_bytes": dbytes, "fwd_ms": round(fa, 4), "bwd_ms": round(ba, 4)}}
        del bits

    # end to end through the public API with host buffers (rank-local); also with the binary W shipped
    # as bits (whit_run_host_wbits), reported beside it
    e2e = None
    e2e_wbits = None
    if not args.no_e2e:
        bits_h = P.whit_pack_mask(w).cpu() if args.config == "hetero" else None
        del wsp, z, gy, gl
        torch.cuda.empty_cache()
        e2e = run_e2e(P, x, d, T, B, io, stream, dev, args.e2e_steps, B_job=B_job)
        if bits_h is not None:
            e2e_wbits = run_e2e(P, x, d, T, B, io, stream, dev, args.e2e_steps, wbits=bits_h, B_job=B_job)

    # CPU oracle baseline (rank 0, N = 1 only), and a conventional CPU banded solver for context
    cpu = None
    cpu_banded = None
    if rank == 0 and ws_n == 1 and not args.no_cpu_baseline:
        cores = min(host_cores(), 32)
        n = args.cpu_sample or 2 * cores
        hin = sample_host_inputs(x, n)
        pool = oracle_pool(cores)
        rate, wall, cpu_s = oracle_rate(hin, n, d, pool)
        nb = 256 * cores
        hb = sample_host_inputs(x, nb)
        banded_rate(hb, cores, d, pool)  # warm the workers' scipy import
        brate, bwall = banded_rate(hb, nb, d, pool)
        pool.close()
        cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": "oracle",
               "sample": f"{n} series of this workload (spread over the batch), O1 dense fp64 + long-double "
                         f"refinement, fwd+bwd, {cores} processes, {wall:.1f} s wall / {cpu_s:.1f} s CPU"}
        cpu_banded = {"value": brate, "unit": UNIT, "cores": cores,
                      "kind": "context: scipy.linalg.solveh_banded (LAPACK pbsv) fp64, band assembled in numpy, "
                              "forward + adjoint solve + gradients",
                      "sample": f"{nb} series of this workload, {cores} processes, {bwall:.2f} s wall"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws_n, "steps": K, "warmup": args.warmup,
            "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong" if strong else "weak",
            "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.config, "B_per_gpu": B, "T": T, "d": d, "lambda": cfg.lam_mode,
                       "io": args.io, "global_batch": B_job, "parallelism": f"dp{ws_n}",
                       "l2": "inputs larger than L2 (each [T][B] plane %.2f GB vs 126 MB L2)" % (T * B * esz / 1e9),
                       "mask": "Sentinel-2 revisit + seasonal clouds, 90-day trailing gap",
                       "failed_series": nfail},
            "roofline": roof, "gpu_launches": 2 * K, "clocks": clocks, "e2e": e2e, "cpu_baseline": cpu,
            "cpu_banded": cpu_banded,
            "w_bits": wbits_line, "e2e_wbits": e2e_wbits, "checksums": checksums,
        }
        print(json.dumps(line), flush=True)
    if distributed:
        dist.destroy_process_group()
    return 0


def run_op(args, P, x, wsp, d, T, B, io, dev, stream, ws_n, rank):
    """NEXT-row measurements on the same workload: 'train' = whit_forward_mse (the paper's masked
    MSE on 20 % held-out dates) + whit_backward; 'variance' = whit_posterior_variance."""
    import torch
    y, w, lam = x["y"], x["w"], x["lam"]
    if args.op == "train":
        gen = torch.Generator(device=dev).manual_seed(1)
        held = (torch.rand(w.shape, device=dev, generator=gen) < 0.2) & (w > 0)
        w = w.masked_fill(held, 0.0)
        lw = held.to(io)
        del held
        z, gz, gy = torch.empty_like(y), torch.empty_like(y), torch.empty_like(y)
        gl, loss = torch.empty_like(lam), torch.empty(B, dtype=io, device=dev)

        def step():
            P.whit_forward_mse(y, w, lam, lw, d, T, B, z, gz, loss, wsp)
            P.whit_backward(gz, wsp, z, gy, gl)
        metric, launches = "training steps (fused masked-MSE fwd + bwd) series/s", 2
    else:
        var = torch.empty_like(w)

        def step():
            P.whit_posterior_variance(w, lam, d, T, B, var, wsp)
        metric, launches = "posterior variance diag(Omega^-1) series/s", 1
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clk = ClockSampler(dev.index or 0)
    clk.start()
    time.sleep(0.15)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    clocks = clk.stop()
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, dev)
    if rank == 0:
        print(json.dumps({"metric": metric, "value": ws_n * B / (ms / 1e3), "unit": UNIT, "n_gpus": ws_n,
                          "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
                          "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                          "config": {"workload": args.config, "op": args.op, "B_per_gpu": B, "T": T, "d": d,
                                     "io": args.io, "l2": "inputs larger than L2"},
                          "gpu_launches": launches * args.steps, "clocks": clocks}), flush=True)
    return 0


def run_irregular(args, P, synth, cfg, io, dev, stream, ws_n, rank):
    """NEXT-2: T = 350 uneven per-series acquisition dates (Table 1's length), d = 2,
    per-date lambda; whit_forward_times + whit_backward over B series per GPU."""
    import torch
    T, d = 350, 2
    B = cfg.B
    off, B = shard(rank, ws_n, B)
    x = synth.make_inputs("hetero", B=B, T=T, d=d, series_offset=off, device=dev, dtype=io, mask="bernoulli")
    tt = synth.make_times(B, T, series_offset=off, device=dev, dtype=io)
    y, w, lam, g = x["y"], x["w"], x["lam"], x["g"]
    wsp = P.Workspace(d, T, B, io, True, device=dev, stream=stream, times=True)
    z, gy, gl = torch.empty_like(y), torch.empty_like(y), torch.empty_like(lam)

    def step():
        P.whit_forward_times(y, w, lam, tt, d, T, B, z, wsp)
        P.whit_backward(g, wsp, z, gy, gl)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, dev)
    if rank == 0:
        print(json.dumps({"metric": "irregular-grid series fwd+bwd solves/s (T=350 acquisitions, d=2, per-date λ)",
                          "value": ws_n * B / (ms / 1e3), "unit": UNIT, "n_gpus": ws_n, "steps": args.steps,
                          "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
                          "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                          "config": {"workload": "irregular", "B_per_gpu": B, "T": T, "d": d, "io": args.io,
                                     "times": "cumulative gaps U{1..12} days"},
                          "paper_context": "Table 1 (V100, PyTorch, T=350, C=10, order 2, batch 28672): 0.14 s "
                                           "-> ~2.0 M band-series/s",
                          "gpu_launches": 2 * args.steps}), flush=True)
    return 0


def run_table1(args, P, synth, io, dev, stream, ws_n, rank):
    """The paper's Table 1 workload: C = 10 bands per pixel on T = 350 uneven
    acquisition dates, order d = 2, per-date lambda; whit_forward_times_bands + whit_backward_bands
    (one shared factor per pixel) over 262,144 pixels per GPU."""
    import torch
    T, d, C, B = 350, 2, 10, 262144
    off, B = shard(rank, ws_n, B)
    x = synth.make_inputs_bands("hetero", C, B=B, T=T, d=d, series_offset=off, device=dev, dtype=io,
                                mask="bernoulli")
    tt = synth.make_times(B, T, series_offset=off, device=dev, dtype=io)
    y, w, lam, g = x["y"], x["w"], x["lam"], x["g"]
    wsp = P.Workspace(d, T, B, io, True, device=dev, stream=stream, C=C, times=True)
    z, gy, gl = torch.empty_like(y), torch.empty_like(y), torch.empty_like(lam)

    def step():
        P.whit_forward_times_bands(y, w, lam, tt, d, T, B, C, z, wsp)
        P.whit_backward_bands(g, wsp, z, gy, gl)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, dev)
    if rank == 0:
        print(json.dumps({"metric": "band-series fwd+bwd solves/s (Table 1 workload: C=10 bands, T=350 uneven "
                                    "dates, d=2, per-date λ)",
                          "value": ws_n * B * C / (ms / 1e3), "unit": "band-series/s", "n_gpus": ws_n,
                          "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
                          "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                          "config": {"workload": "table1", "bands": C, "pixels_per_gpu": B, "T": T, "d": d,
                                     "io": args.io, "times": "cumulative gaps U{1..12} days"},
                          "pixels_per_s": ws_n * B / (ms / 1e3),
                          "paper_context": "Table 1 (V100, PyTorch banded, T=350, C=10, order 2, batch 28672): "
                                           "0.14 s -> ~2.0 M band-series/s",
                          "gpu_launches": 2 * args.steps}), flush=True)
    return 0


def run_s2tile(args, P, synth, dev, ws_n, rank):
    """BASELINE configs[3]: Sentinel-2 tile chunk, 10 bands x 1,048,576 pixels, T = 3288, d = 2,
    per-date lambda per pixel, pixel-sharded over N GPUs.  Each rank holds its 1/8-tile share
    (131,072 pixels x 10 bands: the N = 8 shard, weak scaling) and runs the multi-band
    shared-factor path (whit_forward_bands / whit_backward_bands, NEXT-1)."""
    import torch
    C, Bp, d = 10, 1048576 // 8, 2
    off, Bp = shard(rank, ws_n, Bp)
    x = synth.make_inputs_bands("hetero", C, B=Bp, series_offset=off, device=dev)
    y, w, lam, g = x["y"], x["w"], x["lam"], x["g"]
    T = y.shape[1]
    stream = torch.cuda.current_stream(dev)
    wsp = P.Workspace(d, T, Bp, torch.float32, True, device=dev, stream=stream, C=C)
    z, gy, gl = torch.empty_like(y), torch.empty_like(y), torch.empty_like(lam)

    def step():
        P.whit_forward_bands(y, w, lam, d, T, Bp, C, z, wsp)
        P.whit_backward_bands(g, wsp, z, gy, gl)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clk = ClockSampler(dev.index or 0)
    clk.start()
    time.sleep(0.15)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    clocks = clk.stop()
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, dev)
    nfail = P.whit_failures(wsp)
    # end to end from pinned HOST memory through whit_run_host_bands (pixel chunks streamed through the
    # shared-factor kernels, copies overlapped with compute)
    e2e = None
    if not args.no_e2e:
        del wsp, z, gy, gl
        torch.cuda.empty_cache()
        h = {k: torch.empty(x[k].shape, dtype=torch.float32, pin_memory=True) for k in ("y", "w", "lam", "g")}
        for k in h:
            h[k].copy_(x[k])
        oz = torch.empty(h["y"].shape, dtype=torch.float32, pin_memory=True)
        oy = torch.empty(h["y"].shape, dtype=torch.float32, pin_memory=True)
        ol = torch.empty(h["lam"].shape, dtype=torch.float32, pin_memory=True)
        buf = P.whit_run_host_bands(h["y"], h["w"], h["lam"], h["g"], d, oz, oy, ol, chunk=4096, nbuf=4,
                                    stream=stream)
        torch.cuda.synchronize(dev)
        if dist_is_init():
            import torch.distributed as dist
            dist.barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(args.e2e_steps):
            P.whit_run_host_bands(h["y"], h["w"], h["lam"], h["g"], d, oz, oy, ol, chunk=4096, nbuf=4, dev_buf=buf,
                                  stream=stream)
        f1.record(stream)
        torch.cuda.synchronize(dev)
        ems = max_over_ranks(f0.elapsed_time(f1) / args.e2e_steps, dev)
        e2e = {"value": ws_n * Bp * C / (ems / 1e3), "unit": "band-series/s",
               "h2d_bytes_per_step": sum(t.numel() * 4 for t in h.values()),
               "d2h_bytes_per_step": sum(t.numel() * 4 for t in (oz, oy, ol)), "ms_per_step": ems,
               "steps": args.e2e_steps, "api": "whit_run_host_bands (C-ABI, pinned host buffers, chunk 4096, 4 streams)"}
    if rank == 0:
        print(json.dumps({
            "metric": "band-series fwd+bwd solves/s (Sentinel-2 tile chunk, shared factor per pixel)",
            "value": ws_n * Bp * C / (ms / 1e3), "unit": "band-series/s", "n_gpus": ws_n, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "s2tile", "bands": C, "pixels_per_gpu": Bp, "tile_pixels": 1048576, "T": T,
                       "d": d, "lambda": "per_date", "io": "f32", "parallelism": f"dp{ws_n}",
                       "l2": "inputs larger than L2", "failed_series": nfail},
            "pixels_per_s": ws_n * Bp / (ms / 1e3), "gpu_launches": 2 * args.steps, "clocks": clocks,
            "e2e": e2e}), flush=True)
    return 0


def run_e2e(P, x, d, T, B, io, stream, dev, steps, chunk=8192, nbuf=6, wbits=None, B_job=None):
    """Same metric through the public C-ABI with pinned HOST buffers: whit_run_host streams the
    batch in series chunks (pitched 2-D H2D copies of y, w, lambda, g; whit_forward +
    whit_backward; D2H of z, grad_y, grad_lambda), copies overlapping kernels on nbuf streams.
    With ``wbits`` (host bit-packed W) the weights cross PCIe as bits (whit_run_host_wbits)."""
    import torch
    keys = ("y", "lam", "g") if wbits is not None else ("y", "w", "lam", "g")
    h = {k: torch.empty(x[k].shape, dtype=io, pin_memory=True) for k in keys}
    for k in h:
        h[k].copy_(x[k])
    if wbits is not None:
        h["wbits"] = wbits.pin_memory()
    oz = torch.empty(x["y"].shape, dtype=io, pin_memory=True)
    oy = torch.empty(x["y"].shape, dtype=io, pin_memory=True)
    ol = torch.empty(x["lam"].shape, dtype=io, pin_memory=True)
    h2d = sum(t.numel() * t.element_size() for t in h.values())
    d2h = sum(t.numel() * t.element_size() for t in (oz, oy, ol))
    hw = h.get("w", h["y"])
    bits = h.get("wbits")
    buf = P.whit_run_host(h["y"], hw, h["lam"], h["g"], d, oz, oy, ol, chunk=chunk, nbuf=nbuf, stream=stream,
                          wbits=bits)
    torch.cuda.synchronize(dev)
    ws_n = int(os.environ.get("WORLD_SIZE", "1"))
    import torch.distributed as dist
    if dist.is_initialized():
        dist.barrier()  # ranks share the host's memory and PCIe: start the timed region together
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        P.whit_run_host(h["y"], hw, h["lam"], h["g"], d, oz, oy, ol, chunk=chunk, nbuf=nbuf, dev_buf=buf,
                        stream=stream, wbits=bits)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    ms = max_over_ranks(e0.elapsed_time(e1) / steps, dev)
    return {"value": (B_job or ws_n * B) / (ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h,
            "ms_per_step": ms, "steps": steps,
            "api": f"{'whit_run_host_wbits' if bits is not None else 'whit_run_host'} (C-ABI, pinned host buffers, "
                   f"chunk {chunk}, {nbuf} streams)"}


def main():
    args = parse()
    args.warmup = max(args.warmup, 3)  # the timing rules need >= 3 warm-up steps; the line reports what ran
    if args.impl == "reference":
        return run_reference(args)
    return run_libwhit(args)


if __name__ == "__main__":
    sys.exit(main())
