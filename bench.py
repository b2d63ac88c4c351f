#!/usr/bin/env python
"""Benchmark of the Whittaker hot path (BASELINE.json metric) on 1..N B200s.

A step = one forward (whit_forward) + one backward (whit_backward) over the
whole per-GPU batch of the 'hetero' workload (BASELINE.json configs[2]:
262,144 series x T = 3,288 daily steps, d = 2, per-date lambda, fp32 I/O,
fp64 arithmetic).  Multi-GPU: one process per GPU, each rank solves its own
shard of independent series (weak scaling, no data-path collective;
torch.distributed/NCCL only for the barrier, the max-over-ranks timing and
the checksum gather).  `python bench.py --gpus N` re-launches itself under
torch.distributed.run when it is not already running under it.

Prints ONE JSON line (rank 0).  `--impl reference` times the CPU oracle
(oracle/, test infrastructure) on the host cores instead.  `--dist-check`
runs only the multi-process plumbing (gloo on a CPU-only host) and prints a
check line, no measurement.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# BASELINE.json's metric (the headline: hetero, fwd+bwd); the other workloads name their own
METRIC = "series fwd+bwd solves/s (T=3288, d=2, per-date λ) and % of HBM peak, 1/2/4/8 GPU"
METRICS = {
    "hetero": METRIC,
    "homo": "series fwd+bwd solves/s (T=3288, d=2, scalar λ per series) and % of HBM peak, 1/2/4/8 GPU",
    "toy": "series forward solves/s (T=365, d=2, scalar λ per series)",
}
UNIT = "series/s"
FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback
S2TILE_PIXELS = 1048576
S2TILE_CHUNK = S2TILE_PIXELS // 8  # pixels resident per GPU at a time (the N = 8 shard)


def parse(argv=None):
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
    ap.add_argument("--no-extras", action="store_true", help="skip the bit-packed-W side measurement")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=0, help="series in the CPU-oracle sample (0 = auto)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak (default): the config's B series per GPU; strong: B series for the whole job, "
                         "split over the ranks (s2tile: the whole 1,048,576-pixel tile split over the ranks, "
                         "each rank's share processed in resident chunks of 131,072 pixels)")
    ap.add_argument("--dist-smoke", action="store_true",
                    help="initialise the NCCL process group even at world size 1 (under torchrun) so the "
                         "barrier / all_reduce / all_gather paths of the multi-GPU run execute on one GPU")
    ap.add_argument("--checksum-ranges", type=int, default=0,
                    help="weak scaling, N = 1: also solve the global series ranges [r*B, (r+1)*B) for r < R (untimed) "
                         "and report their output checksums -- rank r of an N = R run must reproduce range r bit for bit")
    ap.add_argument("--dist-check", action="store_true",
                    help="run only the multi-process plumbing (shards, rank-keyed inputs, barrier, max over "
                         "ranks, checksum gather; NCCL with GPUs, gloo without) on a small workload and print a "
                         "check line -- no measurement")
    return ap.parse_args(argv)


# ----------------------------------------------------------------------------- launching
def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def self_launch(argv, gpus: int) -> int:
    """`bench.py --gpus N` outside torchrun: re-execute this script under torch.distributed.run with N
    processes on this node (rendezvous on 127.0.0.1), exactly as the driver launches it for N > 1."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + list(argv)
    return subprocess.call(cmd, cwd=ROOT)


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


def local_checksums(tensors) -> list:
    """int64 sum of each tensor's bit patterns (no communication)."""
    import torch
    return [int(t.contiguous().view(torch.int32 if t.element_size() == 4 else torch.int64).sum(dtype=torch.int64))
            for t in tensors]


def gather_checksums(tensors, world: int) -> dict:
    """Exact per-rank checksums: int64 sum of each tensor's bit patterns (order-independent, so equal
    results give equal sums on any device), all-gathered across ranks (NCCL on the GPU, gloo in the
    CPU tests) outside the timed region."""
    import torch
    import torch.distributed as dist
    sums = torch.tensor(local_checksums(tensors), dtype=torch.int64, device=tensors[0].device)
    allsums = [sums]
    if dist.is_available() and dist.is_initialized():
        allsums = [torch.empty_like(sums) for _ in range(dist.get_world_size())]
        dist.all_gather(allsums, sums)
    return {"kind": "int64 sum of the output bit patterns per rank",
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
            # wait for nvidia-smi's first sample (its start-up can outlast a short timed region), then keep only
            # the samples taken from here on
            t = time.time()
            while not self.lines and time.time() - t < 5.0 and self.proc.poll() is None:
                time.sleep(0.02)
            self.lines.clear()
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


def timed_steps(launches, steps: int, warmup: int, dev, stream, clocks: bool = True):
    """Run `warmup` untimed steps, then time exactly `steps` steps of the launch sequence with CUDA events
    on `stream` (each launch bracketed by its own events), a barrier + synchronize on both sides.
    launches: [(name, fn)].  Returns (ms per step, max over ranks), {name: mean ms per launch}, clocks."""
    import torch
    import torch.distributed as dist
    for _ in range(warmup):
        for _, fn in launches:
            fn()
    torch.cuda.synchronize(dev)
    n = len(launches)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(n + 1)] for _ in range(steps)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clk = ClockSampler(dev.index if dev.index is not None else 0) if clocks else None
    if dist_is_init():
        dist.barrier()
    torch.cuda.synchronize(dev)
    if clk:
        clk.start()  # (returns once the sampler delivers samples)
    t0.record(stream)
    for i in range(steps):
        for j, (_, fn) in enumerate(launches):
            ev[i][j].record(stream)
            fn()
        ev[i][n].record(stream)
    t1.record(stream)
    torch.cuda.synchronize(dev)
    if dist_is_init():
        dist.barrier()
    ck = clk.stop() if clk else None
    per = {name: statistics.mean(ev[i][j].elapsed_time(ev[i][j + 1]) for i in range(steps))
           for j, (name, _) in enumerate(launches)}
    ms = max_over_ranks(t0.elapsed_time(t1) / steps, dev)
    return ms, per, ck


def roofline(kernel_bytes: dict, per_ms: dict, ms_step: float, minimum: dict | None = None, traffic=None,
             extra: dict | None = None):
    """HBM roofline of the dominant kernel (largest mean launch time): ALGORITHMIC bytes of one launch
    (the byte model of DESIGN.md §6) / its mean launch time, against the measured copy peak."""
    peak, peak_src = measured_peak_gbs()
    dom = max(per_ms, key=per_ms.get)
    achieved = kernel_bytes[dom] / (per_ms[dom] / 1e3) / 1e9
    tot = sum(kernel_bytes.values())
    r = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
         "frac": round(achieved / peak, 4), "traffic": None, "kernel": dom, "kernel_ms": round(per_ms[dom], 4),
         "algorithmic_bytes": kernel_bytes[dom], "peak_source": peak_src,
         "launch_ms": {k: round(v, 4) for k, v in per_ms.items()},
         "step_GBps_algorithmic": round(tot / (ms_step / 1e3) / 1e9, 1)}
    if minimum:
        r["minimum_bytes"] = minimum.get(dom)
        r["step_frac_of_min_bytes"] = round(sum(minimum.values()) / (ms_step / 1e3) / 1e9 / peak, 4)
    if traffic is not None:
        r.update(traffic)
    if extra:
        r.update(extra)
    return r


# ----------------------------------------------------------------------------- byte models
def chunk_rows(d: int) -> int:
    """Checkpoint interval / TMA tile rows of the single-series daily-grid kernels (whit::Tile::K)."""
    return 16 if d <= 2 else 12


def algorithmic_bytes(B: int, T: int, d: int, esz: int, per_date: bool, K: int | None = None, wbits: bool = False,
                      wdet: bool = False):
    """Bytes each launch must move in the R-mode design: inputs read in the up sweep and
    re-read in the down sweep, outputs written once, fp64 checkpoints.  K = the checkpoint interval of
    the kernel (16 for d <= 2, 12 for d = 3).  wbits: W read as 1 bit per date (4-B words, one per 32
    dates) instead of an esz plane.  wdet: the forward reads the float W plane once (up sweep) and writes
    its bit plane; the down sweep and both backward sweeps read the bits (binary W detected in the
    forward).  Returns (forward, backward, forward minimum, backward minimum) bytes per launch."""
    K = K or chunk_rows(d)
    C = math.ceil(T / K)
    nfac, nrhs = d + d * (d - 1) // 2, d
    lam_rows = (T - d) if per_date else 0
    lam_dn = lam_rows  # (the d rows by which adjacent down-sweep boxes overlap come from L2, not HBM)
    bitrow = 4 * math.ceil(T / 32) / T                       # bytes of bit-packed w per date
    wrow = bitrow if wbits else esz
    w_fwd = T * (esz + bitrow + bitrow) if wdet else 2 * T * wrow  # wdet: float up, bits written + read
    w_bwd = 2 * T * (bitrow if (wdet or wbits) else esz)
    fwd = (2 * T * esz + w_fwd + (lam_rows + lam_dn) * esz  # y twice, w, lambda twice
           + (T + (T - d)) * esz                             # z, D z written
           + 2 * C * (nfac + nrhs) * 8                       # checkpoints written + read
           + (0 if per_date else esz) + 4) * B               # scalar lambda, info
    bwd = (2 * T * esz + w_bwd + (lam_rows + lam_dn) * esz  # g twice, w, lambda twice
           + (T - d) * esz                                   # D z read
           + T * esz + (lam_rows * esz if per_date else esz)  # grad_y, grad_lambda written
           + C * nrhs * 8 * 2                                # rhs checkpoints written + read
           + C * nfac * 8                                    # factor checkpoints read
           + (0 if per_date else esz) + 4) * B               # scalar lambda, info
    minimum_fwd = ((2 * T + lam_rows) * esz + (2 * T - d) * esz) * B   # single read + z + D z
    minimum_bwd = ((2 * T + lam_rows) * esz + (T - d) * esz + (T + lam_rows) * esz) * B
    return fwd, bwd, minimum_fwd, minimum_bwd


def loss_fwd_extra_bytes(B: int, T: int, esz: int):
    """The fused masked-MSE forward also reads the loss weights (down sweep) and writes grad_z and the loss."""
    return (2 * T * esz + esz) * B


def variance_bytes(B: int, T: int, d: int, esz: int, per_date: bool):
    """Posterior variance: w (+ lambda) read in both sweeps, diag written once, factor checkpoints."""
    K = chunk_rows(d)
    C = math.ceil(T / K)
    nfac = d + d * (d - 1) // 2
    lam = 2 * (T - d) if per_date else 0  # (box overlaps come from L2)
    return (2 * T * esz + lam * esz + T * esz + 2 * C * nfac * 8 + (0 if per_date else esz) + 4) * B


def irregular_bytes(B: int, T: int, d: int, esz: int, per_date: bool, K: int = 8):
    """Single-series uneven grid (K = 8 row chunks): inputs (and the dates) read in both sweeps, outputs once,
    fp64 checkpoints; the dates tile carries K + 2d rows per chunk, the overlap served by L2."""
    C = math.ceil(T / K)
    nfac, nrhs = d + d * (d - 1) // 2, d
    lam = 2 * (T - d) if per_date else 0
    times = 2 * T  # (the 2d rows by which adjacent date boxes overlap come from L2)
    fwd = (2 * T * esz + 2 * T * esz + lam * esz + times * esz + (2 * T - d) * esz + 2 * C * (nfac + nrhs) * 8 + 4) * B
    bwd = (2 * T * esz + 2 * T * esz + lam * esz + times * esz + (T - d) * esz + T * esz
           + ((T - d) if per_date else 1) * esz + 2 * C * nrhs * 8 + C * nfac * 8 + 4) * B
    return fwd, bwd


def bands_bytes(B: int, T: int, d: int, C: int, esz: int, per_date: bool, K: int = 8, irr: bool = False):
    """Shared-factor multi-band kernels (K = 8 row chunks): the factor warp reads w, lambda (, dates) in
    both sweeps once per pixel; each band reads its right-hand side twice and writes its outputs once."""
    Cc = math.ceil(T / K)
    nfac = d + d * (d - 1) // 2
    lam = 2 * (T - d) if per_date else 0  # (box overlaps come from L2)
    times = 2 * T if irr else 0
    shared = (2 * T + lam + times) * esz + Cc * nfac * 8 + 4
    fwd = (shared + Cc * nfac * 8 + C * (2 * T * esz + (2 * T - d) * esz + 2 * Cc * d * 8)) * B
    bwd = (shared + C * (2 * T * esz + (T - d) * esz + T * esz + 2 * Cc * d * 8)
           + ((T - d) if per_date else 1) * esz) * B
    return fwd, bwd


def load_profile_summary():
    """ncu figures of the dominant kernels from the committed profile summary (profiles/ncu_traffic.json):
    DRAM bytes per launch and fp64-pipe utilisation, labelled with their source (not measured in this run)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        return json.load(open(p))
    except Exception:
        return None


def profile_fields(kernel: str, workload: str | None = None) -> dict | None:
    """The committed ncu figures of a launch: '<workload>/<launch>' entries (NEXT-row workloads), else the
    headline's '<launch>' entries (hetero).  None if the profile has no entry for it."""
    prof = load_profile_summary() or {}
    key = f"{workload}/{kernel}" if workload else kernel
    k = prof.get(key)
    if not isinstance(k, dict):
        return None
    out = {"traffic": k.get("dram_bytes_per_launch"),
           "traffic_source": prof.get("workloads_source" if workload else "source")}
    if "fp64_pipe_pct" in k:
        out["fp64_pipe_pct"] = k["fp64_pipe_pct"]
    return out


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
    c = np.array([(-1) ** (d - j) * math.comb(d, j) for j in range(d + 1)], dtype=np.float64)
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


def cpu_baselines(x: dict, d: int, n_oracle: int = 0):
    """The CPU oracle (O1) timed on the host cores on a bounded sample of this workload, plus a conventional
    CPU banded solver for context."""
    cores = min(host_cores(), 32)
    n = n_oracle or 2 * cores
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
    return cpu, cpu_banded


# ----------------------------------------------------------------------------- reference arm
def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    import torch
    import synth
    cfg = synth.CONFIGS[args.config if args.config in synth.CONFIGS else "hetero"]
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
        "impl": "reference", "metric": METRICS.get(cfg.name, METRIC), "value": value, "unit": UNIT, "n_gpus": 0,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": statistics.median(walls) * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg.name, "B": cfg.B, "T": cfg.T, "d": cfg.d, "lambda": cfg.lam_mode,
                   "io": args.io, "sample_series_per_step": n},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": f"{n} series of the {cfg.name} workload per step, O1 dense fp64 + 2 long-double "
                                   f"refinement steps, fwd+bwd, {cores} processes"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- distributed plumbing check
def run_dist_check(args):
    """The multi-GPU code path without a measurement: init (NCCL with CUDA, gloo without), each rank draws
    its shard of a small workload keyed on global series ids, barrier, max over ranks, checksum gather;
    rank 0 redraws the whole job and checks every rank's checksum.  Prints one check line."""
    import torch
    import torch.distributed as dist
    import synth
    ws_n, rank, local = dist_env()
    cuda = torch.cuda.is_available()
    if ws_n > 1 or (args.dist_smoke and "RANK" in os.environ):
        if cuda:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    dev = torch.device("cuda", local) if cuda else torch.device("cpu")
    B, T = 256, 120
    strong = args.scaling == "strong"
    off, Bl = shard(rank, ws_n, B, strong)
    x = synth.make_inputs("hetero", B=Bl, T=T, series_offset=off, device=dev)
    cks = gather_checksums((x["y"], x["w"], x["lam"], x["g"]), ws_n)
    mx = max_over_ranks(float(rank), dev if cuda else None)
    ok = mx == ws_n - 1
    if rank == 0:
        Bjob = B if strong else ws_n * B
        full = synth.make_inputs("hetero", B=Bjob, T=T, device=dev)
        for r in range(ws_n):
            o, n = shard(r, ws_n, B, strong)
            part = [full[k][..., o:o + n].contiguous() for k in ("y", "w", "lam", "g")]
            ok = ok and cks["per_rank"][r] == local_checksums(part)
        print(json.dumps({"dist_check": bool(ok), "world_size": ws_n, "backend": dist.get_backend() if dist_is_init()
                          else None, "scaling": "strong" if strong else "weak", "checksums": cks}), flush=True)
    if dist_is_init():
        dist.barrier()
        dist.destroy_process_group()
    return 0 if ok else 1


# ----------------------------------------------------------------------------- libwhit arm
def base_line(args, metric, value, unit, ws_n, ms, launches, config, **kw):
    line = {"metric": metric, "value": value, "unit": unit, "n_gpus": ws_n, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong" if args.scaling == "strong" else "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "config": config, "gpu_launches": launches}
    line.update(kw)
    return line


def run_libwhit(args):
    import torch
    import torch.distributed as dist

    ws_n, rank, local = dist_env()
    if ws_n != args.gpus and rank == 0:
        print(f"note: --gpus {args.gpus} but WORLD_SIZE={ws_n}; running {ws_n} rank(s)", file=sys.stderr)
    if ws_n > 1 or (args.dist_smoke and "RANK" in os.environ):  # (--dist-smoke needs torchrun's env)
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local if ws_n > 1 else 0)
    torch.cuda.set_device(dev)
    distributed = dist.is_initialized()

    import paper_2604_00048_b200 as P
    import synth

    stream = torch.cuda.current_stream(dev)
    if args.config == "s2tile":
        rc = run_s2tile(args, P, synth, dev, stream, ws_n, rank)
    elif args.op == "table1":
        rc = run_table1(args, P, synth, dev, stream, ws_n, rank)
    elif args.op == "irregular":
        rc = run_irregular(args, P, synth, dev, stream, ws_n, rank)
    elif args.op in ("train", "variance"):
        rc = run_op(args, P, synth, dev, stream, ws_n, rank)
    else:
        rc = run_fwdbwd(args, P, synth, dev, stream, ws_n, rank)
    if distributed:
        dist.destroy_process_group()
    return rc


def run_fwdbwd(args, P, synth, dev, stream, ws_n, rank):
    """The headline: whit_forward + whit_backward (BASELINE metric) on the config's per-GPU batch."""
    import torch
    cfg = synth.CONFIGS[args.config]
    io = torch.float32 if args.io == "f32" else torch.float64
    esz = 4 if io == torch.float32 else 8
    B, T, d = cfg.B, cfg.T, cfg.d
    per_date = cfg.lam_mode == "per_date"
    fwd_only = not cfg.backward
    strong = args.scaling == "strong"
    B_job = B if strong else ws_n * B
    off, B = shard(rank, ws_n, B, strong)
    x = synth.make_inputs(cfg, B=B, series_offset=off, device=dev, dtype=io)
    y, w, lam, g = x["y"], x["w"], x["lam"], x["g"]
    wsp = P.Workspace(d, T, B, io, per_date, device=dev, stream=stream)
    z = torch.empty_like(y)
    gy = torch.empty_like(y)
    gl = torch.empty_like(lam)

    launches = [("whit_forward", lambda: P.whit_forward(y, w, lam, d, T, B, z, wsp))]
    if not fwd_only:
        launches.append(("whit_backward", lambda: P.whit_backward(g, wsp, z, gy, gl)))
    ms_step, per, clocks = timed_steps(launches, args.steps, args.warmup, dev, stream)
    nfail = P.whit_failures(wsp)
    value = B_job / (ms_step / 1e3)

    # per-rank checksums of the outputs (exact: int64 sums of the bit patterns, order-independent), gathered
    # outside the timed region.  Under weak scaling rank r owns global series [r*B, (r+1)*B) at every N, so
    # rank r's checksum is the same at every world size (results are bitwise independent of placement).
    checksums = gather_checksums((z,) if fwd_only else (z, gy, gl), ws_n)
    checksums["tensors"] = "z" if fwd_only else "z, grad_y, grad_lambda"
    if args.checksum_ranges > 1 and ws_n == 1 and not strong:
        # the ranges ranks 1..R-1 of an N = R weak-scaling run own, solved here (untimed) for the bitwise check
        ranges = [checksums["per_rank"][0]]
        for r in range(1, args.checksum_ranges):
            xr = synth.make_inputs(cfg, B=B, series_offset=r * B, device=dev, dtype=io)
            wr = P.Workspace(d, T, B, io, per_date, device=dev, stream=stream)
            zr, gyr, glr = torch.empty_like(xr["y"]), torch.empty_like(xr["y"]), torch.empty_like(xr["lam"])
            P.whit_forward(xr["y"], xr["w"], xr["lam"], d, T, B, zr, wr)
            if not fwd_only:
                P.whit_backward(xr["g"], wr, zr, gyr, glr)
            torch.cuda.synchronize(dev)
            ranges.append(local_checksums((zr,) if fwd_only else (zr, gyr, glr)))
            del xr, wr, zr, gyr, glr
            torch.cuda.empty_cache()
        checksums["ranges_at_n1"] = ranges

    nbin, nwarps = P.whit_wbits_detected(wsp)  # warps of the last forward that read W as bits
    wdet = nbin == nwarps and nwarps > 0
    fb, bb, mf, mb = algorithmic_bytes(B, T, d, esz, per_date, wdet=wdet)
    if 0 < nbin < nwarps:  # mixed (hybrid launch: its twisted part reads the float W): weight the two models
        f1, b1, _, _ = algorithmic_bytes(B, T, d, esz, per_date, wdet=True)
        fr = nbin / nwarps
        fb, bb = fr * f1 + (1 - fr) * fb, fr * b1 + (1 - fr) * bb
    kb = {"whit_forward": fb} if fwd_only else {"whit_forward": fb, "whit_backward": bb}
    mins = {"whit_forward": mf} if fwd_only else {"whit_forward": mf, "whit_backward": mb}
    dom = max(per, key=per.get)
    roof = roofline(kb, per, ms_step, mins, traffic=profile_fields(dom) if args.config == "hetero" else None,
                    extra={"byte_model": "R-mode, binary-W bit plane detected in the forward" if wdet
                           else ("R-mode, %d of %d warps with W as bits (hybrid / twisted launch)" % (nbin, nwarps)
                                 if nbin else "R-mode, float W plane")})
    tw_groups = P.whit_twist_groups(wsp)

    # the same step with the binary W bit-packed by the caller (whit_forward_wbits), beside the headline
    wbits_line = None
    if args.config == "hetero" and not args.no_extras:
        bits = P.whit_pack_mask(w)
        lb = [("whit_forward_wbits", lambda: P.whit_forward_wbits(y, bits, lam, d, T, B, z, wsp)),
              ("whit_backward", lambda: P.whit_backward(g, wsp, z, gy, gl))]
        msb, perb, clkb = timed_steps(lb, args.steps, 3, dev, stream)
        fbb, bbb, _, _ = algorithmic_bytes(B, T, d, esz, per_date, wbits=True)
        wbits_line = {"value": B_job / (msb / 1e3), "unit": UNIT, "ms_per_step": msb,
                      "w_format": "uint32 bit planes [ceil(T/32)][B] (binary W, P:26), whit_forward_wbits",
                      "gpu_launches": 2 * args.steps, "clocks": clkb,
                      "roofline": roofline({"whit_forward_wbits": fbb, "whit_backward": bbb}, perb, msb)}
        del bits

    # end to end through the public API with host buffers (rank-local)
    e2e = None
    e2e_wbits = None
    if not args.no_e2e and not fwd_only:
        bits_h = P.whit_pack_mask(w).cpu() if (args.config == "hetero" and not args.no_extras) else None
        del wsp, z, gy, gl
        torch.cuda.empty_cache()
        cap = 65536 if ws_n > 1 else 0  # (N > 1: a per-rank sample of the shard, see run_e2e)
        e2e = run_e2e(P, x, d, T, B, io, stream, dev, args.e2e_steps, B_job=B_job, max_series=cap)
        if bits_h is not None:
            e2e_wbits = run_e2e(P, x, d, T, B, io, stream, dev, args.e2e_steps, wbits=bits_h, B_job=B_job,
                                max_series=cap)

    # CPU oracle baseline (rank 0, N = 1 only), and a conventional CPU banded solver for context
    cpu = cpu_banded = None
    if rank == 0 and ws_n == 1 and not args.no_cpu_baseline and not fwd_only:
        cpu, cpu_banded = cpu_baselines(x, d, args.cpu_sample)

    if rank == 0:
        config = {"workload": args.config, "B_per_gpu": B, "T": T, "d": d, "lambda": cfg.lam_mode,
                  "io": args.io, "global_batch": B_job, "parallelism": f"dp{ws_n}",
                  "l2": "inputs larger than L2 (each [T][B] plane %.2f GB vs 126 MB L2)" % (T * B * esz / 1e9),
                  "mask": ("Sentinel-2 revisit + seasonal clouds, 90-day trailing gap" if cfg.mask == "s2"
                           else "iid Bernoulli(0.7)"),
                  "step": "whit_forward" if fwd_only else "whit_forward + whit_backward",
                  "failed_series": nfail}
        line = base_line(args, METRICS[args.config], value, UNIT, ws_n, ms_step, len(launches) * args.steps, config,
                         roofline=roof, clocks=clocks, e2e=e2e, cpu_baseline=cpu, cpu_banded=cpu_banded,
                         w_bits=wbits_line, e2e_wbits=e2e_wbits, checksums=checksums)
        line["binary_w"] = {"warps_reading_bits": nbin, "warps": nwarps,
                            "how": "whit_forward detected W in {0, 1} per warp of 32 series (DESIGN §5)"}
        line["path"] = {"twisted_groups": tw_groups[0], "groups": tw_groups[1],
                        "how": "small batches: twisted factorisation; just past one wave: hybrid launch (DESIGN §5)"}
        # the paper's only benchmark of this path, with its hardware: context, not the target
        line["paper_context"] = ("Table 1 (P:151-170; Tesla V100 32 GB, plain PyTorch banded Cholesky, T=350 "
                                 "irregular dates, C=10 bands, order 2, batch 28,672): 0.14 s -> ~205 k pixels/s; "
                                 "scaled linearly to T=3,288 ~21.8 k pixel-series/s")
        print(json.dumps(line), flush=True)
    return 0


def run_op(args, P, synth, dev, stream, ws_n, rank):
    """NEXT-row measurements on the same workload: 'train' = whit_forward_mse (the paper's masked
    MSE on 20 % held-out dates) + whit_backward; 'variance' = whit_posterior_variance."""
    import torch
    cfg = synth.CONFIGS[args.config]
    io = torch.float32 if args.io == "f32" else torch.float64
    esz = 4 if io == torch.float32 else 8
    B, T, d = cfg.B, cfg.T, cfg.d
    per_date = cfg.lam_mode == "per_date"
    off, B = shard(rank, ws_n, B)
    x = synth.make_inputs(cfg, B=B, series_offset=off, device=dev, dtype=io)
    y, w, lam = x["y"], x["w"], x["lam"]
    wsp = P.Workspace(d, T, B, io, per_date, device=dev, stream=stream)
    if args.op == "train":
        gen = torch.Generator(device=dev).manual_seed(1)
        held = (torch.rand(w.shape, device=dev, generator=gen) < 0.2) & (w > 0)
        w = w.masked_fill(held, 0.0)
        lw = held.to(io)
        del held
        z, gz, gy = torch.empty_like(y), torch.empty_like(y), torch.empty_like(y)
        gl, loss = torch.empty_like(lam), torch.empty(B, dtype=io, device=dev)
        launches = [("whit_forward_mse", lambda: P.whit_forward_mse(y, w, lam, lw, d, T, B, z, gz, loss, wsp)),
                    ("whit_backward", lambda: P.whit_backward(gz, wsp, z, gy, gl))]
        metric = "training steps (fused masked-MSE fwd + bwd) series/s"
        kb = None  # after the timed steps: the byte model of the path that ran (binary W as bits or not)
    else:
        var = torch.empty_like(w)
        launches = [("whit_posterior_variance", lambda: P.whit_posterior_variance(w, lam, d, T, B, var, wsp))]
        kb = {"whit_posterior_variance": variance_bytes(B, T, d, esz, per_date)}
        metric = "posterior variance diag(Omega^-1) series/s"
    ms, per, clocks = timed_steps(launches, args.steps, args.warmup, dev, stream)
    if kb is None:
        nbin, nwarps = P.whit_wbits_detected(wsp)
        fb, bb, _, _ = algorithmic_bytes(B, T, d, esz, per_date, wdet=(nbin == nwarps and nwarps > 0))
        kb = {"whit_forward_mse": fb + loss_fwd_extra_bytes(B, T, esz), "whit_backward": bb}
    if rank == 0:
        print(json.dumps(base_line(
            args, metric, ws_n * B / (ms / 1e3), UNIT, ws_n, ms, len(launches) * args.steps,
            {"workload": args.config, "op": args.op, "B_per_gpu": B, "T": T, "d": d, "lambda": cfg.lam_mode,
             "io": args.io, "l2": "inputs larger than L2"},
            roofline=roofline(kb, per, ms, traffic=profile_fields(max(per, key=per.get), args.op)), clocks=clocks)),
            flush=True)
    return 0


def run_irregular(args, P, synth, dev, stream, ws_n, rank):
    """NEXT-2: T = 350 uneven per-series acquisition dates (Table 1's length), d = 2,
    per-date lambda; whit_forward_times + whit_backward over B series per GPU."""
    import torch
    io = torch.float32 if args.io == "f32" else torch.float64
    esz = 4 if io == torch.float32 else 8
    T, d, B = 350, 2, synth.CONFIGS["hetero"].B
    off, B = shard(rank, ws_n, B)
    x = synth.make_inputs("hetero", B=B, T=T, d=d, series_offset=off, device=dev, dtype=io, mask="bernoulli")
    tt = synth.make_times(B, T, series_offset=off, device=dev, dtype=io)
    y, w, lam, g = x["y"], x["w"], x["lam"], x["g"]
    wsp = P.Workspace(d, T, B, io, True, device=dev, stream=stream, times=True)
    z, gy, gl = torch.empty_like(y), torch.empty_like(y), torch.empty_like(lam)
    launches = [("whit_forward_times", lambda: P.whit_forward_times(y, w, lam, tt, d, T, B, z, wsp)),
                ("whit_backward", lambda: P.whit_backward(g, wsp, z, gy, gl))]
    ms, per, clocks = timed_steps(launches, args.steps, args.warmup, dev, stream)
    fb, bb = irregular_bytes(B, T, d, esz, True)
    if rank == 0:
        print(json.dumps(base_line(
            args, "irregular-grid series fwd+bwd solves/s (T=350 acquisitions, d=2, per-date λ)",
            ws_n * B / (ms / 1e3), UNIT, ws_n, ms, 2 * args.steps,
            {"workload": "irregular", "B_per_gpu": B, "T": T, "d": d, "io": args.io,
             "times": "cumulative gaps U{1..12} days", "l2": "inputs larger than L2"},
            roofline=roofline({"whit_forward_times": fb, "whit_backward": bb}, per, ms,
                              traffic=profile_fields(max(per, key=per.get), "irregular")), clocks=clocks,
            paper_context="Table 1 (V100, PyTorch, T=350, C=10, order 2, batch 28672): 0.14 s "
                          "-> ~2.0 M band-series/s")), flush=True)
    return 0


def run_table1(args, P, synth, dev, stream, ws_n, rank):
    """The paper's Table 1 workload: C = 10 bands per pixel on T = 350 uneven
    acquisition dates, order d = 2, per-date lambda; whit_forward_times_bands + whit_backward_bands
    (one shared factor per pixel) over 262,144 pixels per GPU."""
    import torch
    io = torch.float32 if args.io == "f32" else torch.float64
    esz = 4 if io == torch.float32 else 8
    T, d, C, B = 350, 2, 10, 262144
    off, B = shard(rank, ws_n, B)
    x = synth.make_inputs_bands("hetero", C, B=B, T=T, d=d, series_offset=off, device=dev, dtype=io,
                                mask="bernoulli")
    tt = synth.make_times(B, T, series_offset=off, device=dev, dtype=io)
    y, w, lam, g = x["y"], x["w"], x["lam"], x["g"]
    wsp = P.Workspace(d, T, B, io, True, device=dev, stream=stream, C=C, times=True)
    z, gy, gl = torch.empty_like(y), torch.empty_like(y), torch.empty_like(lam)
    launches = [("whit_forward_times_bands", lambda: P.whit_forward_times_bands(y, w, lam, tt, d, T, B, C, z, wsp)),
                ("whit_backward_bands", lambda: P.whit_backward_bands(g, wsp, z, gy, gl))]
    ms, per, clocks = timed_steps(launches, args.steps, args.warmup, dev, stream)
    fb, bb = bands_bytes(B, T, d, C, esz, True, irr=True)
    if rank == 0:
        print(json.dumps(base_line(
            args, "band-series fwd+bwd solves/s (Table 1 workload: C=10 bands, T=350 uneven dates, d=2, per-date λ)",
            ws_n * B * C / (ms / 1e3), "band-series/s", ws_n, ms, 2 * args.steps,
            {"workload": "table1", "bands": C, "pixels_per_gpu": B, "T": T, "d": d, "io": args.io,
             "times": "cumulative gaps U{1..12} days", "l2": "inputs larger than L2"},
            roofline=roofline({"whit_forward_times_bands": fb, "whit_backward_bands": bb}, per, ms,
                              traffic=profile_fields(max(per, key=per.get), "table1")), clocks=clocks,
            pixels_per_s=ws_n * B / (ms / 1e3),
            paper_context="Table 1 (V100, PyTorch banded, T=350, C=10, order 2, batch 28672): "
                          "0.14 s -> ~2.0 M band-series/s")), flush=True)
    return 0


def run_s2tile(args, P, synth, dev, stream, ws_n, rank):
    """BASELINE configs[3]: Sentinel-2 tile chunk, 10 bands x 1,048,576 pixels, T = 3288, d = 2,
    per-date lambda per pixel, pixel-sharded over N GPUs, through the multi-band shared-factor path
    (whit_forward_bands / whit_backward_bands, NEXT-1).

    weak (default): each rank holds one 131,072-pixel chunk (the N = 8 share of the tile) resident.
    strong: the WHOLE tile is split over the ranks (rank r owns pixels [r*1M/N, (r+1)*1M/N)); a rank
    whose share exceeds one resident chunk processes it chunk by chunk -- each chunk's inputs drawn into
    HBM untimed, then its steps timed on the device -- and the tile time is the sum over its chunks
    (max over ranks)."""
    import torch
    C, d = 10, 2
    strong = args.scaling == "strong"
    esz = 4
    if strong:
        off0, Bp_rank = shard(rank, ws_n, S2TILE_PIXELS, strong=True)
    else:
        off0, Bp_rank = shard(rank, ws_n, S2TILE_CHUNK)
    chunks = [(o, min(S2TILE_CHUNK, off0 + Bp_rank - o)) for o in range(off0, off0 + Bp_rank, S2TILE_CHUNK)]
    total_ms, per_sum, clocks, nfail, last = 0.0, {}, None, 0, None
    T = synth.T_DAILY
    for ci, (off, Bp) in enumerate(chunks):
        x = synth.make_inputs_bands("hetero", C, B=Bp, series_offset=off, device=dev)
        y, w, lam, g = x["y"], x["w"], x["lam"], x["g"]
        T = y.shape[1]
        wsp = P.Workspace(d, T, Bp, torch.float32, True, device=dev, stream=stream, C=C)
        z, gy, gl = torch.empty_like(y), torch.empty_like(y), torch.empty_like(lam)
        launches = [("whit_forward_bands", lambda: P.whit_forward_bands(y, w, lam, d, T, Bp, C, z, wsp)),
                    ("whit_backward_bands", lambda: P.whit_backward_bands(g, wsp, z, gy, gl))]
        ms, per, ck = timed_steps(launches, args.steps, args.warmup if ci == 0 else 3, dev, stream,
                                  clocks=(ci == 0))
        clocks = clocks or ck
        total_ms += ms
        for k, v in per.items():
            per_sum[k] = per_sum.get(k, 0.0) + v
        nfail += P.whit_failures(wsp)
        if ci == len(chunks) - 1:
            last = (x, wsp, z, gy, gl)
        else:
            del x, y, w, lam, g, wsp, z, gy, gl
            torch.cuda.empty_cache()
    px_job = S2TILE_PIXELS if strong else ws_n * S2TILE_CHUNK
    fb, bb = bands_bytes(Bp_rank, T, d, C, esz, True)
    roof = roofline({"whit_forward_bands": fb, "whit_backward_bands": bb}, per_sum, total_ms,
                    traffic=profile_fields(max(per_sum, key=per_sum.get), "s2tile") if not strong else None)
    # end to end from pinned HOST memory through whit_run_host_bands (pixel chunks streamed through the
    # shared-factor kernels, copies overlapped with compute), on the last resident chunk
    e2e = None
    x, wsp, z, gy, gl = last
    Bp = x["y"].shape[2]
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
               "steps": args.e2e_steps, "pixels_per_step_per_gpu": Bp,
               "api": "whit_run_host_bands (C-ABI, pinned host buffers, chunk 4096, 4 streams)"}
    if rank == 0:
        print(json.dumps(base_line(
            args, "band-series fwd+bwd solves/s (Sentinel-2 tile chunk, shared factor per pixel)",
            px_job * C / (total_ms / 1e3), "band-series/s", ws_n, total_ms, 2 * args.steps * len(chunks),
            {"workload": "s2tile", "bands": C, "tile_pixels": S2TILE_PIXELS, "pixels_per_gpu": Bp_rank,
             "job_pixels": px_job, "resident_chunk_pixels": S2TILE_CHUNK, "chunks_per_gpu": len(chunks),
             "T": T, "d": d, "lambda": "per_date", "io": "f32", "parallelism": f"dp{ws_n}",
             "l2": "inputs larger than L2", "failed_series": nfail,
             "timing": "sum over the rank's resident chunks of the device-timed steps, max over ranks"},
            pixels_per_s=px_job / (total_ms / 1e3), roofline=roof, clocks=clocks, e2e=e2e)), flush=True)
    return 0


def run_e2e(P, x, d, T, B, io, stream, dev, steps, chunk=8192, nbuf=6, wbits=None, B_job=None, max_series=0):
    """Same metric through the public C-ABI with pinned HOST buffers: whit_run_host streams the
    batch in series chunks (pitched 2-D H2D copies of y, w, lambda, g; whit_forward +
    whit_backward; D2H of z, grad_y, grad_lambda), copies overlapping kernels on nbuf streams.
    With ``wbits`` (host bit-packed W) the weights cross PCIe as bits (whit_run_host_wbits).
    max_series > 0: stream only the first max_series series of the rank's batch (N > 1: eight ranks share the
    host's memory and PCIe, so each pins a 65,536-series sample instead of its whole shard; the rate is
    per series either way, the pipeline being chunked)."""
    import torch
    Bs = min(B, max_series) if max_series else B
    cols = (lambda t: t[..., :Bs]) if Bs < B else (lambda t: t)
    keys = ("y", "lam", "g") if wbits is not None else ("y", "w", "lam", "g")
    h = {k: torch.empty(cols(x[k]).shape, dtype=io, pin_memory=True) for k in keys}
    for k in h:
        h[k].copy_(cols(x[k]))
    if wbits is not None:
        h["wbits"] = cols(wbits).contiguous().pin_memory()
    x = {k: cols(x[k]) for k in ("y", "lam")}
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
    if dist_is_init():
        import torch.distributed as dist
        dist.barrier()  # ranks share the host's memory and PCIe: start the timed region together
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        P.whit_run_host(h["y"], hw, h["lam"], h["g"], d, oz, oy, ol, chunk=chunk, nbuf=nbuf, dev_buf=buf,
                        stream=stream, wbits=bits)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    ms = max_over_ranks(e0.elapsed_time(e1) / steps, dev)
    series = ws_n * Bs if Bs < B else (B_job or ws_n * B)
    return {"value": series / (ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "series_per_step": series,
            "ms_per_step": ms, "steps": steps,
            "api": f"{'whit_run_host_wbits' if bits is not None else 'whit_run_host'} (C-ABI, pinned host buffers, "
                   f"chunk {chunk}, {nbuf} streams)"}


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    args = parse(argv)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(argv, args.gpus)
    args.warmup = max(args.warmup, 3)  # the timing rules need >= 3 warm-up steps; the line reports what ran
    if args.dist_check:
        return run_dist_check(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_libwhit(args)


if __name__ == "__main__":
    sys.exit(main())
