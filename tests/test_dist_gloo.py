"""Multi-process (world size 2, gloo, CPU) coverage of the bench's multi-GPU host logic:
weak-scaling shards, max-over-ranks timing, and rank-independence of each series' inputs
(inputs keyed on the global series id, so per-series results cannot depend on N)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    import synth
    off, B = bench.shard(rank, world, 64)
    # max over ranks of a per-rank "step time"
    mx = bench.max_over_ranks(1.5 + rank)
    # this rank's shard of the hetero workload (short T to keep it quick)
    x = synth.make_inputs("hetero", B=B, T=80, series_offset=off)
    gathered = [None] * world
    dist.all_gather_object(gathered, (off, B, {k: x[k].clone() for k in ("y", "w", "lam", "g")}))
    cks = bench.gather_checksums((x["y"], x["lam"]), world)
    if rank == 0:
        # numpy copies through the queue: a torch tensor would travel as a shared-memory handle that the
        # parent may only open after this process has exited (and the segment with it)
        q.put((mx, [(o, n, {k: v.numpy().copy() for k, v in t.items()}) for o, n, t in gathered], cks))
    dist.barrier()
    dist.destroy_process_group()


def test_world2_shards_timing_and_rank_independent_inputs():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    mx, gathered, cks = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert mx == 2.5
    (o0, b0, x0), (o1, b1, x1) = [(o, n, {k: torch.from_numpy(v) for k, v in t.items()}) for o, n, t in gathered]
    assert (o0, b0, o1, b1) == (0, 64, 64, 64)  # contiguous, disjoint, covering [0, 128)
    import synth
    full = synth.make_inputs("hetero", B=128, T=80)
    for k in ("y", "w", "lam", "g"):
        assert torch.equal(torch.cat([x0[k], x1[k]], dim=-1), full[k]), k
    # gathered checksums: one row per rank, each the exact bit-pattern sum of that rank's shard
    import bench
    assert len(cks["per_rank"]) == 2
    for r, xr in enumerate((x0, x1)):
        assert cks["per_rank"][r] == bench.gather_checksums((xr["y"], xr["lam"]), 1)["per_rank"][0]
    # order-independent: the sum over both shards equals the checksum of the full batch
    tot = bench.gather_checksums((full["y"], full["lam"]), 1)["per_rank"][0]
    assert [a + b for a, b in zip(*cks["per_rank"])] == tot


def test_strong_scaling_shards_cover_the_job():
    """--scaling strong: contiguous ranges of multiples of 4 series covering [0, B) exactly once."""
    import bench
    for B, world in ((262144, 8), (65536, 3), (1000, 4), (4100, 2)):
        parts = [bench.shard(r, world, B, strong=True) for r in range(world)]
        assert parts[0][0] == 0 and sum(n for _, n in parts) == B
        for (o0, n0), (o1, _) in zip(parts, parts[1:]):
            assert o0 + n0 == o1 and n0 % 4 == 0


def test_max_over_ranks_without_group_is_identity():
    import bench
    assert bench.max_over_ranks(3.25) == 3.25


def _bench(*args, timeout=600):
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR",
                                                            "MASTER_PORT")}
    env["CUDA_VISIBLE_DEVICES"] = ""  # CPU host: the plumbing runs over gloo
    return subprocess.run([sys.executable, "bench.py", *args], cwd=root, capture_output=True, text=True,
                          timeout=timeout, env=env)


def _json_lines(out):
    import json
    return [json.loads(l) for l in out.stdout.splitlines() if l.strip().startswith("{")]


@pytest.mark.parametrize("scaling", ["weak", "strong"])
def test_bench_self_launch_world2_dist_check(scaling):
    """`python bench.py --gpus 2` outside torchrun re-launches itself under torch.distributed.run with two
    ranks -- the code path a SCALE run takes -- and the multi-process plumbing (rank-keyed shards,
    barrier, max over ranks, checksum gather) checks out over gloo: one line, from rank 0."""
    out = _bench("--gpus", "2", "--dist-check", "--scaling", scaling)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = _json_lines(out)
    assert len(lines) == 1, out.stdout
    d = lines[0]
    assert d["dist_check"] is True and d["world_size"] == 2 and d["backend"] == "gloo"
    assert d["scaling"] == scaling and len(d["checksums"]["per_rank"]) == 2


def test_bench_self_launch_world2_reference_arm():
    """--impl reference under the self-launch at N = 2: rank 0 alone times the oracle and prints one line."""
    out = _bench("--gpus", "2", "--impl", "reference", "--steps", "1", "--warmup", "1", "--cpu-sample", "2",
                 "--config", "toy")
    assert out.returncode == 0, out.stderr[-3000:]
    lines = _json_lines(out)
    assert len(lines) == 1 and lines[0]["impl"] == "reference" and lines[0]["value"] > 0
