"""N>1 host logic on CPU (gloo, world_size 2): the bench's max-over-ranks
timing reduction and the rank-0-only reference arm under torchrun."""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    sys.path.insert(0, str(ROOT))
    import bench
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, bench.max_over_ranks(10.0 + 5.0 * rank, world, torch.device("cpu"))))
    finally:
        dist.destroy_process_group()


def test_max_over_ranks_gloo():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got == {0: 15.0, 1: 15.0}


def test_max_over_ranks_single():
    sys.path.insert(0, str(ROOT))
    import bench
    assert bench.max_over_ranks(3.5, 1, None) == 3.5


@pytest.mark.slow
def test_reference_arm_under_torchrun_prints_once():
    """`bench.py --impl reference` launched like the driver's N=2 run: rank 0
    times the CPU oracle and prints one JSON line, rank 1 exits 0 silently."""
    env = dict(os.environ, OPENBLAS_NUM_THREADS="1", PYTHONPATH=str(ROOT))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(ROOT / "bench.py"),
           "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "3", "--config", "C1",
           "--cpu-sample-n", "2048"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    rec = json.loads(lines[0])
    assert rec["impl"] == "reference" and rec["n_gpus"] == 2
    assert rec["e2e"]["h2d_bytes_per_step"] == 0 and rec["cpu_baseline"]["kind"] == "port"


# ---------------------------------------------------------------- sharded host logic

def test_shard_spec_geometry():
    """Shard ranges, local <-> global heap numbering and ownership
    (paper_1701_02324_b200/sharded.py ShardSpec) for P = 2, 4, 8."""
    sys.path.insert(0, str(ROOT))
    from paper_1701_02324_b200.sharded import ShardSpec
    from paper_1701_02324_b200.tree import node_ranges
    n, depth = 1000, 4
    beg, end = node_ranges(n, depth)
    for world in (2, 4, 8):
        p = world.bit_length() - 1
        covered = []
        for rank in range(world):
            sp = ShardSpec(n, depth, world, rank)
            assert sp.root == (1 << p) - 1 + rank and sp.local_depth == depth - p
            covered.append((sp.begin, sp.end))
            lb, le = node_ranges(sp.size, sp.local_depth)
            for j in range((1 << (sp.local_depth + 1)) - 1):
                i = sp.global_node(j)
                assert sp.local_node(i) == j and sp.owner(i) == rank
                assert (beg[i] - sp.begin, end[i] - sp.begin) == (lb[j], le[j])
        assert covered[0][0] == 0 and covered[-1][1] == n
        assert all(covered[q][1] == covered[q + 1][0] for q in range(world - 1))
        assert ShardSpec(n, depth, world, 0).owner(0) is None
    for bad in (1, 3, 6):
        with pytest.raises(ValueError):
            ShardSpec(n, depth, bad, 0)
    with pytest.raises(ValueError):
        ShardSpec(n, 1, 4, 0)  # 4 shards need depth >= 2


def _shard_comm_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    sys.path.insert(0, str(ROOT))
    from paper_1701_02324_b200.sharded import ShardComm, or_reduce_bitmaps, sum_in_rank_order
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = ShardComm()
        inp = torch.arange(3, dtype=torch.float64) + 10 * rank
        out = torch.empty(3 * world, dtype=torch.float64)
        comm.all_gather(out, inp)
        bm = torch.tensor([1 << rank, 0, 1 << (rank + 4)], dtype=torch.int32)
        allbm = torch.empty(3 * world, dtype=torch.int32)
        comm.all_gather(allbm, bm)
        orb = or_reduce_bitmaps(allbm, world)
        s = torch.tensor([1.0 + rank])
        comm.all_reduce_sum_(s)
        part = torch.tensor([0.1, 1e16, -1e16] if rank == 0 else [0.2, 1.0, 3.0], dtype=torch.float64)
        ro = sum_in_rank_order(comm, part)  # the sharded KRR predict's reduction
        q.put((rank, out.tolist(), orb.tolist(), comm.all_reduce_max(rank * 7), float(s.item()), ro.tolist()))
    finally:
        dist.destroy_process_group()


def test_shard_comm_gloo():
    """The sharded path's collectives (all-gather into the top plan's
    layout, bitmap OR, error-flag max, GMRES sums) over gloo, world 2."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_comm_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = {r: rest for r, *rest in (q.get(timeout=120) for _ in procs)}
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(2):
        out, orb, mx, sm, ro = got[r]
        assert ro == [0.1 + 0.2, 1e16 + 1.0, -1e16 + 3.0]  # (p0 + p1) bits on every rank
        assert out == [0.0, 1.0, 2.0, 10.0, 11.0, 12.0]
        assert orb == [3, 0, (1 << 4) | (1 << 5)]
        assert mx == 7 and sm == 3.0


def _agree_worker(rank, world, port, q):
    import torch.distributed as dist
    sys.path.insert(0, str(ROOT))
    from paper_1701_02324_b200.sharded import ShardComm, agree_on_failure
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = ShardComm()
        agree_on_failure(comm, None, "never")  # nobody failed: returns on every rank
        err = RuntimeError("skeletonization failed at node 9 (level 3)") if rank == 1 else None
        try:
            agree_on_failure(comm, err, "skeletonization failed on rank {rank}")
            q.put((rank, "no error"))
        except RuntimeError as exc:
            q.put((rank, str(exc)))
    finally:
        dist.destroy_process_group()


def test_sharded_failure_agreement_gloo():
    """A shard-level failure on one rank raises on every rank before the
    next collective (sharded.build_skeletons_sharded): the
    failing rank with its own message, the others naming it."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_agree_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got == {0: "skeletonization failed on rank 1", 1: "skeletonization failed at node 9 (level 3)"}
