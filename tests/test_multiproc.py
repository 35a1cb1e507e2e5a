"""World-size-2 gloo run of the sharded benchmark's host logic on CPU:
disjoint sequence shards, barrier, max-over-ranks timing, rank-0 report."""

import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1708_06301_b200 import sharding
    r, w, local = sharding.world()
    seeds = sharding.rank_sequences(r, w, per_rank=4)
    sharding.barrier()
    elapsed = 10.0 + 5.0 * r          # rank 1 is slower
    ms = sharding.max_over_ranks(elapsed)
    gathered = [None] * w
    dist.all_gather_object(gathered, seeds)
    out[rank] = (seeds, ms, gathered, local)
    dist.destroy_process_group()


def test_two_rank_sharding_and_timing():
    world = 2
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    s0, ms0, all0, l0 = res[0]
    s1, ms1, all1, l1 = res[1]
    assert set(s0).isdisjoint(s1) and len(s0) == len(s1) == 4
    assert ms0 == ms1 == 15.0                 # max over ranks, identical everywhere
    assert all0 == all1 == [s0, s1]
    assert (l0, l1) == (0, 1)


def test_single_process_is_identity():
    from paper_1708_06301_b200 import sharding
    assert sharding.max_over_ranks(3.5) == 3.5
    assert sharding.rank_sequences(0, 1, 3, seed0=7) == [7, 8, 9]
    with pytest.raises(ValueError):
        sharding.rank_sequences(2, 2, 3)


def _bench_shard_worker(rank, world, port, out):
    """The bench's strong-scaling split (bench.py main): 64 sequences over
    `world` ranks, B = 64 / world each, global sequence indices."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1708_06301_b200 import scenes, sharding
    B = 64 // world
    seqs = sharding.rank_sequences(rank, world, B, seed0=0)
    specs = [scenes.config_sequence(5, s, n_frames=2) for s in seqs]
    ms = sharding.max_over_ranks(10.0 + rank)
    out[rank] = (seqs, [sp.texture_seed for sp in specs], ms)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_bench_strong_scaling_shards_the_64_sequences(world):
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_bench_shard_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    allseq = sorted(s for r in range(world) for s in res[r][0])
    assert allseq == list(range(64))                       # every sequence exactly once
    assert all(len(res[r][0]) == 64 // world for r in range(world))
    seeds = [t for r in range(world) for t in res[r][1]]
    assert len(set(seeds)) == 64                            # distinct scenes per sequence
    assert {res[r][2] for r in range(world)} == {10.0 + world - 1}   # max over ranks


def test_bench_relaunches_itself_as_n_ranks(monkeypatch):
    """`python bench.py --gpus N` outside torchrun re-launches as N ranks
    through torch.distributed.run on 127.0.0.1 (bench.relaunch)."""
    import bench
    calls = []
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd: calls.append(cmd) or 0)
    assert bench.relaunch(["--gpus", "4", "--steps", "2"], 4) == 0
    cmd = calls[0]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--nnodes=1" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[-4:] == ["--gpus", "4", "--steps", "2"] and cmd[-5].endswith("bench.py")
