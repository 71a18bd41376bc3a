"""Multi-process (gloo, world_size 2) coverage of the env-sharding host logic:
disjoint reproducible shards, per-gid initial states / actions, and the one
all_reduce per measurement window."""
import os
import sys

import numpy as np
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, out_dir):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    import bench
    from paper_2106_14405_b200.shard import layout_of, reduce_window, shard_env_ids

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    E = 6
    gids = shard_env_ids(rank, world, E)
    states = bench.idle_states(gids, bench.settled_pool())
    stats, times = reduce_window({"envs": E, "acc": float(rank + 1)}, {"ms": 10.0 * (rank + 1)})
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), gids=gids, layouts=layout_of(gids),
             states=np.stack([np.frombuffer(s, np.uint8) for s in states]),
             envs=stats["envs"], acc=stats["acc"], ms=times["ms"])
    dist.destroy_process_group()


def test_two_rank_sharding(tmp_path):
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    r0, r1 = (np.load(tmp_path / f"r{r}.npz") for r in (0, 1))
    assert set(r0["gids"]).isdisjoint(r1["gids"])
    assert sorted(np.concatenate([r0["gids"], r1["gids"]])) == list(range(12))
    assert float(r0["envs"]) == float(r1["envs"]) == 12.0
    assert float(r0["acc"]) == 3.0 and float(r0["ms"]) == float(r1["ms"]) == 20.0
    # a shard is a pure function of its global ids: rank 1's states equal a single-process rebuild
    sys.path.insert(0, ROOT)
    import bench

    solo = bench.idle_states(r1["gids"], bench.settled_pool())
    assert all(np.array_equal(np.frombuffer(a, np.uint8), b) for a, b in zip(solo, r1["states"]))
    assert (r1["layouts"] == r1["gids"] % 3).all()
