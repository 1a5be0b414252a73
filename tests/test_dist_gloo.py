"""World-size-2 gloo tests of the N>1 path on CPU (no GPU needed).

The multi-GPU design: every rank evaluates a contiguous row
shard of the candidate space and the packed (score, canonical index) keys are
MIN-allreduced; the combine is exact, so every rank decodes the same move.
Here each rank evaluates its shard of canonical u-rows with the oracle
(test infrastructure), packs keys the way the ABI does, and MIN-allreduces
them over gloo; the result must equal the unsharded oracle key.  The shard
plan is the library's own (tga_shard_range), and the 128-byte NCCL unique id
travels through torch.distributed.broadcast_object_list as in bench.py.
"""
import os
import socket

import numpy as np
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


def _pack(score: int, idx: int) -> int:
    # signed int64 image that orders like the ABI's uint64 key (score << 32 | idx)
    return (int(score) << 32) | int(idx)


def _worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle as O
    import tga_gen as G
    from paper_2506_17357_b200 import tga as T
    # 1) unique-id broadcast (bench.py: obj = [uid if rank == 0 else None])
    obj = [bytes(range(128)) if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    assert obj[0] == bytes(range(128))
    # 2) sharded evaluation + exact MIN combine
    inst, sol = G.x_like(11, n=60, target_routes=5)
    orc = O.Oracle.from_instance(inst)
    Q = O.canonical_q(sol)
    lo, hi = T.shard_range(Q, rank, world)
    res = {}
    for v in range(O.N_VARIANTS):
        m = orc.best_move(sol, v, u_lo=lo, u_hi=hi)
        key = _pack(int(m.score), m.u * Q + m.v) if m.found else np.iinfo(np.int64).max
        t = torch.tensor([key], dtype=torch.int64)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        res[v] = int(t.item())
    # 3) max-over-ranks timing
    t = torch.tensor([float(rank + 1)])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    res["tmax"] = float(t.item())
    res["range"] = (lo, hi)
    out_q.put((rank, res))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_keys_allreduce_min_equals_unsharded(world):
    from paper_2506_17357_b200 import build
    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    import oracle as O
    import tga_gen as G
    inst, sol = G.x_like(11, n=60, target_routes=5)
    orc = O.Oracle.from_instance(inst)
    Q = O.canonical_q(sol)
    # shards are disjoint and cover [0, Q)
    ranges = sorted(results[r]["range"] for r in range(world))
    assert ranges[0][0] == 0 and ranges[-1][1] == Q
    assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
    for v in range(O.N_VARIANTS):
        m = orc.best_move(sol, v)
        exp = _pack(int(m.score), m.u * Q + m.v) if m.found else np.iinfo(np.int64).max
        assert results[0][v] == results[1][v] == exp, v
    assert results[0]["tmax"] == results[1]["tmax"] == float(world)
