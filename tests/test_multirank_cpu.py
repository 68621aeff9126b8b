"""Multi-rank allocator checks over torch.distributed gloo (world sizes 2, 4 and 8: the 1/2/4/8-GPU parity target),
the CPU stand-in for 1/2/4/8 GPUs:
 * tenant/batch sharding: every rank replays its own op log; rank 0 replays all
   logs in the oracle and checks every rank's state hash bit-exactly;
 * head sharding (TP): all ranks replay the same log; their state hashes agree."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, results):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from allocator_fuzz import make_log, replay_lib, replay_oracle, state_hash
    # tenant sharding: per-rank log
    _, st = replay_lib(make_log(1000 + rank, n_ops=150))
    hashes = [None] * world
    dist.all_gather_object(hashes, state_hash(st))
    ok_shard = True
    if rank == 0:
        for r in range(world):
            _, est = replay_oracle(make_log(1000 + r, n_ops=150))
            ok_shard &= state_hash(est) == hashes[r]
    # head sharding: identical logs -> identical tables on every rank
    _, st2 = replay_lib(make_log(7, n_ops=150))
    h2 = [None] * world
    dist.all_gather_object(h2, state_hash(st2))
    if rank == 0:
        results.put((ok_shard, len(set(h2)) == 1))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_gloo_ranks(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(180)
    assert all(p.exitcode == 0 for p in ps)
    ok_shard, ok_tp = q.get(timeout=10)
    assert ok_shard and ok_tp
