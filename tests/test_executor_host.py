"""Host logic of the engine-driven executor (paper_2301_11913_b200/executor.py),
no GPU: the point-to-point operations every rank derives from the shared engine
schedule must pair up (same keys in the same order for every ordered rank
pair, so NCCL matches them), every cross-rank visit input must arrive before
its consumer starts, and a world-size-2 gloo run must agree on the schedule."""
import os
import random

import pytest

from paper_2301_11913_b200.engine import HOP, START, Engine
from paper_2301_11913_b200.executor import hop_action, wire_key
from paper_2301_11913_b200.swarm import Placement


def schedule(world, S, tpp, seed, n=4000):
    from paper_2301_11913_b200.engine import EngineConfig
    pl = Placement(world, S)
    cfg = EngineConfig(n_stages=S, initial_peers=[[1.0] * pl.layout[s] for s in range(S)],
                       forward_service_seconds=1.0, trainers_per_peer=tpp, allreduce_period=20.0,
                       allreduce_stall=0.5, duration_seconds=1e9, bucket_seconds=1e8)
    e = Engine(cfg, seed)
    recs = []
    while len(recs) < n:
        recs += e.next(256)
    return pl, recs


@pytest.mark.parametrize("world,S,tpp,seed", [(1, 4, 1, 0), (2, 4, 2, 1), (4, 4, 1, 2), (8, 4, 1, 3),
                                              (8, 4, 3, 4), (4, 2, 2, 5), (2, 2, 1, 6), (6, 3, 2, 7)])
def test_p2p_ops_pair_up_and_precede_consumers(world, S, tpp, seed):
    """The executor's issue logic: at a HOP each rank notes its half of a
    cross-rank transfer (hop_action); both halves are issued at the consuming
    visit's START record.  Per ordered rank pair the send and receive sequences
    must be identical (NCCL matches them in order), every remote input must be
    received at its consumer's START, and every noted transfer must be issued."""
    pl, recs = schedule(world, S, tpp, seed)
    sends = {}   # (a, b) -> keys a sends to b, in a's issue order
    recvs = {}   # (a, b) -> keys b receives from a, in b's issue order
    xfer = {r: {} for r in range(world)}   # rank -> key -> its noted half
    remote = {}  # trainer -> did its latest hop cross ranks
    for r in recs:
        if r.kind == HOP:
            remote[r.trainer] = r.from_worker >= 0 and pl.rank_of_peer(r.from_worker) != pl.rank_of_peer(r.worker)
            for rank in range(world):
                act = hop_action(pl, S, r, rank)
                if act is not None:
                    assert act[2] not in xfer[rank], "a buffer's previous transfer was never issued"
                    xfer[rank][act[2]] = act
        elif r.kind == START:
            key = wire_key(S, r.trainer, r.stage, bool(r.backward))
            issued = set()
            for rank in range(world):
                if key is not None and key in xfer[rank]:
                    op, peer, k = xfer[rank].pop(key)
                    if op == "send":
                        sends.setdefault((rank, peer), []).append(k)
                    else:
                        recvs.setdefault((peer, rank), []).append(k)
                        issued.add(rank)
            if key is not None and remote.get(r.trainer):
                assert pl.rank_of_peer(r.worker) in issued, "remote input not received at its consumer's START"
    assert sends.keys() == recvs.keys()
    for pair in sends:
        assert sends[pair] == recvs[pair], pair
    if world >= 2 and S >= 2:
        assert sends, "expected cross-rank traffic"


def test_world1_has_no_transfers():
    pl, recs = schedule(1, 4, 2, 9)
    assert all(hop_action(pl, 4, r, 0) is None for r in recs if r.kind == HOP)


def _gloo_worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    _, recs = schedule(world, 2, 1, 11, n=500)
    import torch
    sig = torch.tensor([hash(tuple((r.kind, r.trainer, r.stage, r.worker, r.from_worker) for r in recs)) % (2 ** 61)],
                       dtype=torch.int64)
    allsig = [torch.zeros_like(sig) for _ in range(world)]
    dist.all_gather(allsig, sig)
    out.put((rank, [int(s) for s in allsig]))
    dist.destroy_process_group()


def test_gloo_ranks_agree_on_the_schedule():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = random.randint(20000, 40000)
    ps = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, sigs in res:
        assert len(set(sigs)) == 1
