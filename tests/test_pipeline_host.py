"""CPU: the multi-GPU host logic of the SWARM pipeline — placement, replicated
routing plans, and point-to-point ordering — including a world_size-2 gloo run
that checks every rank derives the same routes without exchanging them."""
import os

import pytest
import torch.multiprocessing as mp


def _placements():
    from paper_2301_11913_b200.swarm import Placement
    return {w: Placement(w, 4) for w in (1, 2, 4, 8)}


def test_placement_protocol():
    pls = _placements()
    assert pls[1].local_stages(0) == [0, 1, 2, 3]
    assert [pls[2].local_stages(r) for r in range(2)] == [[0, 1], [2, 3]]
    assert [pls[4].local_stages(r) for r in range(4)] == [[0], [1], [2], [3]]
    assert [pls[8].local_stages(r) for r in range(8)] == [[0], [0], [1], [1], [2], [2], [3], [3]]
    assert pls[8].P == 2 and [pls[8].rank_of_peer(p) for p in range(8)] == list(range(8))
    with pytest.raises(ValueError):
        from paper_2301_11913_b200.swarm import Placement
        Placement(3, 4)


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_routes_balanced_and_deterministic(world):
    from paper_2301_11913_b200.swarm import Placement, RoutePlanner
    pl = Placement(world, 4)
    a = RoutePlanner(pl, pl.P, 0.25).plan(32)
    b = RoutePlanner(pl, pl.P, 0.25).plan(32)
    assert a == b
    for s in range(4):
        counts = {}
        for r in a:
            assert pl.stage_of_peer(r[s]) == s
            counts[r[s]] = counts.get(r[s], 0) + 1
        assert set(counts.values()) == {32 // pl.P}  # IWRR spreads homogeneous peers evenly


@pytest.mark.parametrize("world", [2, 4, 8])
def test_p2p_orders_agree(world):
    """For every ordered rank pair, the sender's send sequence equals the
    receiver's receive sequence (NCCL p2p cannot deadlock on order)."""
    from paper_2301_11913_b200.swarm import Placement, RoutePlanner, message_log
    pl = Placement(world, 4)
    routes = RoutePlanner(pl, pl.P, 0.25).plan(16)
    logs = {r: message_log(pl, routes, r) for r in range(world)}
    total = 0
    for a in range(world):
        for b in range(world):
            sends = [(ph, mb) for op, peer, ph, mb in logs[a] if op == "send" and peer == b]
            recvs = [(ph, mb) for op, peer, ph, mb in logs[b] if op == "recv" and peer == a]
            assert sends == recvs, (a, b)
            total += len(sends)
    # forward: every microbatch crosses each inter-rank stage boundary once, same for backward
    boundaries = sum(1 for s in range(3) if pl.local_stages(0) != [] and
                     (world >= 4 or (s + 1) % pl.per_rank == 0))
    assert total == 2 * 16 * boundaries


def _gloo_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2301_11913_b200.swarm import Placement, RoutePlanner, visit_schedule
    pl = Placement(world * 4, 4)  # emulate an 8-GPU box's routing on 2 CPU ranks
    routes = RoutePlanner(pl, pl.P, 0.125).plan(24)
    gathered = [None] * world
    dist.all_gather_object(gathered, routes)
    sched = visit_schedule(Placement(world, 4), RoutePlanner(Placement(world, 4), 1, 0.125).plan(8), rank)
    ok = all(g == routes for g in gathered)
    q.put((rank, ok, sched))
    dist.destroy_process_group()


def test_replicated_routing_gloo():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict((r, (ok, sched)) for r, ok, sched in (q.get(timeout=120) for _ in procs))
    for p in procs:
        p.join(timeout=60)
    assert out[0][0] and out[1][0]
    # world 2: rank 0 runs stages 0-1, rank 1 stages 2-3 of every microbatch
    assert out[0][1] == [(mb, s) for mb in range(8) for s in (0, 1)]
    assert out[1][1] == [(mb, s) for mb in range(8) for s in (2, 3)]


def test_rebalance_moves_from_overprovisioned_stage():
    """Layout (3,1,2,2): the queue proxy makes stage 1 the max-load stage and
    Alg. 2 moves the lowest-id idle peer of stage 0 there; after the move the
    layout is (2,2,2,2) and the decision is a no-op."""
    from paper_2301_11913_b200.routing import decide
    from paper_2301_11913_b200.swarm import Placement, RoutePlanner, queue_proxy_table
    pl = Placement(8, 4, [3, 1, 2, 2])
    planner = RoutePlanner(pl, 2, 0.25)
    visits = [0] * 8
    for route in planner.plan(24):
        for p in route:
            visits[p] += 1
    assert visits == [8, 8, 8, 24, 12, 12, 12, 12]
    d = decide(queue_proxy_table(pl, visits))
    assert (d.mover, d.from_stage, d.to_stage) == (0, 0, 1)
    # migration: routers ban then re-add the mover on its new stage
    planner.ban(0)
    pl.stage_of[0] = 1
    planner.add(0, 1)
    visits = [0] * 8
    for route in planner.plan(24):
        for p in route:
            visits[p] += 1
    assert all(v == 12 for v in visits)
    d = decide(queue_proxy_table(pl, visits))
    assert d.mover is None


def test_peer_failure_reroutes():
    from paper_2301_11913_b200.swarm import Placement, RoutePlanner
    pl = Placement(8, 4)
    planner = RoutePlanner(pl, 2, 0.25)
    planner.remove(5)
    pl.alive.discard(5)
    routes = planner.plan(16)
    assert all(5 not in r for r in routes)
    assert sum(r[2] == 4 for r in routes) == 16  # stage 2 is down to peer 4
    assert pl.local_stages(5) == [] and pl.members(2) == [4]
