"""CPU tests of the multi-process ghost-exchange plan (the path that runs one
process per GPU over NCCL): world_size 2 and 4 over torch.distributed gloo.

Each process builds the host-only plan the device runtime uses, fills its
arena's owned slots from one global vector, runs the plan's pack ->
send/recv -> gather on the CPU (gloo stands in for NCCL) and checks that every
ghost slot then holds its owner's value -- the state the reference's
sync_all reaches (reference tests/test_communication.cpp:182-226)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1805_10167_b200 import hytegrid as H
from tests.helpers import keyed_uniform


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def emulate_sync(plan, arena, rank):
    """plan's pack -> blocks -> gather on host arrays (gloo as the transport)."""
    import torch
    send = arena[plan.array("pack_src")] if plan.npack else np.zeros(0)
    recv = np.zeros(plan.ntotal - plan.nlocal)
    reqs = []
    for src_rank, dst_rank, so, ro, cnt in plan.array("sends"):
        assert src_rank == rank
        reqs.append(dist.isend(torch.from_numpy(send[so:so + cnt].copy()), dst=int(dst_rank)))
    bufs = []
    for src_rank, dst_rank, so, ro, cnt in plan.array("recvs"):
        assert dst_rank == rank
        t = torch.zeros(int(cnt), dtype=torch.float64)
        reqs.append(dist.irecv(t, src=int(src_rank)))
        bufs.append((ro, cnt, t))
    for r in reqs:
        r.wait()
    for ro, cnt, t in bufs:
        recv[ro:ro + cnt] = t.numpy()
    dst, src = plan.array("gather_dst"), plan.array("gather_src")
    arena[dst[:plan.nlocal]] = arena[src]
    arena[dst[plan.nlocal:]] = recv


def _worker(rank, world, port, mesh, level, partitioner, out, kind=0):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        if partitioner == "greedy":
            assignment = H.partition_greedy_edgecut(mesh, world, max(level, 1))
        else:
            assignment = H.partition_round_robin(mesh, world)
        plan = H.ExchangePlan(mesh, world, assignment, [rank], level, kind)
        # a P2 level's owned set is P1's at level + 1 (plan indices use that numbering)
        glob = keyed_uniform(mesh, level + kind, seed=17)
        arena = np.full(plan.arena_size, np.nan)
        arena[plan.array("owned_slots")] = glob[plan.array("owned_global")]
        emulate_sync(plan, arena, rank)
        dst, owner = plan.array("gather_dst"), plan.array("owner_global")
        ok = bool(np.array_equal(arena[dst], glob[owner]))
        # every ghost of this process's primitives is covered exactly once
        ok &= len(np.unique(dst)) == dst.size
        # blocks are symmetric: what I receive from q, q sends to me
        counts = {(int(s), int(d)): int(c) for s, d, _, _, c in plan.array("sends")}
        counts.update({(int(s), int(d)): int(c) for s, d, _, _, c in plan.array("recvs")})
        gathered = [None] * world
        dist.all_gather_object(gathered, counts)
        for other in gathered:
            for key, c in other.items():
                for mine in gathered:
                    if key in mine:
                        ok &= mine[key] == c
        out[rank] = ok
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,partitioner,mesh_name,level", [
    (2, "greedy", "ring8", 3), (2, "greedy", "channel44", 4), (2, "greedy", "annulus", 3),
    (2, "rr", "ring8", 0), (2, "rr", "square_rev", 1), (4, "greedy", "channel44", 4), (4, "greedy", "annulus", 2),
    (3, "rr", "ring8", 2)])
def test_multiprocess_exchange_plan(world, partitioner, mesh_name, level):
    mesh = {"ring8": H.meshgen.square_ring8(), "channel44": H.meshgen.channel(4, 4),
            "annulus": H.meshgen.annulus(8, 2, 1.0, 2.0), "square_rev": H.meshgen.unit_square_reversed()}[mesh_name]
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    mp.start_processes(_worker, args=(world, _free_port(), mesh, level, partitioner, out), nprocs=world,
                       join=True, start_method="spawn")
    assert all(out[r] for r in range(world)), dict(out)


@pytest.mark.parametrize("world,mesh_name,level", [(2, "ring8", 2), (3, "annulus", 1), (2, "square_rev", 0),
                                                  (4, "channel44", 2)])
def test_multiprocess_exchange_plan_p2(world, mesh_name, level):
    """P2 plans (fine halo rows 1-2 per edge face, vertex ghosts per edge and face)
    over gloo: every ghost holds its owner's value afterwards, blocks symmetric"""
    mesh = {"ring8": H.meshgen.square_ring8(), "channel44": H.meshgen.channel(4, 4),
            "annulus": H.meshgen.annulus(8, 2, 1.0, 2.0), "square_rev": H.meshgen.unit_square_reversed()}[mesh_name]
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    mp.start_processes(_worker, args=(world, _free_port(), mesh, level, "rr", out, 1), nprocs=world,
                       join=True, start_method="spawn")
    assert all(out[r] for r in range(world)), dict(out)


@pytest.mark.parametrize("ranks", [1, 2, 3])
def test_single_process_plan_matches_owner_values(ranks):
    """All ranks co-resident in one process (the reference's model): local
    gathers + in-process blocks reproduce owner values."""
    mesh = H.meshgen.square_ring8()
    level = 3
    assignment = H.partition_round_robin(mesh, ranks)
    plan = H.ExchangePlan(mesh, ranks, assignment, list(range(ranks)), level)
    glob = keyed_uniform(mesh, level, seed=3)
    arena = np.full(plan.arena_size, np.nan)
    arena[plan.array("owned_slots")] = glob[plan.array("owned_global")]
    send = arena[plan.array("pack_src")]
    recv = np.zeros(plan.ntotal - plan.nlocal)
    for _, _, so, ro, cnt in plan.array("inproc"):
        recv[ro:ro + cnt] = send[so:so + cnt]
    dst, src = plan.array("gather_dst"), plan.array("gather_src")
    arena[dst[:plan.nlocal]] = arena[src]
    arena[dst[plan.nlocal:]] = recv
    assert np.array_equal(arena[dst], glob[plan.array("owner_global")])
    assert plan.n_sends == plan.n_recvs == 0
    if ranks == 1:
        assert plan.npack == 0 and plan.ntotal == plan.nlocal


def test_ghost_counts_match_reference_storage():
    """Per level: 3n face border ghosts per face, 2 + n per adjacent face per
    edge (line ends + halo row 1), one per incident edge per vertex."""
    mesh = H.meshgen.channel(3, 2, 2.0, 1.5)
    nv, ne, nf = H.mesh_counts(mesh)
    for level in range(0, 5):
        n = 1 << level
        plan = H.ExchangePlan(mesh, 1, np.zeros(nv + ne + nf, np.int32), [0], level)
        # sum over edges of adjacent faces = 3 nf; sum over vertices of incident edges = 2 ne
        expect = 3 * n * nf + 2 * ne + n * (3 * nf) + 2 * ne
        assert plan.ntotal == expect, (level, plan.ntotal, expect)
