"""World-size-2 gloo tests of the host-side multi-rank logic on CPU (no GPU here):
the exchange plan (libgs host function gs_exchange_plan) driven by an all-gathered count
matrix, the sparse exchange it implies (payload moved by gloo point-to-point), identical
division points on every rank from all-gathered per-block costs (libgs gs_division_points),
and the NEXT-3 peer-memory plan (gs_p2p_offsets: put offsets and gradient return offsets).
Expected values come from the oracle (whole-scene exchange sets and Algorithm 1)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, dp, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2406_18533_b200._lib as L
        sc = synth.scene_c0(4)
        cam = synth.cameras_c0()[0]
        lo, hi = sc.n * rank // world, sc.n * (rank + 1) // world
        shard = sc.slice(lo, hi)
        mb = oracle.membership(shard, cam)
        mask = oracle.exchange_sets(mb["vis"], mb["rect"], 0, 4, 4, dp)
        send_lists = [lo + np.nonzero(mask >> g & 1)[0] for g in range(world)]
        counts = torch.tensor([len(x) for x in send_lists], dtype=torch.int64)
        mat = [torch.zeros(world, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(mat, counts)
        mat = torch.stack(mat).numpy()
        soff, roff = L.exchange_plan(mat, world, rank)
        payload = torch.from_numpy(np.concatenate(send_lists).astype(np.int64))
        recv = torch.zeros(int(roff[-1]), dtype=torch.int64)
        reqs = []
        for g in range(world):
            if g == rank:
                recv[roff[g]:roff[g + 1]] = payload[soff[g]:soff[g + 1]]
                continue
            if soff[g + 1] > soff[g]:
                reqs.append(dist.isend(payload[soff[g]:soff[g + 1]].contiguous(), g))
            if roff[g + 1] > roff[g]:
                buf = torch.zeros(int(roff[g + 1] - roff[g]), dtype=torch.int64)
                reqs.append((dist.irecv(buf, g), g, buf))
        for r in reqs:
            if isinstance(r, tuple):
                r[0].wait()
                recv[roff[r[1]]:roff[r[1] + 1]] = r[2]
            else:
                r.wait()
        # per-block costs of the owned blocks -> all-gather -> Algorithm 1 on every rank
        B = 16
        rng = np.random.default_rng(9)
        cost = rng.integers(0, 5000, B)
        own = torch.from_numpy(cost[dp[rank]:dp[rank + 1]].astype(np.int64))
        sizes = [int(dp[g + 1] - dp[g]) for g in range(world)]
        parts = [torch.zeros(s, dtype=torch.int64) for s in sizes]
        dist.all_gather(parts, own) if len(set(sizes)) == 1 else [
            dist.broadcast(parts[g], g) if g != rank else dist.broadcast(own, g) for g in range(world)]
        if len(set(sizes)) != 1:
            parts[rank] = own
        row = torch.cat(parts).numpy()
        out_q.put((rank, recv.numpy(), L.division_points(row, world), mat))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("dp", [[0, 8, 16], [0, 5, 16]])
def test_two_rank_exchange_and_dp(dp):
    dp = np.array(dp, np.int64)
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, dp, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, recv, dpn, mat = q.get(timeout=120)
        res[r] = (recv, dpn, mat)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sc = synth.scene_c0(4)
    mb = oracle.membership(sc, synth.cameras_c0()[0])
    mask = oracle.exchange_sets(mb["vis"], mb["rect"], 0, 4, 4, dp)
    rng = np.random.default_rng(9)
    cost = rng.integers(0, 5000, 16)
    for r in range(world):
        want = np.nonzero(mask >> r & 1)[0]
        np.testing.assert_array_equal(res[r][0], want)  # ascending source rank == gid order
        np.testing.assert_array_equal(res[r][1], oracle.division_points(cost, world))
    np.testing.assert_array_equal(res[0][2], res[1][2])


def _p2p_worker(rank, world, port, dp, out_q):
    """NEXT-3 plan across processes: each rank 'puts' its buckets at the destination offsets
    gs_p2p_offsets gives (transport emulated by gloo with the offset carried along), receivers
    return a per-record value to the owner offsets; owners must get back exactly what they sent."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2406_18533_b200._lib as L
        sc = synth.scene_c0(5)
        cam = synth.cameras_c0()[0]
        lo, hi = sc.n * rank // world, sc.n * (rank + 1) // world
        mb = oracle.membership(sc.slice(lo, hi), cam)
        mask = oracle.exchange_sets(mb["vis"], mb["rect"], 0, 4, 4, dp)
        send_lists = [lo + np.nonzero(mask >> g & 1)[0] for g in range(world)]
        counts = torch.tensor([len(x) for x in send_lists], dtype=torch.int64)
        mat = [torch.zeros(world, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(mat, counts)
        C = torch.stack(mat).numpy()
        seg, put, soff, own = L.p2p_offsets(C, world, rank)
        # forward "put": (offset in destination buffer, payload) to every destination
        recv = np.full(int(seg[-1]), -1, np.int64)
        for d in range(world):  # one collective round per destination d
            msg = [int(put[d]), send_lists[d].tolist()]
            got = [None] * world
            dist.all_gather_object(got, msg)
            if d == rank:
                for m in got:
                    recv[m[0]:m[0] + len(m[1])] = m[1]
        # reverse: the value of record j (its gid * 10 + rank) goes to owner s at own[s] + (j - seg[s])
        back = []
        for s in range(world):
            back.append((s, int(own[s]), (recv[seg[s]:seg[s + 1]] * 10 + rank).tolist()))
        allback = [None] * world
        dist.all_gather_object(allback, back)
        dsend = np.full(int(soff[-1]), -1, np.int64)
        for lst in allback:
            for s, o, vals in lst:
                if s == rank:
                    dsend[o:o + len(vals)] = vals
        out_q.put((rank, recv, dsend, np.concatenate(send_lists), soff))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("dp", [[0, 8, 16], [0, 3, 16]])
def test_two_rank_p2p_plan(dp):
    dp = np.array(dp, np.int64)
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_p2p_worker, args=(r, world, port, dp, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, recv, dsend, sent, soff = q.get(timeout=120)
        res[r] = (recv, dsend, sent, soff)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sc = synth.scene_c0(5)
    mb = oracle.membership(sc, synth.cameras_c0()[0])
    mask = oracle.exchange_sets(mb["vis"], mb["rect"], 0, 4, 4, dp)
    for r in range(world):
        np.testing.assert_array_equal(res[r][0], np.nonzero(mask >> r & 1)[0])  # = the NCCL path's order
        recv_dst = np.concatenate([np.full(int(res[r][3][d + 1] - res[r][3][d]), d) for d in range(world)])
        np.testing.assert_array_equal(res[r][1], res[r][2] * 10 + recv_dst)  # every gradient back home
