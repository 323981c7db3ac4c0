"""NEXT-3 across processes: two processes on cuda:0 run one training step with
exchange='p2p' -- symmetric buffers exported as CUDA IPC handles, opened by the peer
(gs_ipc_open), records put into the peer's receive buffer and gradients reduced into the
owner's buffer through the mapping, device-side barriers -- and their parameter gradients
must equal the single-rank step's (record gradients summed in another float order: the
1e-3 metric of SURVEY #31).  On one GPU the two processes' kernels time-slice, so the
barrier spins until the peer's context is scheduled (bounded: a timeout fails the test)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import synth

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _grads(world, rank, port, q):
    import torch.distributed as dist
    import paper_2406_18533_b200._lib as L
    from paper_2406_18533_b200.engine import GrendelTrainer
    try:
        if world > 1:
            os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
            dist.init_process_group("gloo", rank=rank, world_size=world)
        sc = synth.scene_c0(3)
        cams = synth.cameras_c0()
        gt = torch.from_numpy(synth.gt_image(3, cams[0])[None]).cuda()
        lo, hi = sc.n * rank // world, sc.n * (rank + 1) // world
        sh = sc.slice(lo, hi)
        ctx = L.Context(0, rank, world)  # no NCCL communicator: both ranks share cuda:0
        p = L.GaussianParams.from_arrays(sh.pos, sh.log_scale, sh.rot, sh.opac_logit, sh.sh, "cuda:0", lo)
        tr = GrendelTrainer(ctx, p, 64, 64, 1, 1, cost_mode=L.COST_WORK, rebalance=False,
                            exchange="p2p" if world > 1 else "nccl", count_gather="torch")
        loss = tr.step(cams, gt)
        torch.cuda.synchronize()
        if world > 1:
            L.p2p_status(ctx)
        g = [t.cpu().numpy() for t in (tr.g.pos_op, tr.g.log_scale, tr.g.rot, tr.g.sh)]
        q.put((rank, float(loss.item()), g, None))
    except Exception as e:  # reported to the parent
        q.put((rank, None, None, repr(e)))
    finally:
        if world > 1:
            dist.destroy_process_group()


def _run(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_grads, args=(world, r, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        r, loss, g, err = q.get(timeout=300)
        assert err is None, err
        out[r] = (loss, g)
    for p in procs:
        p.join(timeout=60)
    return out


def test_two_process_p2p_step_equals_single_rank():
    one = _run(1)[0]
    two = _run(2)
    assert abs(two[0][0] + two[1][0] - one[0]) <= 1e-6 * abs(one[0])  # loss partials sum to the whole
    for k in range(4):  # parameter-gradient planes, shards concatenated
        got = np.concatenate([two[0][1][k], two[1][1][k]], axis=-2)
        want = one[1][k]
        err = np.abs(got - want)
        assert err.max() <= 1e-3 * np.abs(want).max() + 1e-30, (k, err.max(), np.abs(want).max())
