"""Real multi-rank steps (P:190 sparse all-to-all and its reverse; P:200-226 rebalancing;
SURVEY §8(e) checks P11, P16, P17), one process per rank:

* ``transport="ipc"`` (always runs, one GPU): two processes share cuda:0; the exchanges are
  NEXT-3's peer-memory puts (CUDA IPC mappings, device barriers); the count matrix and the
  cost row either go through a gloo process group (sync_free=False) or are exchanged on the
  devices (gs_project_put_dev, gs_p2p_put_costs); Algorithm 1 runs on every rank from the
  whole row (gs_rebalance_row);
* ``transport="nccl"`` (runs where torch.cuda.device_count() >= 2, skipped otherwise): G
  ranks on G GPUs with NCCL communicators from gs_nccl_unique_id -- gs_exchange,
  gs_exchange_grads, gs_rebalance (NCCL cost all-gather), gs_halo_exchange (an L1 + D-SSIM
  step), gs_redistribute.

Each rank's rendered blocks (T, n_last) stitched over ranks are bit-identical to the
single-rank run on the same gid order (P11); the ranks' parameter gradients concatenated are
within the 1e-3 metric of the single-rank ones (P17); every rank computes the same next
division points, equal to Algorithm 1 on the single-rank run's WORK cost row (partition
invariant).  Scenes: C0, and 2 views of 4591x3436 over a 2M-Gaussian Rubble-shaped scene."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import oracle
import synth

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case(name):
    if name == "c0":
        sc = synth.scene_c0(5)
        cams = synth.cameras_c0()
        gt = synth.gt_image(5, cams[0])[None]
        return sc, cams, gt
    sc = synth.scene_rubble(2_000_000)
    pool = synth.cameras_rubble(64)
    cams = [pool[3], pool[11]]
    for k, c in enumerate(cams):
        c.image_id = k
    gt = np.stack([synth.gt_image(2, c) for c in cams])
    return sc, cams, gt


def _worker(transport, world, rank, port, case, q, sync_free=True):
    import torch.distributed as dist
    import paper_2406_18533_b200._lib as L
    from paper_2406_18533_b200.engine import GrendelTrainer
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dev_i = rank if transport == "nccl" else 0
        torch.cuda.set_device(dev_i)
        dev = torch.device("cuda", dev_i)
        if world > 1:
            dist.init_process_group("nccl" if transport == "nccl" else "gloo", rank=rank, world_size=world,
                                    **({"device_id": dev} if transport == "nccl" else {}))
        nid = None
        if transport == "nccl" and world > 1:
            obj = [L.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            nid = obj[0]
        sc, cams, gt = _case(case)
        lo, hi = sc.n * rank // world, sc.n * (rank + 1) // world
        sh = sc.slice(lo, hi)
        ctx = L.Context(dev_i, rank, world, nid)
        p = L.GaussianParams.from_arrays(sh.pos, sh.log_scale, sh.rot, sh.opac_logit, sh.sh, dev, lo)
        W, H = cams[0].width, cams[0].height
        exch = "p2p" if transport == "ipc" and world > 1 else "nccl"
        tr = GrendelTrainer(ctx, p, W, H, len(cams), len(cams), cost_mode=L.COST_WORK, rebalance=True,
                            exchange=exch, count_gather="torch" if transport == "ipc" else "nccl",
                            sync_free=sync_free)
        gt_t = torch.from_numpy(gt).to(dev)
        loss = tr.step(cams, gt_t, next_cams=cams)
        torch.cuda.synchronize()
        if exch == "p2p":
            L.p2p_status(ctx)
        no = tr.last["n_owned"]
        out = dict(loss=float(loss.item()), T=tr.T.t[:no].cpu().numpy(), nl=tr.nl.t[:no].cpu().numpy(),
                   cost=tr.cost.t[:no].cpu().numpy(), dp_next=np.asarray(tr.dp).copy(),
                   g=[t.cpu().numpy() for t in (tr.g.pos_op, tr.g.log_scale, tr.g.rot, tr.g.sh)])
        if transport == "nccl" and world > 1:
            # an L1 + D-SSIM step (the halo exchange) from the same parameters, and a redistribution
            p2 = L.GaussianParams.from_arrays(sh.pos, sh.log_scale, sh.rot, sh.opac_logit, sh.sh, dev, lo)
            tr2 = GrendelTrainer(ctx, p2, W, H, len(cams), len(cams), cost_mode=L.COST_WORK, rebalance=False,
                                 loss="ssim")
            out["ssim_loss"] = float(tr2.step(cams, gt_t).item())
            pn, mn, vn = L.redistribute(ctx, p2, p2.zeros_like(), p2.zeros_like(), seed=7)
            out["redist"] = np.sort(pn.pos_op.cpu().numpy()[:, 0])
        q.put((rank, out, None))
    except Exception as e:  # reported to the parent
        import traceback
        q.put((rank, None, traceback.format_exc()))
    finally:
        if world > 1:
            dist.destroy_process_group()


def _run(transport, world, case, sync_free=True):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(transport, world, r, port, case, q, sync_free)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        r, o, err = q.get(timeout=600)
        assert err is None, err
        out[r] = o
    for p in procs:
        p.join(timeout=60)
    return [out[r] for r in range(world)]


def _check(one, many, G):
    # P11: stitched blocks bit-identical to the single-rank run (uniform DP of the first step)
    np.testing.assert_array_equal(np.concatenate([m["T"] for m in many]).view(np.uint32),
                                  one["T"].view(np.uint32))
    np.testing.assert_array_equal(np.concatenate([m["nl"] for m in many]), one["nl"])
    np.testing.assert_array_equal(np.concatenate([m["cost"] for m in many]), one["cost"])  # WORK: invariant
    assert abs(sum(m["loss"] for m in many) - one["loss"]) <= 1e-6 * abs(one["loss"])
    # P17: parameter gradients (shards concatenated) against the single-rank run -- two GPU
    # runs, so the difference is the fp32 atomic summation order: l2 within 1e-3, the max norm
    # within 3e-3 (DESIGN.md §9 "GPU against GPU": the single-rank run against itself already
    # differs by 5.7e-4 of the group maximum in the scale and rotation groups of this crop)
    for k in range(4):
        got = np.concatenate([m["g"][k] for m in many], axis=-2)
        want = one["g"][k]
        d = got - want
        assert np.abs(d).max() <= 3e-3 * np.abs(want).max() + 1e-30, (k, np.abs(d).max() / np.abs(want).max())
        assert np.linalg.norm(d) <= 1e-3 * np.linalg.norm(want) + 1e-30, (k, np.linalg.norm(d) / np.linalg.norm(want))
    # A9: identical next division points on every rank = Algorithm 1 on the WORK row
    want_dp = oracle.division_points(one["cost"], G)
    for m in many:
        np.testing.assert_array_equal(m["dp_next"], want_dp)


@pytest.mark.parametrize("case,sync_free", [("c0", False), ("c0", True), ("c2crop", True)])
def test_two_processes_ipc_match_single_rank(case, sync_free):
    one = _run("ipc", 1, case)[0]
    two = _run("ipc", 2, case, sync_free)
    _check(one, two, 2)


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs (NCCL ranks need one GPU each)")
@pytest.mark.parametrize("case", ["c0", "c2crop"])
def test_nccl_ranks_match_single_rank(case):
    G = min(torch.cuda.device_count(), 4)
    one = _run("nccl", 1, case)[0]
    many = _run("nccl", G, case)
    _check(one, many, G)
    # the D-SSIM loss with halos equals the single-rank loss; redistribution moves every
    # Gaussian exactly once
    one_ssim = _run_ssim_single(case)
    assert abs(sum(m["ssim_loss"] for m in many) - one_ssim) <= 1e-5 * abs(one_ssim)
    got = np.sort(np.concatenate([m["redist"] for m in many]))
    sc, _, _ = _case(case)
    np.testing.assert_array_equal(got, np.sort(sc.pos[:, 0].astype(np.float32)))


def _run_ssim_single(case):
    import paper_2406_18533_b200._lib as L
    from paper_2406_18533_b200.engine import GrendelTrainer
    sc, cams, gt = _case(case)
    p = L.GaussianParams.from_arrays(sc.pos, sc.log_scale, sc.rot, sc.opac_logit, sc.sh, "cuda:0")
    tr = GrendelTrainer(L.Context(0, 0, 1), p, cams[0].width, cams[0].height, len(cams), len(cams),
                        cost_mode=L.COST_WORK, rebalance=False, loss="ssim")
    return float(tr.step(cams, torch.from_numpy(gt).cuda()).item())
