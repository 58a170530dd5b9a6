"""N = 2 latent (CFG) parallelism protocol on CPU over gloo (reading C23).

Each rank evaluates ONE classifier-free-guidance branch of every request (rank 0 the
conditional, rank 1 the unconditional pass) with the fp64 oracle, places its v at
offset rank * B*Ni*C of the exchange buffer exactly as dit_step's EPI_FINAL does
(vcfg + lp_rank * vcount), all-gathers over gloo (the ncclAllGather of dit_step), and
applies the guided Euler update.  Both ranks must end with identical latents equal to
the single-process CFG step of oracle/sd3_step.py -- i.e. the one all-gather per step
is the only exchange the split needs.
"""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, errq):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import dataclasses
        import synth
        from oracle import flux_step as O
        from oracle import sd3_step as S
        cfg = synth.SD3_TINY
        W = O.weights_to_f64(synth.make_weights_bf16(cfg))
        batch = synth.make_batch(cfg, 2, 4, 4, 8, cfg_scale=5.5)
        B, ni, C = batch.batch, batch.img_tokens, cfg.in_channels
        # this rank's branch only (rank 0: prompts, rank 1: negative prompts)
        mine = dataclasses.replace(batch, cfg_scale=None,
                                   txt=batch.txt if rank == 0 else batch.txt_neg,
                                   pooled=batch.pooled if rank == 0 else batch.pooled_neg)
        _, v_mine = S.dit_step(cfg, W, mine)
        buf = torch.zeros(world * B * ni * C, dtype=torch.float64)
        buf[rank * B * ni * C:(rank + 1) * B * ni * C] = torch.from_numpy(v_mine.reshape(-1))
        parts = list(buf.chunk(world))
        dist.all_gather(parts, parts[rank].clone())
        v_c, v_u = (p.numpy().reshape(B, ni, C) for p in parts)
        v = np.stack([S.cfg_combine(v_c[b], v_u[b], batch.cfg_scale[b]) for b in range(B)])
        x = batch.latents.astype(np.float64) + (batch.sigma_next.astype(np.float64) -
                                                batch.sigma.astype(np.float64))[:, None, None] * v
        x_ref, v_ref = S.dit_step(cfg, W, batch)
        np.testing.assert_array_equal(v, v_ref)
        np.testing.assert_array_equal(x, x_ref)
        # both ranks hold the same next latents (no scatter needed)
        other = torch.from_numpy(x.reshape(-1)).clone()
        dist.broadcast(other, src=0)
        np.testing.assert_array_equal(other.numpy(), x.reshape(-1))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        errq.put(f"rank {rank}: {e!r}")
        raise


def test_latent_parallel_world2_gloo():
    ctx = mp.get_context("spawn")
    errq = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, errq)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, errs
    assert all(p.exitcode == 0 for p in procs)
