"""Sequence and latent parallelism across PROCESSES (one GPU per call here, so two processes on
the same B200), through the real cross-process machinery: every rank's workspace exported as a
CUDA IPC handle (dit_peer_handle), the handles all-gathered over a gloo group (standing in for
the NCCL all-gather sp_init / lp_init do), peers mapped with cudaIpcOpenMemHandle
(sp_init_peers / lp_init_peers), and the fused exchanges' system-scope flag barriers
(fence.sys + st.release.sys / ld.acquire.sys) crossing the process boundary.

Ulysses SP (pin P10): 2 ranks, bitwise equal to the one-GPU step over two
consecutive steps (the flag epochs advance).  Latent parallelism (reading C23):
rank 0 the conditional, rank 1 the unconditional pass, v stored into the peer by the final
GEMM's epilogue; both ranks' latents equal the one-GPU CFG step bitwise over three steps (the
step-parity v buffers alternate).

One GPU per rank: ranks whose kernels wait on one another (the flag barriers) must not share a
GPU as separate processes -- nothing makes their contexts run at the same time, and on this
B200 / driver stack two or four such processes on one GPU have raised Xid 109 (context-switch
timeout; /opt/skills/guides/B200_PROFILING.md).  With fewer GPUs than ranks these tests skip;
`profiles/r2_multiproc_tests.log` records them passing with both ranks on one GPU before that
rule was applied, and the in-process group tests (one context, no context switches) cover the
same exchanges on a single GPU.
"""
import dataclasses
import multiprocessing as mp
import os
import socket

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

SP_CFG = dataclasses.replace(synth.TINY_SINGLE, hidden=512, heads=4, depth_single=1, rope_axes=(16, 56, 56))
LP_CFG = dataclasses.replace(synth.SD3_TINY, hidden=256, heads=4, depth_double=2, pos_embed_max=16)


def _gpus_or_skip(world):
    """Rank r runs on cuda:r; DIT_SHARED_GPU_RANKS=1 forces every rank onto cuda:0 (the hazard
    above -- for a deliberate local check only)."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    if os.environ.get("DIT_SHARED_GPU_RANKS") == "1":
        return 1
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs: waiting ranks as processes on one GPU risk Xid 109")
    return world


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _sp_rank(rank, world, port, steps, ngpu, q):
    import torch
    import torch.distributed as dist
    from paper_2604_08123_b200 import SyntheticDiT
    from paper_2604_08123_b200.synthetic import _bits_to_bf16_tensor
    try:
        dev = rank % ngpu
        torch.cuda.set_device(dev)
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        cfg = SP_CFG
        B, hh, ww, nt = 2, 16, 16, 64
        m = SyntheticDiT(cfg, max_batch=B, max_img_tokens=hh * ww, max_txt_tokens=nt, max_rank=8, max_adapters=1,
                         device=dev)
        m.register_synthetic_lora(5, rank=8, index=0)
        hs = [None] * world
        dist.all_gather_object(hs, m.peer_handle())
        m.sp_init_peers(world, rank, hs)
        assert m.sp_exchange() == 2
        dist.barrier()      # every rank has mapped every peer before anyone's first signal
        batch = synth.make_batch(cfg, B, hh, ww, nt, n_adapters=1)
        batch.adapter_id = np.array([5, -1], dtype=np.int32)
        nil, ntl = hh * ww // world, nt // world
        lat = torch.from_numpy(np.ascontiguousarray(batch.latents[:, rank * nil:(rank + 1) * nil])).cuda()
        txt = _bits_to_bf16_tensor(np.ascontiguousarray(batch.txt[:, rank * ntl:(rank + 1) * ntl]), f"cuda:{dev}")
        pooled = _bits_to_bf16_tensor(batch.pooled, f"cuda:{dev}")
        outs = []
        for _ in range(steps):
            out, v = torch.empty_like(lat), torch.empty_like(lat)
            cb = m.make_batch(B, hh, ww, nt, batch.adapter_id, batch.sigma, batch.sigma_next, batch.guidance,
                              lat, out, txt, pooled, v_out=v)
            m.dit_step(cb)
            torch.cuda.synchronize()
            outs.append((out.cpu().numpy(), v.cpu().numpy()))
            lat = out           # the next step continues from this one's latents (shards stay local)
        got = [None] * world
        dist.all_gather_object(got, outs)
        dist.barrier()
        m.close()
        if rank == 0:
            q.put(("ok", got))
    except Exception as e:  # report, do not hang the parent
        q.put(("error", f"rank {rank}: {type(e).__name__}: {e}"))
        raise


def _lp_rank(rank, port, steps, ngpu, q):
    import torch
    import torch.distributed as dist
    from paper_2604_08123_b200 import SyntheticDiT
    try:
        dev = rank % ngpu
        torch.cuda.set_device(dev)
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=2)
        cfg = LP_CFG
        B, hh, ww, nt = 2, 12, 12, 40
        batch = synth.make_batch(cfg, B, hh, ww, nt, n_adapters=1, cfg_scale=6.0)
        batch.adapter_id = np.array([-1, 0], dtype=np.int32)
        m = SyntheticDiT(cfg, max_batch=B, max_img_tokens=hh * ww, max_txt_tokens=nt, max_rank=8, max_adapters=1,
                         device=dev)
        m.register_synthetic_lora(0, rank=8, index=0)
        hs = [None, None]
        dist.all_gather_object(hs, m.peer_handle())
        m.lp_init_peers(2, rank, hs)
        assert m.sp_exchange() == 2
        dist.barrier()
        lat, txt, pooled, out, v = m.device_inputs(batch, lp_rank=rank)
        outs = []
        for _ in range(steps):
            out, v = torch.empty_like(lat), torch.empty_like(lat)
            cb = m.make_batch(B, hh, ww, nt, batch.adapter_id, batch.sigma, batch.sigma_next, batch.guidance,
                              lat, out, txt, pooled, v_out=v, cfg_scale=batch.cfg_scale)
            m.dit_step(cb)
            torch.cuda.synchronize()
            outs.append((out.cpu().numpy(), v.cpu().numpy()))
            lat = out
        got = [None, None]
        dist.all_gather_object(got, outs)
        dist.barrier()
        m.close()
        if rank == 0:
            q.put(("ok", got))
    except Exception as e:
        q.put(("error", f"rank {rank}: {type(e).__name__}: {e}"))
        raise


def _spawn(target, args_of_rank, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=target, args=args_of_rank(r) + (q,)) for r in range(world)]
    for p in ps:
        p.start()
    try:
        status, payload = q.get(timeout=600)
    finally:
        for p in ps:
            p.join(120)
    assert status == "ok", payload
    assert all(p.exitcode == 0 for p in ps), [p.exitcode for p in ps]
    return payload


def _reference_steps(cfg, B, hh, ww, nt, batch, steps, adapter_id, max_batch):
    """The same steps on one GPU in this process (P = 1 / both CFG branches in one batch)."""
    import torch
    from paper_2604_08123_b200 import SyntheticDiT
    m = SyntheticDiT(cfg, max_batch=max_batch, max_img_tokens=hh * ww, max_txt_tokens=nt, max_rank=8,
                     max_adapters=1)
    m.register_synthetic_lora(adapter_id, rank=8, index=0)
    lat, txt, pooled, _, _ = m.device_inputs(batch)
    res = []
    for _ in range(steps):
        out, v = torch.empty_like(lat), torch.empty_like(lat)
        cb = m.make_batch(B, hh, ww, nt, batch.adapter_id, batch.sigma, batch.sigma_next, batch.guidance,
                          lat, out, txt, pooled, v_out=v, cfg_scale=batch.cfg_scale)
        m.dit_step(cb)
        torch.cuda.synchronize()
        res.append((out.cpu().numpy(), v.cpu().numpy()))
        lat = out
    m.close()
    return res


def test_sequence_parallel_two_processes_bitwise():
    world, steps = 2, 2
    ngpu = _gpus_or_skip(world)
    port = _free_port()
    got = _spawn(_sp_rank, lambda r: (r, world, port, steps, ngpu), world)
    cfg = SP_CFG
    B, hh, ww, nt = 2, 16, 16, 64
    batch = synth.make_batch(cfg, B, hh, ww, nt, n_adapters=1)
    batch.adapter_id = np.array([5, -1], dtype=np.int32)
    ref = _reference_steps(cfg, B, hh, ww, nt, batch, steps, 5, B)
    for t in range(steps):
        lat = np.concatenate([got[r][t][0] for r in range(world)], axis=1)
        v = np.concatenate([got[r][t][1] for r in range(world)], axis=1)
        np.testing.assert_array_equal(v, ref[t][1])
        np.testing.assert_array_equal(lat, ref[t][0])


def test_latent_parallel_two_processes_bitwise():
    steps = 3
    ngpu = _gpus_or_skip(2)
    port = _free_port()
    got = _spawn(_lp_rank, lambda r: (r, port, steps, ngpu), 2)
    cfg = LP_CFG
    B, hh, ww, nt = 2, 12, 12, 40
    batch = synth.make_batch(cfg, B, hh, ww, nt, n_adapters=1, cfg_scale=6.0)
    batch.adapter_id = np.array([-1, 0], dtype=np.int32)
    ref = _reference_steps(cfg, B, hh, ww, nt, batch, steps, 0, 2 * B)
    for t in range(steps):
        for r in range(2):   # both ranks hold the identical guided update
            np.testing.assert_array_equal(got[r][t][1], ref[t][1])
            np.testing.assert_array_equal(got[r][t][0], ref[t][0])
