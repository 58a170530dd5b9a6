"""ControlNet hand-off across processes with device ready flags.

A producer PROCESS -- standing in for a ControlNet executor on another GPU -- maps the
DiT executor's registered residual buffer and ready flag through CUDA IPC
(dit_ipc_export / dit_ipc_open), waits until the DiT's dit_step has been enqueued, and
then pushes the residual with controlnet_push (grid copy + system-scope release of the
flag).  The DiT's fc2 epilogue acquires the flag mid-step (deferred fetch, PAPER.md:
1058-1076) and the result must equal, bitwise, the step with the residual resident from
the start.  Same GPU here (one GPU per call); across GPUs only the mapping changes (the
stores go over NVLink).
"""
import dataclasses
import multiprocessing as mp
import os
import time

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu


def _producer(h_res, h_flag, bits, value, dev, conn):
    import torch
    from paper_2604_08123_b200 import dit
    from paper_2604_08123_b200.synthetic import _bits_to_bf16_tensor
    torch.cuda.set_device(dev)
    dst = dit.ipc_open(h_res)
    flag = dit.ipc_open(h_flag)
    src = _bits_to_bf16_tensor(bits, f"cuda:{dev}")
    torch.cuda.synchronize()
    conn.send("ready")
    conn.recv()                       # the consumer has enqueued its dit_step
    time.sleep(0.05)
    dit.controlnet_push(dst, src, flag, value)
    torch.cuda.synchronize()
    dit.ipc_close(dst)
    dit.ipc_close(flag)
    conn.send("pushed")


def test_controlnet_push_from_another_process(request):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    if os.environ.get("DIT_SHARED_GPU_RANKS") == "1":
        pdev = 0
    elif torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs: a producer process on the consumer's GPU risks Xid 109")
    else:
        pdev = 1
    from paper_2604_08123_b200 import SyntheticDiT
    cfg = dataclasses.replace(synth.TINY_SINGLE, hidden=256, heads=2, rope_axes=(16, 56, 56))
    B, hh, ww, nt = 2, 8, 8, 16
    m = SyntheticDiT(cfg, max_batch=B, max_img_tokens=hh * ww, max_txt_tokens=nt)
    batch = synth.make_batch(cfg, B, hh, ww, nt)
    bits = synth.controlnet_residual_bf16(1, 0, hh * ww, cfg.hidden)
    lat_ref, v_ref = m.step(batch, injections=[(1, 0, bits, 1.0)])

    R = torch.zeros(hh * ww, cfg.hidden, dtype=torch.bfloat16, device="cuda")
    flag = torch.zeros(4, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    from paper_2604_08123_b200 import dit
    ctx = mp.get_context("spawn")
    parent, child = ctx.Pipe()
    p = ctx.Process(target=_producer, args=(dit.ipc_export(R), dit.ipc_export(flag[1:2]), bits, 7, pdev, child))
    p.start()
    try:
        assert parent.poll(120) and parent.recv() == "ready"
        m.controlnet_inject_flag(1, 0, R, flag[1:2], 7)
        parent.send("go")
        lat, v = m.step(batch)        # blocks in the fc2 epilogue until the producer's flag lands
        assert parent.poll(60) and parent.recv() == "pushed"
    finally:
        p.join(60)
    assert p.exitcode == 0
    assert int(flag[1].item()) == 7 and int(flag[0].item()) == 0 and int(flag[2].item()) == 0
    np.testing.assert_array_equal(v, v_ref)
    np.testing.assert_array_equal(lat, lat_ref)
    # and the residual mattered
    _, v_plain = m.step(batch)
    assert np.abs(v_plain - v_ref).max() > 1e-3
