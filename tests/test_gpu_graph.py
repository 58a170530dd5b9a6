"""CUDA-graph replay of the denoise step (dit_graph_create / dit_graph_launch): the captured step
replayed with new per-step scalars (sigma pairs of a 4-step schedule, ControlNet scales) must
equal the plain dit_step bitwise, with LoRA on one request and a ControlNet residual on the other;
two graphs ping-pong the latents buffers, as a serving loop would."""
import dataclasses

import numpy as np
import pytest

import synth
from tests.test_gpu_parity import _model

pytestmark = pytest.mark.gpu

CFG = dataclasses.replace(synth.TINY_SINGLE, hidden=256, heads=2, depth_single=2, rope_axes=(16, 56, 56))
B, HH, WW, NT = 2, 8, 8, 16


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return torch


def test_graph_replay_equals_dit_step(torch_cuda):
    torch = torch_cuda
    from paper_2604_08123_b200.synthetic import _bits_to_bf16_tensor
    batch = synth.make_batch(CFG, B, HH, WW, NT, n_adapters=1)
    batch.adapter_id = np.array([3, -1], dtype=np.int32)
    sig = synth.flux_sigmas(4, HH * WW)
    R = _bits_to_bf16_tensor(synth.controlnet_residual_bf16(1, 0, HH * WW, CFG.hidden), "cuda")

    def run(use_graph):
        m = _model(CFG, B, HH * WW, NT, rank=8, adapters=1)
        m.register_synthetic_lora(3, rank=8, index=0)
        lat, txt, pooled, out, v = m.device_inputs(batch)
        bufs = [lat, out]
        torch.cuda.synchronize()
        s = torch.cuda.Stream()
        graphs = [None, None]
        res = []
        with torch.cuda.stream(s):
            for t in range(4):
                src, dst = bufs[t % 2], bufs[(t + 1) % 2]
                sg = np.full(B, sig[t], np.float32)
                sn = np.full(B, sig[t + 1], np.float32)
                cn_scale = np.array([1.0, 0.5 + 0.25 * t], np.float32)
                cb = m.make_batch(B, HH, WW, NT, batch.adapter_id, sg, sn, batch.guidance, src, dst, txt, pooled,
                                  v_out=v, cn_scale=cn_scale)
                m.controlnet_inject(1, 0, R, 0.8)
                if not use_graph:
                    m.dit_step(cb, stream=s)
                else:
                    if graphs[t % 2] is None:
                        graphs[t % 2] = m.graph_create(cb, stream=s)
                        m.controlnet_inject(1, 0, R, 0.8)      # capture consumed the registration
                    m.graph_launch(graphs[t % 2], cb, stream=s)
                s.synchronize()
                res.append((dst.cpu().numpy(), v.cpu().numpy()))
        for g in graphs:
            if g is not None:
                m.graph_destroy(g)
        m.close()
        return res

    plain = run(False)
    replay = run(True)
    for t in range(4):
        np.testing.assert_array_equal(replay[t][1], plain[t][1])
        np.testing.assert_array_equal(replay[t][0], plain[t][0])
    assert not np.array_equal(plain[0][1], plain[1][1])           # the steps really differ


def test_graph_rejects_a_different_batch(torch_cuda):
    torch = torch_cuda
    from paper_2604_08123_b200.dit import DitError
    batch = synth.make_batch(CFG, B, HH, WW, NT)
    m = _model(CFG, B, HH * WW, NT)
    lat, txt, pooled, out, v = m.device_inputs(batch)
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    cb = m.make_batch(B, HH, WW, NT, batch.adapter_id, batch.sigma, batch.sigma_next, batch.guidance, lat, out, txt,
                      pooled)
    g = m.graph_create(cb, stream=s)
    out2 = torch.empty_like(out)
    cb2 = m.make_batch(B, HH, WW, NT, batch.adapter_id, batch.sigma, batch.sigma_next, batch.guidance, lat, out2,
                       txt, pooled)
    with pytest.raises(DitError) as e:
        m.graph_launch(g, cb2, stream=s)                           # another output buffer
    assert e.value.code == 1
    m.controlnet_inject(0, 0, torch.zeros(HH * WW, CFG.hidden, dtype=torch.bfloat16, device="cuda"))
    with pytest.raises(DitError):
        m.graph_launch(g, cb, stream=s)                            # registrations differ from the capture
    m.lib.controlnet_clear(m.ctx)
    m.graph_launch(g, cb, stream=s)
    s.synchronize()
    m.graph_destroy(g)
    m.close()
