"""Asynchronous LoRA loading and hot-patching ("pause
execution, hot-patch the base model in GPU memory, resume", :965-973, :1588-1592).

An adapter is registered (or merged) on a SIDE stream whose work is held back on the host
(dit_debug_host_delay) while the next dit_step is enqueued at once on the compute stream.  The
library orders the step after the copies / the merge with events on the step's own stream -- no
host synchronisation -- so the result must equal, bitwise, the fully synchronous sequence; and
the step must finish only after the delayed copies (it waited for them)."""
import ctypes as C
import dataclasses

import numpy as np
import pytest

import synth
from tests.test_gpu_parity import _model

pytestmark = pytest.mark.gpu

CFG = dataclasses.replace(synth.TINY_SINGLE, hidden=256, heads=2, depth_single=2, rope_axes=(16, 56, 56))
B, HH, WW, NT, RANK = 2, 8, 8, 16, 16


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return torch


def _adapter_tensors(torch, index, pinned_host):
    from paper_2604_08123_b200.dit import fill_synthetic
    out = {}
    for spec in synth.lora_manifest(CFG, RANK, index):
        t = torch.empty(spec.shape, dtype=torch.bfloat16, device="cuda")
        fill_synthetic(t, 3000 + index, spec.tensor_id, spec.scale, spec.offset)
        out[spec.name] = t.cpu().pin_memory() if pinned_host else t
    torch.cuda.synchronize()
    return out


def _batch():
    batch = synth.make_batch(CFG, B, HH, WW, NT, n_adapters=1)
    batch.adapter_id = np.array([7, -1], dtype=np.int32)
    return batch


def _timed_step(torch, m, batch):
    lat, txt, pooled, out, v = m.device_inputs(batch)
    cb = m.make_batch(B, HH, WW, NT, batch.adapter_id, batch.sigma, batch.sigma_next, batch.guidance, lat, out, txt,
                      pooled, v_out=v)
    e1 = torch.cuda.Event(enable_timing=True)
    m.dit_step(cb)
    e1.record()
    return out, v, e1


@pytest.mark.parametrize("source", ["device", "pinned_host"])
def test_register_on_side_stream_then_step_bitwise(torch_cuda, source):
    torch = torch_cuda
    from paper_2604_08123_b200 import dit
    lib = dit.load_library()
    batch = _batch()
    ref = _model(CFG, B, HH * WW, NT, rank=RANK, adapters=1)
    ref.lora_register(7, RANK, 1.0, _adapter_tensors(torch, 0, False))
    torch.cuda.synchronize()
    lat_ref, v_ref = ref.step(batch)
    ref.close()

    m = _model(CFG, B, HH * WW, NT, rank=RANK, adapters=1)
    tens = _adapter_tensors(torch, 0, source == "pinned_host")
    side = torch.cuda.Stream()
    delay_ms = 60.0
    e0 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(side)
    assert lib.dit_debug_host_delay(C.c_void_p(side.cuda_stream), int(delay_ms * 1e6)) == 0
    m.lora_register(7, RANK, 1.0, tens, stream=side)   # returns at once; copies run after the delay
    out, v, e1 = _timed_step(torch, m, batch)           # enqueued right away on the compute stream
    torch.cuda.synchronize()
    np.testing.assert_array_equal(v.cpu().numpy(), v_ref)
    np.testing.assert_array_equal(out.cpu().numpy(), lat_ref)
    assert e0.elapsed_time(e1) >= delay_ms - 1.0       # the step waited for the copies
    m.close()


def test_merge_on_side_stream_then_step_bitwise(torch_cuda):
    """Hot patch at a step boundary: register + merge on a delayed side stream, step at once."""
    torch = torch_cuda
    from paper_2604_08123_b200 import dit
    lib = dit.load_library()
    batch = _batch()
    batch.adapter_id = np.array([7, 7], dtype=np.int32)     # a patched replica serves its adapter only
    ref = _model(CFG, B, HH * WW, NT, rank=RANK, adapters=1)
    ref.lora_register(7, RANK, 1.0, _adapter_tensors(torch, 0, False))
    ref.lora_merge(7)
    torch.cuda.synchronize()
    lat_ref, v_ref = ref.step(batch)
    ref.lora_unmerge()
    ref.close()

    m = _model(CFG, B, HH * WW, NT, rank=RANK, adapters=1)
    _, v_base = m.step(dataclasses.replace(batch, adapter_id=np.array([-1, -1], dtype=np.int32)))
    tens = _adapter_tensors(torch, 0, False)
    side = torch.cuda.Stream()
    torch.cuda.synchronize()
    assert lib.dit_debug_host_delay(C.c_void_p(side.cuda_stream), int(50e6)) == 0
    m.lora_register(7, RANK, 1.0, tens, stream=side)
    m.lora_merge(7, stream=side)
    out, v, _ = _timed_step(torch, m, batch)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(v.cpu().numpy(), v_ref)
    np.testing.assert_array_equal(out.cpu().numpy(), lat_ref)
    # unmerge restores the base model exactly
    m.lora_unmerge()
    _, v_after = m.step(dataclasses.replace(batch, adapter_id=np.array([-1, -1], dtype=np.int32)))
    np.testing.assert_array_equal(v_after, v_base)
    m.close()


def test_load_weights_rejected_while_merged(torch_cuda):
    """replacing base weights under a merged copy would leave the step on a stale patch."""
    torch = torch_cuda
    from paper_2604_08123_b200.dit import DitError
    m = _model(CFG, B, HH * WW, NT, rank=RANK, adapters=1)
    m.lora_register(7, RANK, 1.0, _adapter_tensors(torch, 0, False))
    m.lora_merge(7)
    name = "double.0.img.qkv.w"
    with pytest.raises(DitError) as e:
        m.dit_load_weights({name: m.weights[name].clone()})
    assert e.value.code == 1
    m.lora_unmerge()
    m.dit_load_weights({name: m.weights[name].clone()})     # accepted once unmerged
    m.close()
