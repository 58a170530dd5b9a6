"""Integer plan tables, event-deferred ControlNet inputs and the longest attention, on the GPU.

* LoRA segment indexing (north_star: "bit-exact for LoRA segment indexing"): the row -> slot,
  tile -> slots and shrink work-list tables the LAST dit_step uploaded (read back from the device,
  dit_debug_plan) equal an independent CPU emulation written here from the definitions in
  DESIGN.md §5.1 (256-row tiles, distinct slots sorted, (tile, slot) pairs in tile order), at the
  cfg3 shape (B = 8, 512 + 4096 tokens, 4 rank-64 adapters), with CFG doubling, after slot reuse.
* Deferred ControlNet input with a CUDA event (the fetch "returns immediately
  if the data is available, or blocks until the data arrives", stall =
  max(0, t_cn - t_flux)): the producer's event is waited on right before the consuming GEMM, so a
  late producer stalls the step only at the consumption point.
* Attention at cfg5 length (N = 16 896) against torch fp32 on sampled query rows.
"""
import ctypes as C
import dataclasses

import numpy as np
import pytest

import synth
from tests.test_gpu_parity import _model

pytestmark = pytest.mark.gpu

TM = 256   # GEMM rows per 2-SM tile


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return torch


def emulate_plan(seq_slot, rows_per_seq, slot_cap):
    """Independent CPU emulation of the segmented-LoRA plan of one GEMM row space."""
    M = len(seq_slot) * rows_per_seq
    row_slot = np.repeat(np.asarray(seq_slot, dtype=np.int32), rows_per_seq)
    tiles = (M + TM - 1) // TM
    tile_slots = np.zeros((tiles, slot_cap), dtype=np.int32)
    tile_cnt = np.zeros(tiles, dtype=np.int32)
    shrink = []
    for t in range(tiles):
        sl = sorted({int(x) for x in row_slot[t * TM:(t + 1) * TM] if x >= 0})
        tile_cnt[t] = len(sl)
        tile_slots[t, :len(sl)] = sl
        shrink += [(t, x) for x in sl]
    return row_slot, tile_slots.ravel(), tile_cnt, np.asarray(shrink, dtype=np.int32).ravel()


def _check_plan(m, seq_slot, nt, ni, slot_cap):
    for which, rows in ((0, nt), (1, ni), (2, nt + ni)):
        exp = emulate_plan(seq_slot, rows, slot_cap)
        for kind in range(4):
            got = np.asarray(m.debug_plan(which, kind), dtype=np.int32)
            np.testing.assert_array_equal(got, exp[kind], err_msg=f"row space {which} table {kind}")


def test_lora_plan_tables_bit_exact_cfg3_shape(torch_cuda):
    cfg = synth.flux_reduced(1, 1)      # full Flux width; depth does not change the plan
    B, hh, ww, nt = 8, 64, 64, 512
    m = _model(cfg, B, hh * ww, nt, rank=64, adapters=4)
    ids = [11, 22, 33, 44]
    for i, a in enumerate(ids):         # registration order -> first free pool slot (0, 1, 2, 3)
        m.register_synthetic_lora(a, rank=64, index=i)
    slot_of = {a: i for i, a in enumerate(ids)}
    batch = synth.make_batch(cfg, B, hh, ww, nt, n_adapters=4)
    batch.adapter_id = np.array([ids[x] for x in synth.adapter_ids(B, 4)], dtype=np.int32)
    batch.adapter_id[5] = -1            # one base-model request in the batch
    m.step(batch)
    seq_slot = [slot_of.get(int(a), -1) for a in batch.adapter_id]
    _check_plan(m, seq_slot, nt, hh * ww, B)
    # the host planner export agrees with what the step uploaded
    lat, txt, pooled, out, v = m.device_inputs(batch)
    cb = m.make_batch(B, hh, ww, nt, batch.adapter_id, batch.sigma, batch.sigma_next, batch.guidance, lat, out,
                      txt, pooled)
    ra = m.debug_row_adapter(cb, 1 << 20)
    np.testing.assert_array_equal(ra, np.concatenate([np.repeat(seq_slot, nt), np.repeat(seq_slot, hh * ww)]))
    # slot reuse: unregister 22 (slot 1), register 55 -> takes slot 1
    m.lora_unregister(22)
    m.register_synthetic_lora(55, rank=32, index=5)
    batch.adapter_id = np.array([55, 11, 55, 44, -1, 33, 11, 55], dtype=np.int32)
    slot_of = {11: 0, 55: 1, 33: 2, 44: 3}
    m.step(batch)
    _check_plan(m, [slot_of.get(int(a), -1) for a in batch.adapter_id], nt, hh * ww, B)
    m.close()


def test_lora_plan_tables_with_cfg_doubling(torch_cuda):
    """CFG on one GPU: 2B sequences, sequence q carries request q % B's adapter (reading C22)."""
    cfg = dataclasses.replace(synth.SD3_TINY, hidden=128, heads=2, pos_embed_max=40)
    B, hh, ww, nt = 3, 20, 20, 40
    m = _model(cfg, 2 * B, hh * ww, nt, rank=8, adapters=2)
    m.register_synthetic_lora(7, rank=8, index=0)
    m.register_synthetic_lora(9, rank=4, index=1)
    batch = synth.make_batch(cfg, B, hh, ww, nt, n_adapters=2, cfg_scale=4.0)
    batch.adapter_id = np.array([9, -1, 7], dtype=np.int32)
    m.step(batch)
    seq = [1, -1, 0] * 2
    _check_plan(m, seq, nt, hh * ww, 2 * B)
    m.close()


def _cn_setup(torch_cuda):
    cfg = dataclasses.replace(synth.TINY_SINGLE, hidden=512, heads=4, depth_double=4, depth_single=8,
                              rope_axes=(16, 56, 56))
    B, hh, ww, nt = 2, 32, 32, 128
    m = _model(cfg, B, hh * ww, nt)
    batch = synth.make_batch(cfg, B, hh, ww, nt)
    return cfg, m, batch


def test_controlnet_event_deferred_fetch_and_stall_point(torch_cuda):
    """A producer on another stream writes the residual `delay` after the step is enqueued and
    records a CUDA event; the step waits on it only right before the consuming GEMM.  (1) bitwise
    equal to the resident residual; (2) with the residual consumed by the LAST block the step ends
    about `delay` after it started (everything before the consumption point ran during the delay);
    consumed by the FIRST block, the rest of the step runs after the delay."""
    torch = torch_cuda
    from paper_2604_08123_b200 import dit
    from paper_2604_08123_b200.synthetic import _bits_to_bf16_tensor
    cfg, m, batch = _cn_setup(torch)
    ni, D = batch.img_tokens, cfg.hidden
    last = cfg.depth_double + cfg.depth_single - 1
    bits = synth.controlnet_residual_bf16(1, 0, ni, D)
    lib = dit.load_library()
    prod = torch.cuda.Stream()
    src = _bits_to_bf16_tensor(bits, "cuda")

    def run(block, delay_ms):
        lat, txt, pooled, out, v = m.device_inputs(batch)
        R = torch.zeros(ni, D, dtype=torch.bfloat16, device="cuda")
        cb = m.make_batch(batch.batch, batch.img_h, batch.img_w, batch.txt_tokens, batch.adapter_id, batch.sigma,
                          batch.sigma_next, batch.guidance, lat, out, txt, pooled, v_out=v)
        torch.cuda.synchronize()
        ready = torch.cuda.Event()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        # the "ControlNet executor": its output lands `delay_ms` later (a host-side stall of its stream
        # occupies no SM, so the DiT's persistent kernels keep every SM), then its event
        with torch.cuda.stream(prod):
            assert lib.dit_debug_host_delay(C.c_void_p(prod.cuda_stream), int(delay_ms * 1e6)) == 0
            R.copy_(src)
            ready.record(prod)
        m.controlnet_inject(1, block, R, 1.0, ready_event=ready)
        e0.record()
        m.dit_step(cb)
        e1.record()
        torch.cuda.synchronize()
        return out.cpu().numpy(), v.cpu().numpy(), e0.elapsed_time(e1)

    # resident reference and the plain step time
    for blk in (0, last):
        lat_ref, v_ref = m.step(batch, injections=[(1, blk, bits, 1.0)])
        lat, v, _ = run(blk, 30.0)
        np.testing.assert_array_equal(v, v_ref)
        np.testing.assert_array_equal(lat, lat_ref)
    t_plain = min(run(last, 0.0)[2] for _ in range(3))
    delay = max(40.0, 8 * t_plain)
    t_late = min(run(last, delay)[2] for _ in range(2))
    t_early = min(run(0, delay)[2] for _ in range(2))
    # the wait sits at the consumption point: consumed last, the step is hidden under the delay
    assert t_late < delay + 0.35 * t_plain + 1.0, (t_late, delay, t_plain)
    assert t_late >= delay - 1.0, (t_late, delay)
    # consumed first: (almost) the whole step runs after the data arrives
    assert t_early > delay + 0.6 * t_plain, (t_early, delay, t_plain)
    m.close()


def test_controlnet_registrations_cleared_on_failed_step_and_by_clear(torch_cuda):
    """a failed dit_step (here a rejected batch) must not leave registrations behind, and
    controlnet_clear drops pending ones: the next step equals the plain step bitwise."""
    torch = torch_cuda
    from paper_2604_08123_b200.dit import DitError
    cfg = synth.TINY_SINGLE
    m = _model(cfg, 2, 16, 8)
    batch = synth.make_batch(cfg, 2, 4, 4, 8)
    _, v_plain = m.step(batch)
    r = torch.ones(16, cfg.hidden, dtype=torch.bfloat16, device="cuda")
    m.controlnet_inject(1, 0, r)
    bad = dataclasses.replace(batch, txt_tokens=batch.txt_tokens * 4)    # exceeds max_txt_tokens
    with pytest.raises(DitError):
        m.step(bad)
    _, v = m.step(batch)
    np.testing.assert_array_equal(v, v_plain)
    m.controlnet_inject(1, 0, r)
    assert m.lib.controlnet_clear(m.ctx) == 0
    _, v = m.step(batch)
    np.testing.assert_array_equal(v, v_plain)
    m.close()


def test_attention_cfg5_length_vs_torch_fp32(torch_cuda):
    """The tcgen05 attention at cfg5's joint length (512 + 16384 = 16 896 tokens, 24 heads of 128)
    against torch fp32 on 512 sampled query rows per head (every key)."""
    torch = torch_cuda
    from paper_2604_08123_b200 import dit
    lib = dit.load_library()
    B, H, N, d = 1, 24, 512 + 128 * 128, 128
    g = torch.Generator(device="cuda").manual_seed(16896)
    q, k, v = (torch.randn(B, H, N, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    out = torch.zeros(B * N, H * d, device="cuda", dtype=torch.bfloat16)
    s = torch.cuda.current_stream()
    assert lib.dit_debug_attention(q.data_ptr(), k.data_ptr(), v.data_ptr(), B, H, N, d, out.data_ptr(),
                                   C.c_void_p(s.cuda_stream)) == 0
    torch.cuda.synchronize()
    assert torch.isfinite(out.float()).all()
    rows = torch.cat([torch.arange(0, 256, device="cuda"),            # first query block, text rows
                      torch.randint(256, N - 256, (128,), device="cuda", generator=g),
                      torch.arange(N - 128, N, device="cuda")])      # the ragged last block
    kf, vf = k[0].float(), v[0].float()
    qf = q[0][:, rows].float()
    p = torch.softmax(qf @ kf.transpose(-1, -2) / d ** 0.5, dim=-1)
    ref = (p @ vf).permute(1, 0, 2).reshape(len(rows), H * d)
    got = out[rows].float()
    err = ((got - ref).abs().max() / ref.abs().max()).item()
    cos = torch.nn.functional.cosine_similarity(got.flatten(), ref.flatten(), dim=0).item()
    assert err < 1e-2, err
    assert cos > 0.9999, cos
