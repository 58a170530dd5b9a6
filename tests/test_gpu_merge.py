"""Merged-LoRA (weight patching) mode: lora_merge / lora_unmerge.

PAPER.md:335-345 (adapters patch the base weights, no per-step overhead), :391-400 (hot-patch
at a step boundary).  The merged copy W' = bf16(W + s B A) is checked against numpy, a merged
step against the fp64 oracle (whose unmerged LoRA equals the merged form, pin P2), and
lora_unmerge against the pre-merge step bit for bit."""
from __future__ import annotations

import numpy as np
import pytest

import synth
from oracle import flux_step as O
from oracle.flux_step import bf16_to_f64
from tests.helpers import oracle_adapter
from tests.test_gpu_parity import _model, check, torch_cuda  # noqa: F401 (fixture)

pytestmark = pytest.mark.gpu


def _bf16_rne(x64: np.ndarray) -> np.ndarray:
    b = np.asarray(x64, dtype=np.float32).view(np.uint32).astype(np.uint64)
    return ((b + 0x7FFF + ((b >> 16) & 1)) >> 16).astype(np.uint16)


def _merged_modules(m, cfg):
    """The merged buffer of the model, split per adapted linear (pool order, 256-byte aligned)."""
    buf = m._merged
    pad = (-buf.data_ptr()) % 256
    raw = buf.cpu().numpy()[pad:]
    W = synth.make_weights_bf16(cfg)
    out, off = {}, 0
    for mod, _, _ in synth.lora_targets(cfg):
        o, i = W[mod + ".w"].shape
        out[mod] = raw[off:off + o * i * 2].view(np.uint16).reshape(o, i)
        off = (off + o * i * 2 + 255) // 256 * 256
    return out


@pytest.mark.parametrize("wide,rank", [(False, 8), (True, 100)])
def test_merged_weights_match_numpy(torch_cuda, wide, rank):
    """rank 8 (r_alloc 64) on 64-wide tiles; rank 100 (r_alloc 128, two K panels) on a 256-wide model
    (ragged 128 x 128 merge tiles at the F + D = 1280 / 768 edges)."""
    import dataclasses
    cfg = (dataclasses.replace(synth.TINY_SINGLE, hidden=256, heads=2, rope_axes=(16, 56, 56)) if wide
           else synth.TINY_SINGLE)
    scale = 0.75
    m = _model(cfg, 2, 16, 8, rank=rank, adapters=2)
    m.register_synthetic_lora(5, rank=rank, index=1, scale=scale)
    m.lora_merge(5)
    torch_cuda.cuda.synchronize()
    got = _merged_modules(m, cfg)
    W = synth.make_weights_bf16(cfg)
    L = synth.make_lora_bf16(cfg, rank, 1)
    for mod, _, _ in synth.lora_targets(cfg):
        ref = bf16_to_f64(W[mod + ".w"]) + scale * bf16_to_f64(L[mod + ".lora_B"]) @ bf16_to_f64(L[mod + ".lora_A"])
        want = _bf16_rne(ref)
        g = got[mod]
        # same value up to one bf16 ulp (fp32 accumulation order), and almost always exact; more
        # than one ulp only where W and s B A cancel (absolute error far below the tensor's scale)
        ulp = np.abs(g.astype(np.int64) - want.astype(np.int64))
        far = ulp > 1
        if far.any():
            err = np.abs(bf16_to_f64(g) - ref)[far]
            assert err.max() <= 1e-5 * np.abs(ref).max(), (mod, int(ulp.max()), float(err.max()))
        assert (ulp == 0).mean() > 0.99, (mod, float((ulp == 0).mean()))


@pytest.mark.parametrize("cfg_name", ["TINY", "TINY_SINGLE"])
def test_merged_step_parity_and_exact_restore(torch_cuda, cfg_name):
    cfg = getattr(synth, cfg_name)
    rank = 8
    m = _model(cfg, 2, 16, 8, rank=rank, adapters=2)
    m.register_synthetic_lora(3, rank=rank, index=0)
    batch = synth.make_batch(cfg, 2, 4, 4, 8, n_adapters=1)
    batch.adapter_id = np.array([3, 3], dtype=np.int32)
    lat_u, v_u = m.step(batch)                       # unmerged (segmented LoRA)
    base = synth.make_batch(cfg, 2, 4, 4, 8, n_adapters=1)
    base.adapter_id = np.array([-1, -1], dtype=np.int32)
    lat_b, v_b = m.step(base)                        # bare base model
    m.lora_merge(3)
    lat_m, v_m = m.step(batch)                       # patched replica
    W = O.weights_to_f64(synth.make_weights_bf16(cfg))
    x_o, v_o = O.dit_step(cfg, W, batch, {3: oracle_adapter(cfg, rank, 0)[0]})
    check(v_m, v_o, "v merged")
    check(lat_m, x_o, "latents merged")
    # the merged and segmented forms agree to rounding (not bitwise: W' is rounded to bf16)
    assert np.abs(v_m - v_u).max() / np.abs(v_u).max() < 2e-2
    with pytest.raises(Exception):
        m.step(base)                                 # a patched replica only serves its adapter
    m.lora_unmerge()
    lat_u2, v_u2 = m.step(batch)
    lat_b2, v_b2 = m.step(base)
    np.testing.assert_array_equal(v_u2, v_u)         # restore is exact
    np.testing.assert_array_equal(lat_b2, lat_b)
    np.testing.assert_array_equal(v_b2, v_b)


def test_merge_error_paths(torch_cuda):
    import torch
    from paper_2604_08123_b200.dit import DitError
    cfg = synth.TINY_SINGLE
    m = _model(cfg, 2, 16, 8, rank=8, adapters=2)
    m.register_synthetic_lora(1, rank=8, index=0)
    m.register_synthetic_lora(2, rank=4, index=1)
    codes = lambda f: (lambda e: e.code)(pytest.raises(DitError, f).value)
    assert codes(lambda: m.lora_merge(9)) == 7                       # DIT_ENOENT
    small = torch.empty(1024, dtype=torch.uint8, device="cuda")
    assert codes(lambda: m.lora_merge(1, merged=small)) == 2         # DIT_ENOMEM
    assert codes(lambda: m.lora_unmerge()) == 7                      # nothing merged
    m.lora_merge(1)
    assert codes(lambda: m.lora_merge(2)) == 4                       # DIT_EEXIST
    assert codes(lambda: m.lora_unregister(1)) == 1                  # merged adapter is pinned
    batch = synth.make_batch(cfg, 2, 4, 4, 8, n_adapters=2)
    batch.adapter_id = np.array([1, 2], dtype=np.int32)
    assert codes(lambda: m.step(batch)) == 10                        # DIT_EADAPTER
    m.lora_unmerge()
    m.lora_unregister(1)


@pytest.mark.parametrize("wide,rank", [(False, 8), (True, 100)])
def test_inplace_merge_exact_restore(torch_cuda, wide, rank):
    """In-place hot patch: W' over the base weights, no second copy.
    The merged step equals the copy-merged step bitwise (same W'); lora_unmerge gives back every
    base weight BIT FOR BIT (inverse + undo log of the unrecoverable elements); a too-small undo
    log is refused with DIT_ENOMEM before anything is written."""
    import dataclasses
    torch = torch_cuda
    from paper_2604_08123_b200.dit import DitError
    cfg = (dataclasses.replace(synth.TINY_SINGLE, hidden=256, heads=2, rope_axes=(16, 56, 56)) if wide
           else synth.TINY_SINGLE)
    hh, ww, nt = (8, 8, 16) if wide else (4, 4, 8)
    batch = synth.make_batch(cfg, 2, hh, ww, nt, n_adapters=1)
    batch.adapter_id = np.array([5, 5], dtype=np.int32)
    ref = _model(cfg, 2, hh * ww, nt, rank=rank, adapters=1)
    ref.register_synthetic_lora(5, rank=rank, index=1, scale=0.75)
    ref.lora_merge(5)
    lat_copy, v_copy = ref.step(batch)
    ref.lora_unmerge()
    ref.close()

    m = _model(cfg, 2, hh * ww, nt, rank=rank, adapters=1)
    m.register_synthetic_lora(5, rank=rank, index=1, scale=0.75)
    base = dataclasses.replace(batch, adapter_id=np.array([-1, -1], dtype=np.int32))
    _, v_base = m.step(base)
    before = {k: t.clone() for k, t in m.weights.items()}
    small = torch.empty(1, dtype=torch.int64, device="cuda")
    with pytest.raises(DitError) as e:
        m.lora_merge_inplace(5, undo=small)          # 8 bytes: too small for any real adapter
    assert e.value.code == 2
    for k, t in m.weights.items():
        assert torch.equal(t, before[k]), k          # refused before anything was written
    n = m.lora_merge_inplace(5)
    torch.cuda.synchronize()
    changed = sum(int((m.weights[mod + ".w"] != before[mod + ".w"]).sum()) for mod, _, _ in synth.lora_targets(cfg))
    assert changed > 0 and 0 < n < changed            # patched in place; only some elements logged
    lat, v = m.step(batch)
    np.testing.assert_array_equal(v, v_copy)
    np.testing.assert_array_equal(lat, lat_copy)
    m.lora_unmerge()
    for k, t in m.weights.items():
        assert torch.equal(t, before[k]), k          # exact restore
    _, v_after = m.step(base)
    np.testing.assert_array_equal(v_after, v_base)
    m.close()
