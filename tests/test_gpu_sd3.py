"""GPU parity of the SD3 / SD3.5 MMDiT step, classifier-free guidance and latent (CFG)
parallelism (readings C21, C22) against the fp64 oracle
(oracle/sd3_step.py), through the C ABI.

Tolerance as tests/test_gpu_parity.py (north_star: max_rel <= 2e-2, cosine >= 0.999 per
output tensor per request); the bitwise checks rest on batch invariance (row-independent
GEMMs with a fixed K order, pins P3/P9).
"""
import dataclasses

import numpy as np
import pytest

import synth
from oracle import flux_step as O
from oracle import sd3_step as S
from tests.helpers import oracle_adapter
from tests.test_gpu_parity import check

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return torch


def _model(cfg, B, ni, nt, rank=0, adapters=0):
    from paper_2604_08123_b200 import SyntheticDiT
    return SyntheticDiT(cfg, max_batch=B, max_img_tokens=ni, max_txt_tokens=nt, max_rank=rank, max_adapters=adapters)


def _cn(cfg, slots, ni):
    """slot -> {block: residual bits}, and the oracle's ControlNetInput lists (every joint block)."""
    bits = {s: {i: synth.controlnet_residual_bf16(s, i, ni, cfg.hidden) for i in range(cfg.depth_double)}
            for s in slots}
    cns = {s: [O.ControlNetInput(double={i: O.bf16_to_f64(r) for i, r in d.items()}, single={},
                                 n_res=cfg.depth_double, n_res_single=0)] for s, d in bits.items()}
    return bits, cns


# d = 32 (mma.sync attention, QK-norm), d = 64 without QK-norm (SD3-medium head size), d = 128
# (tcgen05 attention with the identity RoPE table)
CFGS = {
    "tiny_d32": dataclasses.replace(synth.SD3_TINY, pos_embed_max=16),
    "d64_noqk": dataclasses.replace(synth.SD3_TINY, hidden=128, heads=2, depth_double=3, qk_norm=False,
                                    pos_embed_max=24, pos_embed_base=8),
    "d128": dataclasses.replace(synth.SD3_TINY, hidden=256, heads=2, depth_double=2, pos_embed_max=16),
}


@pytest.mark.parametrize("name", list(CFGS))
@pytest.mark.parametrize("with_cfg", [True, False])
def test_sd3_step_parity(torch_cuda, name, with_cfg):
    """Mixed LoRA ([0, -1]) + ControlNet on two sequences, ragged tiles (10 x 15 grid, 40 text tokens)."""
    cfg = CFGS[name]
    B, hh, ww, nt = 2, 10, 15, 40
    ni = hh * ww
    m = _model(cfg, 2 * B, ni, nt, rank=8, adapters=1)
    m.register_synthetic_lora(0, rank=8, index=0, scale=0.8)
    batch = synth.make_batch(cfg, B, hh, ww, nt, n_adapters=1, cfg_scale=4.5 if with_cfg else None)
    batch.adapter_id = np.array([0, -1], dtype=np.int32)
    slots = [0, 3] if with_cfg else [1]
    bits, cns = _cn(cfg, slots, ni)
    lat, v = m.step(batch, controlnet=bits)
    W = O.weights_to_f64(synth.make_weights_bf16(cfg))
    x_o, v_o = S.dit_step(cfg, W, batch, {0: oracle_adapter(cfg, 8, 0, scale=0.8)[0]}, cns)
    check(v, v_o, f"{name} v")
    check(lat, x_o, f"{name} latents_out")


def test_sd3_cfg_scale_zero_is_unconditional_bitwise(torch_cuda):
    """g = 0 gives v_u + 0 (v_c - v_u) = v_u exactly, and the unconditional sequence does not
    depend on its batch-mates: the CFG step equals a plain step on the negative prompts bitwise."""
    cfg = CFGS["d128"]
    B, hh, ww, nt = 2, 8, 8, 24
    m = _model(cfg, 2 * B, hh * ww, nt)
    batch = synth.make_batch(cfg, B, hh, ww, nt, cfg_scale=0.0)
    lat, v = m.step(batch)
    plain = dataclasses.replace(batch, cfg_scale=None, txt=batch.txt_neg, pooled=batch.pooled_neg)
    lat_u, v_u = m.step(plain)
    np.testing.assert_array_equal(v, v_u)
    np.testing.assert_array_equal(lat, lat_u)
    # and g = 1 against the conditional pass (v_u + (v_c - v_u) is v_c up to one rounding)
    lat1, v1 = m.step(dataclasses.replace(batch, cfg_scale=np.ones(B, np.float32)))
    _, v_c = m.step(dataclasses.replace(batch, cfg_scale=None))
    assert np.abs(v1 - v_c).max() <= 1e-5 * np.abs(v_c).max()


@pytest.mark.parametrize("exchange", ["fused", "allgather"])
def test_latent_parallel_local_group_bitwise(torch_cuda, exchange, monkeypatch):
    """Latent parallelism: rank 0 runs the conditional, rank 1 the
    unconditional pass, v exchanged per step; both ranks' latents_out equal the one-GPU CFG
    step bitwise (in-process 2-rank group on one GPU).  exchange "fused": the final GEMM's
    epilogue stores v into the peer's buffer + a device flag barrier (3 steps: the step-parity
    double buffer alternates); "allgather": the all-gather path."""
    import concurrent.futures as cf
    import torch
    from paper_2604_08123_b200 import dit as D
    monkeypatch.setenv("DIT_SP_NCCL", "0" if exchange == "fused" else "1")
    cfg = CFGS["d64_noqk"]
    B, hh, ww, nt = 2, 12, 12, 40
    ni = hh * ww
    batch = synth.make_batch(cfg, B, hh, ww, nt, n_adapters=1, cfg_scale=6.0)
    batch.adapter_id = np.array([-1, 0], dtype=np.int32)
    ref = _model(cfg, 2 * B, ni, nt, rank=8, adapters=1)
    ref.register_synthetic_lora(0, rank=8, index=0)
    lat1, v1 = ref.step(batch)
    group = D.load_library().dit_local_group_create(2)
    ms = []
    for r in range(2):
        m = _model(cfg, B, ni, nt, rank=8, adapters=1)
        m.register_synthetic_lora(0, rank=8, index=0)
        m.lp_init_local(group, r)
        ms.append(m)
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]

    def run(r):
        with torch.cuda.stream(streams[r]):
            return ms[r].step(batch, lp_rank=r, sync=False)

    for _ in range(3 if exchange == "fused" else 1):
        with cf.ThreadPoolExecutor(2) as ex:
            outs = list(ex.map(run, range(2)))
        torch.cuda.synchronize()
        for m in ms:
            assert m.sp_exchange() == (2 if exchange == "fused" else 1)
        for out, v in outs:
            np.testing.assert_array_equal(v.cpu().numpy(), v1)
            np.testing.assert_array_equal(out.cpu().numpy(), lat1)
    W = O.weights_to_f64(synth.make_weights_bf16(cfg))
    x_o, v_o = S.dit_step(cfg, W, batch, {0: oracle_adapter(cfg, 8, 0)[0]})
    check(v1, v_o, "v")
    for m in ms:
        m.close()
    D.load_library().dit_local_group_destroy(group)


def test_sd3_medium_width_parity(torch_cuda):
    """SD3-medium width (D = 1536, 24 x 64 heads, no QK-norm), 2 joint blocks (the second
    context_pre_only), 48 x 48 latent grid (2304 tokens) + 333 text tokens, B = 1 with CFG 7."""
    cfg = dataclasses.replace(synth.SD3_MEDIUM, depth_double=2)
    hh = ww = 48
    nt = synth.SD3_TXT_TOKENS
    m = _model(cfg, 2, hh * ww, nt)
    batch = synth.make_batch(cfg, 1, hh, ww, nt, cfg_scale=7.0)
    lat, v = m.step(batch)
    W = O.weights_to_f64(synth.make_weights_bf16(cfg))
    x_o, v_o = S.dit_step(cfg, W, batch)
    check(v, v_o, "v")
    check(lat, x_o, "latents_out")


def test_sd3_and_cfg_error_paths(torch_cuda):
    from paper_2604_08123_b200 import dit as D
    cfg = synth.SD3_TINY   # 8 x 8 position table
    m = _model(cfg, 2, 64, 8)
    # CFG doubles the batch: 2 requests need 4 sequences > B_max 2
    with pytest.raises(D.DitError) as e:
        m.step(synth.make_batch(cfg, 2, 4, 4, 8, cfg_scale=3.0))
    assert e.value.code == D.CODES["DIT_EBATCH"]
    # grid larger than the position table
    m2 = _model(cfg, 1, 100, 8)
    with pytest.raises(D.DitError) as e:
        m2.step(synth.make_batch(cfg, 1, 10, 10, 8))
    assert e.value.code == D.CODES["DIT_ESHAPE"]
    # latent parallelism: world must be 2, and it needs cfg_scale
    with pytest.raises(D.DitError) as e:
        m.lp_init(3, 0, b"\0" * 128)
    assert e.value.code == D.CODES["DIT_EPARALLEL"]
    group = D.load_library().dit_local_group_create(2)
    m.lp_init_local(group, 0)
    with pytest.raises(D.DitError) as e:
        m.step(synth.make_batch(cfg, 1, 4, 4, 8))
    assert e.value.code == D.CODES["DIT_EINVAL"]
    with pytest.raises(D.DitError) as e:   # SP and LP are exclusive
        m.sp_init_local(D.load_library().dit_local_group_create(2), 0)
    assert e.value.code == D.CODES["DIT_EPARALLEL"]
    m.close()
    m2.close()
    D.load_library().dit_local_group_destroy(group)
    # SD3 config validation: no single blocks
    bad = dataclasses.replace(cfg, depth_single=1)
    with pytest.raises(D.DitError):
        _model(bad, 1, 16, 8)


@pytest.mark.parametrize("exchange", ["fused", "a2a"])
def test_sd3_cfg_with_sequence_parallel_bitwise(torch_cuda, exchange, monkeypatch):
    """CFG (2B sequences) under Ulysses SP at P = 2 (in-process group): bitwise = P = 1."""
    from tests.test_gpu_parity import _shard_step
    from paper_2604_08123_b200 import dit as D
    monkeypatch.setenv("DIT_SP_NCCL", "1" if exchange == "a2a" else "0")
    cfg = CFGS["d128"]
    B, hh, ww, nt, P = 2, 8, 8, 16, 2
    batch = synth.make_batch(cfg, B, hh, ww, nt, cfg_scale=4.0)
    ref = _model(cfg, 2 * B, hh * ww, nt)
    lat1, v1 = ref.step(batch)
    ref.close()
    group = D.load_library().dit_local_group_create(P)
    ms = []
    for r in range(P):
        m = _model(cfg, 2 * B, hh * ww, nt)
        m.sp_init_local(group, r)
        ms.append(m)
    # _shard_step shards latents / txt per rank; CFG needs both prompts' rows per rank
    both = dataclasses.replace(batch, txt=np.concatenate([batch.txt, batch.txt_neg]),
                               pooled=np.concatenate([batch.pooled, batch.pooled_neg]))
    latP, vP = _shard_step(ms, both, P, cfg_scale=batch.cfg_scale)
    np.testing.assert_array_equal(vP, v1)
    np.testing.assert_array_equal(latP, lat1)
    for m in ms:
        m.close()
    D.load_library().dit_local_group_destroy(group)


def test_sd35_large_width_parity(torch_cuda):
    """SD3.5-Large width (D = 2432 = 9.5 GEMM tiles, 38 x 64 heads, QK-RMSNorm), 2 joint blocks,
    32 x 32 latent grid + 333 text tokens, B = 1 with CFG 3.5, a rank-16 LoRA."""
    cfg = dataclasses.replace(synth.SD35_LARGE, depth_double=2)
    hh = ww = 32
    nt = synth.SD3_TXT_TOKENS
    m = _model(cfg, 2, hh * ww, nt, rank=16, adapters=1)
    m.register_synthetic_lora(3, rank=16, index=0, scale=0.5)
    batch = synth.make_batch(cfg, 1, hh, ww, nt, cfg_scale=3.5)
    batch.adapter_id = np.array([3], dtype=np.int32)
    lat, v = m.step(batch)
    W = O.weights_to_f64(synth.make_weights_bf16(cfg))
    x_o, v_o = S.dit_step(cfg, W, batch, {3: oracle_adapter(cfg, 16, 0, scale=0.5)[0]})
    check(v, v_o, "v")
    check(lat, x_o, "latents_out")
