"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle.

Tolerance (BASELINE.json north_star): per output tensor per request
max|G - O| / max|O| <= 2e-2 and cosine >= 0.999 (reading C16).  Integer
artefacts (segment tables, shard map) are bit-exact.
"""
import dataclasses

import numpy as np
import pytest

import synth
from oracle import flux_step as O
from tests.helpers import cosine, max_rel, oracle_adapter, residuals

pytestmark = pytest.mark.gpu

TOL_REL, TOL_COS = 2e-2, 0.999


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return torch


def check(g, o, what=""):
    import json
    import os
    log = os.environ.get("PARITY_LOG")
    for b in range(o.shape[0]):
        r, c = max_rel(g[b], o[b]), cosine(g[b], o[b])
        if log:
            with open(log, "a") as f:
                f.write(json.dumps({"test": os.environ.get("PYTEST_CURRENT_TEST", "?").split(" ")[0], "what": what,
                                    "request": b, "max_rel": r, "cos": c}) + "\n")
        assert r <= TOL_REL and c >= TOL_COS, f"{what} request {b}: max_rel={r:.3e} cos={c:.6f}"


def _model(cfg, B, ni, nt, rank=0, adapters=0):
    from paper_2604_08123_b200 import SyntheticDiT
    return SyntheticDiT(cfg, max_batch=B, max_img_tokens=ni, max_txt_tokens=nt, max_rank=rank, max_adapters=adapters)


def test_device_generator_bitwise(torch_cuda):
    torch = torch_cuda
    from paper_2604_08123_b200.dit import fill_synthetic
    for spec in synth.weight_manifest(synth.TINY_SINGLE)[:12]:
        t = torch.empty(spec.shape, dtype=torch.bfloat16, device="cuda")
        fill_synthetic(t, 0, spec.tensor_id, spec.scale, spec.offset)
        got = t.cpu().view(torch.int16).numpy().view(np.uint16)
        np.testing.assert_array_equal(got, synth.tensor_bf16_bits(spec))
    t = torch.empty(1 << 20, dtype=torch.bfloat16, device="cuda")
    fill_synthetic(t, 3001, 77, 0.37, 1.0)
    np.testing.assert_array_equal(t.cpu().view(torch.int16).numpy().view(np.uint16),
                                  synth.counter_bf16_bits(3001, 77, 1 << 20, 0.37, 1.0))


@pytest.mark.parametrize("cfg_name", ["TINY", "TINY_SINGLE"])
def test_tiny_step_parity(torch_cuda, cfg_name):
    cfg = getattr(synth, cfg_name)
    m = _model(cfg, 2, 16, 8)
    batch = synth.make_batch(cfg, 2, 4, 4, 8)
    lat, v = m.step(batch)
    W = O.weights_to_f64(synth.make_weights_bf16(cfg))
    x_o, v_o = O.dit_step(cfg, W, batch)
    check(v, v_o, "v")
    check(lat, x_o, "latents_out")


def test_tiny_lora_controlnet_two_steps(torch_cuda):
    """T0 protocol: mixed adapters (rank 4, ids [0, -1]), ControlNet on block 0, 2 Euler steps with hand-off."""
    cfg = synth.TINY_SINGLE
    m = _model(cfg, 2, 16, 8, rank=4, adapters=1)
    m.register_synthetic_lora(0, rank=4, index=0, scale=1.0)
    ad, _ = oracle_adapter(cfg, 4, 0)
    W = O.weights_to_f64(synth.make_weights_bf16(cfg))
    batch = synth.make_batch(cfg, 2, 4, 4, 8, n_adapters=1)
    batch.adapter_id = np.array([0, -1], dtype=np.int32)
    sig = np.array([1.0, 0.75, 0.0], dtype=np.float32)
    res_bits = {0: {0: synth.controlnet_residual_bf16(0, 0, 16, cfg.hidden)}}
    res = {0: {0: O.bf16_to_f64(res_bits[0][0])}}
    x_o = batch.latents.astype(np.float64)
    for k in range(2):
        batch.sigma[:] = sig[k]
        batch.sigma_next[:] = sig[k + 1]
        lat, v = m.step(batch, controlnet=res_bits)
        ob = dataclasses.replace(batch, latents=x_o)
        x_o, v_o = O.dit_step(cfg, W, ob, {0: ad}, res, n_res=cfg.depth_double)
        check(v, v_o, f"v step {k}")
        check(lat, x_o, f"latents step {k}")
        batch.latents = lat          # hand-off: out(step k) -> in(step k+1)


def test_ragged_multi_tile(torch_cuda):
    """Several 128-row tiles with a ragged tail, odd grid, 3 requests, 2 adapters."""
    cfg = dataclasses.replace(synth.TINY_SINGLE, hidden=128, heads=4, depth_single=1)
    m = _model(cfg, 3, 150, 40, rank=8, adapters=2)
    for a in range(2):
        m.register_synthetic_lora(10 + a, rank=8, index=a, scale=0.5 + a)
    batch = synth.make_batch(cfg, 3, 10, 15, 40, n_adapters=2)
    batch.adapter_id = np.array([11, -1, 10], dtype=np.int32)
    lat, v = m.step(batch)
    W = O.weights_to_f64(synth.make_weights_bf16(cfg))
    ads = {10 + a: oracle_adapter(cfg, 8, a, scale=0.5 + a)[0] for a in range(2)}
    x_o, v_o = O.dit_step(cfg, W, batch, ads)
    check(v, v_o, "v")
    check(lat, x_o, "latents")


def test_batch_invariance_bitwise(torch_cuda):
    """P3/P9 on GPU: a request's output does not depend on its batch-mates (bitwise)."""
    cfg = dataclasses.replace(synth.TINY_SINGLE, hidden=128, heads=4)
    m = _model(cfg, 3, 256, 128, rank=8, adapters=2)
    m.register_synthetic_lora(0, rank=8, index=0)
    m.register_synthetic_lora(1, rank=8, index=1)
    full = synth.make_batch(cfg, 3, 16, 16, 128, n_adapters=2)
    full.adapter_id = np.array([1, -1, 0], dtype=np.int32)
    _, v = m.step(full)
    for b in range(3):
        one = dataclasses.replace(full, latents=full.latents[b:b + 1], txt=full.txt[b:b + 1],
                                  pooled=full.pooled[b:b + 1], sigma=full.sigma[b:b + 1],
                                  sigma_next=full.sigma_next[b:b + 1], guidance=full.guidance[b:b + 1],
                                  adapter_id=full.adapter_id[b:b + 1], cn_scale=full.cn_scale[b:b + 1])
        _, v1 = m.step(one)
        np.testing.assert_array_equal(v1[0], v[b])


D128 = dataclasses.replace(synth.TINY_SINGLE, hidden=256, heads=2, rope_axes=(16, 56, 56), depth_single=1)


@pytest.mark.parametrize("grid,nt", [((10, 15), 40), ((32, 32), 256), ((4, 4), 8)])
def test_head_dim_128_tcgen05_attention(torch_cuda, grid, nt):
    """d = 128 routes attention to the tcgen05 kernel: ragged KV tails, many KV tiles, tiny N."""
    cfg = D128
    hh, ww = grid
    m = _model(cfg, 2, hh * ww, nt, rank=8, adapters=1)
    m.register_synthetic_lora(3, rank=8, index=0)
    batch = synth.make_batch(cfg, 2, hh, ww, nt, n_adapters=1)
    batch.adapter_id = np.array([-1, 3], dtype=np.int32)
    lat, v = m.step(batch)
    W = O.weights_to_f64(synth.make_weights_bf16(cfg))
    x_o, v_o = O.dit_step(cfg, W, batch, {3: oracle_adapter(cfg, 8, 0)[0]})
    check(v, v_o, "v")
    check(lat, x_o, "latents")


def _shard_step(models, batch, P, cfg_scale=None):
    """Run one dit_step on P in-process ranks (one host thread + stream each); gather v, latents."""
    import concurrent.futures as cf
    import torch
    from paper_2604_08123_b200.synthetic import _bits_to_bf16_tensor
    B, ni, nt = batch.batch, batch.img_tokens, batch.txt_tokens
    nil, ntl = ni // P, nt // P
    outs, vs, keep = [], [], []
    cbs, streams = [], []
    for r, m in enumerate(models):
        lat = torch.from_numpy(np.ascontiguousarray(batch.latents[:, r * nil:(r + 1) * nil])).to(m.dev)
        txt = _bits_to_bf16_tensor(np.ascontiguousarray(batch.txt[:, r * ntl:(r + 1) * ntl]), m.dev)
        pooled = _bits_to_bf16_tensor(batch.pooled, m.dev)
        out, v = torch.empty_like(lat), torch.empty_like(lat)
        keep += [lat, txt, pooled]
        outs.append(out)
        vs.append(v)
        cbs.append(m.make_batch(B, batch.img_h, batch.img_w, nt, batch.adapter_id, batch.sigma, batch.sigma_next,
                                batch.guidance, lat, out, txt, pooled, v_out=v, cn_scale=batch.cn_scale,
                                cfg_scale=cfg_scale))
        streams.append(torch.cuda.Stream())
    torch.cuda.synchronize()
    with cf.ThreadPoolExecutor(P) as ex:
        list(ex.map(lambda r: models[r].dit_step(cbs[r], stream=streams[r]), range(P)))
    torch.cuda.synchronize()
    v = np.concatenate([x.cpu().numpy() for x in vs], axis=1)
    lat = np.concatenate([x.cpu().numpy() for x in outs], axis=1)
    return lat, v


@pytest.mark.parametrize("exchange", ["fused", "a2a"])
@pytest.mark.parametrize("P,hidden,heads", [(2, 512, 4), (4, 512, 4), (2, 128, 4), (4, 128, 4)])
def test_sequence_parallel_local_group(torch_cuda, P, hidden, heads, exchange, monkeypatch):
    """Ulysses SP at P ranks (in-process group, one GPU): bitwise equal to P = 1 (pin P10) and oracle parity.

    hidden 512 / 4 heads -> d = 128 (tcgen05 attention); hidden 128 / 4 heads -> d = 32 (mma.sync kernel).
    exchange "fused": the QKV / attention epilogues store straight into the owning rank's buffers with
    device flag barriers (the default); "a2a": send buffers + all-to-all + gather/scatter kernels
    (DIT_SP_NCCL=1, the NCCL path's data layout).
    """
    from paper_2604_08123_b200 import dit as D
    monkeypatch.setenv("DIT_SP_NCCL", "1" if exchange == "a2a" else "0")
    d = hidden // heads
    cfg = dataclasses.replace(synth.TINY_SINGLE, hidden=hidden, heads=heads, depth_single=1,
                              rope_axes=(16, 56, 56) if d == 128 else (4, 14, 14))
    B, hh, ww, nt = 2, 16, 16, 64
    ref = _model(cfg, B, hh * ww, nt, rank=8, adapters=1)
    ref.register_synthetic_lora(5, rank=8, index=0)
    batch = synth.make_batch(cfg, B, hh, ww, nt, n_adapters=1)
    batch.adapter_id = np.array([5, -1], dtype=np.int32)
    lat1, v1 = ref.step(batch)
    group = D.load_library().dit_local_group_create(P)
    models = []
    for r in range(P):
        m = _model(cfg, B, hh * ww, nt, rank=8, adapters=1)
        m.register_synthetic_lora(5, rank=8, index=0)
        m.sp_init_local(group, r)
        models.append(m)
    latP, vP = _shard_step(models, batch, P)
    np.testing.assert_array_equal(vP, v1)
    np.testing.assert_array_equal(latP, lat1)
    W = O.weights_to_f64(synth.make_weights_bf16(cfg))
    x_o, v_o = O.dit_step(cfg, W, batch, {5: oracle_adapter(cfg, 8, 0)[0]})
    check(vP, v_o, "v")
    for m in models:
        m.close()
    D.load_library().dit_local_group_destroy(group)


@pytest.mark.parametrize("d", [128, 64])
@pytest.mark.parametrize("B,H,N", [(3, 70, 333), (1, 3, 129), (2, 150, 1000)])
def test_attention_kernel_vs_torch_fp32(torch_cuda, B, H, N, d):
    """tcgen05 attention alone (d = 128 Flux, d = 64 SD3) against a plain PyTorch fp32 reference:
    more work items than SMs (persistent CTAs walk several), ragged query blocks and KV tails."""
    import ctypes as C
    import torch
    from paper_2604_08123_b200 import dit
    lib = dit.load_library()
    g = torch.Generator(device="cuda").manual_seed(B * 1000 + H * 10 + N)
    q, k, v = (torch.randn(B, H, N, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    out = torch.zeros(B * N, H * d, device="cuda", dtype=torch.bfloat16)
    s = torch.cuda.current_stream()
    assert lib.dit_debug_attention(q.data_ptr(), k.data_ptr(), v.data_ptr(), B, H, N, d, out.data_ptr(),
                                   C.c_void_p(s.cuda_stream)) == 0
    torch.cuda.synchronize()
    qf, kf, vf = q.float(), k.float(), v.float()
    p = torch.softmax((qf @ kf.transpose(-1, -2)) / d ** 0.5, dim=-1)
    ref = (p @ vf).permute(0, 2, 1, 3).reshape(B * N, H * d)
    got = out.float()
    err = ((got - ref).abs().max() / ref.abs().max()).item()
    cos = torch.nn.functional.cosine_similarity(got.flatten(), ref.flatten(), dim=0).item()
    # bf16 P and O (2^-9 relative rounding) bound the error; every row must be written
    assert torch.isfinite(got).all()
    assert err < 1e-2, err
    assert cos > 0.9999, cos


def test_single_block_controlnet_and_fan_in(torch_cuda):
    """SURVEY.md §8(f) f4 (reading C20): ControlNet residuals on single blocks (image rows of the
    joint sequence) and two ControlNets feeding the same blocks (summed), vs the oracle."""
    from oracle.flux_step import ControlNetInput
    cfg = synth.TINY_SINGLE
    m = _model(cfg, 2, 16, 8)
    batch = synth.make_batch(cfg, 2, 4, 4, 8, n_adapters=0)
    batch.adapter_id = np.array([-1, -1], dtype=np.int32)
    batch.cn_scale = np.array([0.9, 1.3], dtype=np.float32)
    ni, D, Ld = batch.img_tokens, cfg.hidden, cfg.depth_double
    bits = lambda b, i: synth.controlnet_residual_bf16(b, i, ni, D)
    f64 = lambda x: O.bf16_to_f64(x)
    inj, cns = [], {}
    for b in range(2):
        # ControlNet A: double block 0 and single blocks 0, 1; ControlNet B: double 0 and single 1
        A = ControlNetInput(double={0: f64(bits(b, 0))}, single={0: f64(bits(b, 1)), 1: f64(bits(b, 2))},
                            n_res=1, n_res_single=2, scale=0.6)
        Bc = ControlNetInput(double={0: f64(bits(b, 3))}, single={1: f64(bits(b, 4))},
                             n_res=1, n_res_single=2, scale=-0.5)
        cns[b] = [A, Bc]
        inj += [(b, 0, bits(b, 0), 0.6), (b, Ld + 0, bits(b, 1), 0.6), (b, Ld + 1, bits(b, 2), 0.6),
                (b, 0, bits(b, 3), -0.5), (b, Ld + 1, bits(b, 4), -0.5)]
    lat, v = m.step(batch, injections=inj)
    W = O.weights_to_f64(synth.make_weights_bf16(cfg))
    x_o, v_o = O.dit_step(cfg, W, batch, controlnets=cns)
    check(v, v_o, "v")
    check(lat, x_o, "latents")
    _, v0 = O.dit_step(cfg, W, batch)
    assert max_rel(v_o, v0) > 1e-2                 # the residuals matter at this scale


def test_controlnet_inject_limits(torch_cuda):
    import torch
    from paper_2604_08123_b200.dit import DitError
    cfg = synth.TINY_SINGLE
    m = _model(cfg, 2, 16, 8)
    r = torch.zeros(16, cfg.hidden, dtype=torch.bfloat16, device="cuda")
    blocks = cfg.depth_double + cfg.depth_single
    m.controlnet_inject(0, blocks - 1, r)                      # last single block: accepted
    m.controlnet_inject(0, blocks - 1, r)                      # second ControlNet (fan-in 2)
    with pytest.raises(DitError) as e:
        m.controlnet_inject(0, blocks - 1, r)                  # a third: DIT_ENOSPC
    assert e.value.code == 6
    with pytest.raises(DitError) as e:
        m.controlnet_inject(0, blocks, r)                      # past the last block: DIT_EINVAL
    assert e.value.code == 1


def test_controlnet_device_flag_deferred_fetch(torch_cuda):
    """SURVEY.md §8(f) f2, consumer side: a residual published by a device flag.
    A producer on another stream writes the residual ~3 ms AFTER the step is enqueued (no event,
    no host sync); the consuming epilogue must acquire the flag and see the data: the result equals,
    bit for bit, the step with the residual resident from the start."""
    import ctypes as C
    import torch
    from paper_2604_08123_b200.synthetic import _bits_to_bf16_tensor
    cfg = synth.TINY_SINGLE
    m = _model(cfg, 2, 16, 8)
    batch = synth.make_batch(cfg, 2, 4, 4, 8, n_adapters=0)
    batch.adapter_id = np.array([-1, -1], dtype=np.int32)
    ni, D, Ld = batch.img_tokens, cfg.hidden, cfg.depth_double
    src = [_bits_to_bf16_tensor(synth.controlnet_residual_bf16(b, 7, ni, D), "cuda") for b in range(2)]
    # reference: residuals resident (request 0 on double block 0, request 1 on single block 1)
    ref_lat, ref_v = m.step(batch, injections=[(0, 0, synth.controlnet_residual_bf16(0, 7, ni, D), 0.8),
                                               (1, Ld + 1, synth.controlnet_residual_bf16(1, 7, ni, D), 0.8)])
    for delay_ns in (3_000_000, 0):
        dst = [torch.full_like(s, 1000.0) for s in src]        # garbage until published
        flag = torch.zeros(4, dtype=torch.int32, device="cuda")
        side = torch.cuda.Stream()
        torch.cuda.synchronize()
        for b in range(2):
            assert m.lib.dit_debug_delayed_publish(dst[b].data_ptr(), src[b].data_ptr(), src[b].numel() * 2,
                                                   C.c_void_p(flag.data_ptr() + 4 * b), 5, delay_ns,
                                                   C.c_void_p(side.cuda_stream)) == 0
        m.controlnet_inject_flag(0, 0, dst[0], flag[0:1], 5, scale=0.8)
        m.controlnet_inject_flag(1, Ld + 1, dst[1], flag[1:2], 5, scale=0.8)
        lat, v = m.step(batch)
        np.testing.assert_array_equal(v, ref_v)
        np.testing.assert_array_equal(lat, ref_lat)


@pytest.mark.parametrize("M,N,K", [(300, 520, 192), (4096, 3072, 3072), (1000, 21504, 64)])
def test_debug_gemm_vs_torch_fp32(torch_cuda, M, N, K):
    """The step's tcgen05 GEMM alone (dit_debug_gemm, EPI_BIAS) against a PyTorch fp32 matmul:
    ragged M / N tails, a single K block, a Flux-size projection."""
    import ctypes as C
    import torch
    from paper_2604_08123_b200 import dit
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    x = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn(N, K, device="cuda", generator=g) * K ** -0.5).to(torch.bfloat16)
    bias = torch.randn(N, device="cuda", generator=g).to(torch.bfloat16)
    y = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
    s = torch.cuda.current_stream()
    assert dit.load_library().dit_debug_gemm(x.data_ptr(), w.data_ptr(), bias.data_ptr(), y.data_ptr(), M, N, K,
                                             C.c_void_p(s.cuda_stream)) == 0
    torch.cuda.synchronize()
    ref = x.float() @ w.float().T + bias.float()
    err = ((y.float() - ref).abs().max() / ref.abs().max()).item()
    assert err < 8e-3, err
