"""N > 1 host logic on CPU: the Ulysses SP layouts at world size 2 over gloo.

Each rank builds integer-coded q/k/v for its LOCAL tokens, lays them out with
the library's own index maps (dit_sp_layout = the functions the CUDA kernels
use), exchanges them with a real all_to_all over gloo, and checks bit-exactly
that (1) every rank ends up with the FULL sequence of its heads in global
[txt; img] order (a2a #1 + gather), and (2) attention outputs return to the
token owners in the stream-split row order the projection GEMM reads
(a2a #2 + scatter).  The expected layouts are written here independently from
DESIGN.md §6, not from the library.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _code(sec, b, head, n, B, H, N):
    return ((sec * B + b) * H + head) * N + n


def _worker(rank, world, port, B, H, Nt, Ni, errq):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2604_08123_b200 import dit
        N = Nt + Ni
        nt, ni = Nt // world, Ni // world
        nloc, Hl = nt + ni, H // world

        def grow(r, i):          # txt slice then img slice, global txt-first order
            return r * nt + i if i < nt else Nt + r * ni + (i - nt)

        # shard map
        sm = dit.sp_layout(0, world, rank, B, H, Nt, Ni)
        exp = np.array([b * N + grow(rank, i) for b in range(B) for i in range(nloc)])
        np.testing.assert_array_equal(sm, exp)

        # a2a #1: local q/k/v -> my heads, full sequence
        codes = np.array([_code(sec, b, h, grow(rank, i), B, H, N)
                          for sec in range(3) for b in range(B) for h in range(H) for i in range(nloc)])
        send_idx = dit.sp_layout(1, world, rank, B, H, Nt, Ni)
        send = np.full(world * 3 * B * Hl * nloc, -1, dtype=np.int64)
        send[send_idx] = codes
        assert (send >= 0).all()
        recv = torch.empty(send.size, dtype=torch.int64)
        dist.all_to_all_single(recv, torch.from_numpy(send))
        gidx = dit.sp_layout(2, world, rank, B, H, Nt, Ni)
        attn = np.full(3 * B * Hl * N, -1, dtype=np.int64)
        attn[gidx] = recv.numpy()
        exp_attn = np.array([_code(sec, b, rank * Hl + hl, n, B, H, N)
                             for sec in range(3) for b in range(B) for hl in range(Hl) for n in range(N)])
        np.testing.assert_array_equal(attn, exp_attn)

        # a2a #2: "attention" = identity on q: O[b][n][hl] -> owners, stream-split local rows
        rows = dit.sp_layout(3, world, rank, B, H, Nt, Ni)
        send2 = np.full(world * B * nloc * Hl, -1, dtype=np.int64)
        k = 0
        for b in range(B):
            for n in range(N):
                for hl in range(Hl):
                    send2[rows[k] * Hl + hl] = _code(0, b, rank * Hl + hl, n, B, H, N)
                    k += 1
        recv2 = torch.empty(send2.size, dtype=torch.int64)
        dist.all_to_all_single(recv2, torch.from_numpy(send2))
        srows = dit.sp_layout(4, world, rank, B, H, Nt, Ni)
        out = np.full((B * nloc, H), -1, dtype=np.int64)
        r2 = recv2.numpy().reshape(world * B * nloc, Hl)
        for j, lr in enumerate(srows):
            rs = j // (B * nloc)
            out[lr, rs * Hl:(rs + 1) * Hl] = r2[j]
        exp_out = np.full((B * nloc, H), -1, dtype=np.int64)
        for b in range(B):
            for i in range(nloc):
                lr = b * nt + i if i < nt else B * nt + b * ni + (i - nt)
                exp_out[lr] = [_code(0, b, h, grow(rank, i), B, H, N) for h in range(H)]
        np.testing.assert_array_equal(out, exp_out)

        # fused exchange (the default at P > 1): the same codes stored one-sidedly at the
        # peer addresses the QKV / attention epilogues compute (dit_sp_layout 5 / 6); every
        # rank's puts are all-gathered and each rank keeps those addressed to it
        span = 3 * B * Hl * N
        dst = dit.sp_layout(5, world, rank, B, H, Nt, Ni)
        puts = [torch.empty(2 * codes.size, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(puts, torch.from_numpy(np.concatenate([dst, codes])))
        attn_f = np.full(span, -1, dtype=np.int64)
        for pr in puts:
            d_, c_ = pr.numpy()[:codes.size], pr.numpy()[codes.size:]
            mine = d_ // span == rank
            assert (attn_f[d_[mine] % span] == -1).all()           # every slot written once
            attn_f[d_[mine] % span] = c_[mine]
        np.testing.assert_array_equal(attn_f, exp_attn)
        odst = dit.sp_layout(6, world, rank, B, H, Nt, Ni)
        ocodes = np.array([_code(0, b, rank * Hl + hl, n, B, H, N)
                           for b in range(B) for n in range(N) for hl in range(Hl)])
        puts = [torch.empty(2 * ocodes.size, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(puts, torch.from_numpy(np.concatenate([odst, ocodes])))
        out_f = np.full(B * nloc * H, -1, dtype=np.int64)
        for pr in puts:
            d_, c_ = pr.numpy()[:ocodes.size], pr.numpy()[ocodes.size:]
            mine = d_ >> 40 == rank
            idx = d_[mine] & ((1 << 40) - 1)
            assert (out_f[idx] == -1).all()
            out_f[idx] = c_[mine]
        np.testing.assert_array_equal(out_f.reshape(B * nloc, H), exp_out)
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        errq.put(f"rank {rank}: {e}\n{traceback.format_exc()}")


@pytest.mark.parametrize("B,H,Nt,Ni", [(2, 4, 8, 16), (3, 24, 512, 4096 // 16)])
def test_sp_layouts_world2_gloo(B, H, Nt, Ni):
    ctx = mp.get_context("spawn")
    errq = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, B, H, Nt, Ni, errq)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, "\n".join(errs)
    assert all(p.exitcode == 0 for p in procs)


def test_sp_layout_rejects_unshardable():
    from paper_2604_08123_b200 import dit
    with pytest.raises(dit.DitError):
        dit.sp_layout(0, 3, 0, 1, 24, 512, 4096)    # 3 does not divide 512
