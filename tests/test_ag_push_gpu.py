"""GPU parity: the AG+GEMM PUSH producers (ag_gemm.hpp:241-260).

The TMA-engine producer (`ag_push_tma_kernel`, default for W <= 8: TMA loads
of the shard, TMA stores into every peer inbox, the own block read in place)
and the register-copy producer (`ag_push_kernel`, TFB_PUSH_LSU) place the
same bytes and raise the same flags, so C is bitwise equal between them, the
gathered operand is the logical A bit for bit, and every (m-block, source)
flag is raised exactly once -- over box widths 64 / 128 / 256 columns,
ragged M, K- and M-sharded A, and a caller-supplied gathered buffer (the own
block is then stored too)."""
import ctypes as C

import numpy as np
import pytest

import paper_2511_02168_b200 as tf
from paper_2511_02168_b200 import _abi

pytestmark = pytest.mark.gpu
TOL = 4e-3


def bf16_problem(seed, m, n, k, oracle):
    p = tf.ag.make_problem(seed, m, n, k)
    p.a, _ = oracle.round_bf16(p.a)
    p.b, _ = oracle.round_bf16(p.b)
    return p


def same(a, b):
    return np.array_equal(np.asarray(a).view(np.uint32), np.asarray(b).view(np.uint32))


@pytest.mark.parametrize("w,m,n,k", [(2, 300, 256, 2 * 64),     # 64-column boxes, ragged M
                                     (2, 256, 512, 2 * 128),    # 128-column boxes
                                     (4, 384, 256, 4 * 512),    # 256-column boxes, 2 per row
                                     (8, 130, 264, 8 * 192),    # 64-column boxes, W = 8, ragged M / N
                                     (2, 300, 256, 2 * 512)])   # 64-row boxes: the last one wholly past M
def test_tma_and_register_producers_agree(oracle, monkeypatch, w, m, n, k):
    import torch
    p = bf16_problem(w * 100 + m, m, n, k, oracle)
    tma = tf.ag.run_push(p, tf.WorldConfig(world_size=w), dtype=1)
    monkeypatch.setenv("TFB_PUSH_LSU", "1")
    lsu = tf.ag.run_push(p, tf.WorldConfig(world_size=w), dtype=1)
    ref = (torch.from_numpy(p.a).double() @ torch.from_numpy(p.b).double()).float().numpy()
    for r in range(w):
        assert same(tma.c[r], lsu.c[r]), r
        assert same(tma.gathered[r], p.a), r
        assert tma.flag_counts[r] == [1] * len(tma.flag_counts[r]), r
        assert float(np.abs(tma.c[r] - ref).max() / np.abs(ref).max()) <= TOL


@pytest.mark.parametrize("w", [2, 4])
def test_m_sharded_push_producers_agree(oracle, monkeypatch, w):
    p = bf16_problem(7 + w, 128 * w * 2, 256, 512, oracle)
    tma = tf.ag.run_push(p, tf.WorldConfig(world_size=w), dtype=1, shard_m=True)
    monkeypatch.setenv("TFB_PUSH_LSU", "1")
    lsu = tf.ag.run_push(p, tf.WorldConfig(world_size=w), dtype=1, shard_m=True)
    for r in range(w):
        assert same(tma.c[r], lsu.c[r]), r
        assert same(tma.gathered[r], p.a), r


def test_push_into_caller_gathered_buffers(oracle):
    """A caller's gathered buffer gets the whole operand, own block included."""
    import torch
    W, m, n, k = 4, 256, 256, 4 * 256
    p = bf16_problem(41, m, n, k, oracle)
    kw = k // W
    with tf.World(W, [0] * W, 64 << 20) as w:
        shards = w.alloc("ag.a", m * kw * 2)
        A = torch.from_numpy(p.a).bfloat16()
        for r in range(W):
            s = A[:, r * kw:(r + 1) * kw].contiguous().cuda()
            w.memcpy(shards[r], s.data_ptr(), s.numel() * 2)
        B = [torch.from_numpy(p.b).bfloat16().cuda() for _ in range(W)]
        Cs = [torch.empty(m, n, dtype=torch.bfloat16, device="cuda") for _ in range(W)]
        G = [torch.full((m, k), float("nan"), dtype=torch.bfloat16, device="cuda") for _ in range(W)]
        torch.cuda.synchronize()
        w.barrier()
        shape = _abi.AgShape(m, n, k, 0, 0, 0, 1)
        for _ in range(2):  # twice: the caller buffers are not parity-buffered
            _abi.check(w.lib.tf_ag_gemm(w.handle, _abi.TF_AG_PUSH, C.byref(shape), _abi.ptr_array(shards),
                                        _abi.ptr_array([b.data_ptr() for b in B]),
                                        _abi.ptr_array([c.data_ptr() for c in Cs]),
                                        _abi.ptr_array([g.data_ptr() for g in G]), None))
        torch.cuda.synchronize()
        ref = (torch.from_numpy(p.a).double() @ torch.from_numpy(p.b).double()).float().numpy()
        for r in range(W):
            assert same(G[r].float().cpu().numpy(), p.a), r
            c = Cs[r].float().cpu().numpy()
            assert float(np.abs(c - ref).max() / np.abs(ref).max()) <= TOL, r
