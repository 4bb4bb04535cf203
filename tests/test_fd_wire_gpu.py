"""GPU placement parity of the Flash Decode exchange (SURVEY §8(c) item 4,
flash_decode.hpp:353-370): every source's [m | l | o] wire row in every
rank's inbox against the CPU oracle's partial of that source's shard
(tf_oracle.c restates attention_partial + serialize_partial,
tilemath.hpp:145-181, 244-258), and the BSP stages exposed through the C
ABI (tf_fd_partial_async / tf_fd_combine_async) bitwise equal to the fused
schedule's rows and output.

A wire row is a (max, normalizer, unnormalised sum) triple: a kernel whose
running max differs in the last bit represents the same partial with l and
o scaled by exp(m - m_ref).  Rows are compared after that rescale: m to
1e-6 relative, l to 1e-6 (fp32 path) / the bf16 path's bar, o normalised by
the source's max |o|."""
import ctypes as C

import numpy as np
import pytest
import torch

import paper_2511_02168_b200 as tf
from paper_2511_02168_b200 import _abi

import _tol  # noqa: E402  (tests/_tol.py)

pytestmark = pytest.mark.gpu
V = tf.fd.Variant


def _rows_close(got, want, o_tol):
    """got, want: H x (d+2) wire rows of one source."""
    m, l, o = got[:, 0].astype(np.float64), got[:, 1].astype(np.float64), got[:, 2:].astype(np.float64)
    mr, lr, orf = want[:, 0].astype(np.float64), want[:, 1].astype(np.float64), want[:, 2:].astype(np.float64)
    assert np.all(np.abs(m - mr) <= 1e-6 * np.maximum(1.0, np.abs(mr))), (m, mr)
    s = np.exp(m - mr)[:, None]
    assert np.all(np.abs(l * s[:, 0] - lr) <= max(1e-6, o_tol) * lr), (l, lr)
    scale = np.abs(orf).max(axis=1, keepdims=True)
    assert float((np.abs(o * s - orf) / scale).max()) <= o_tol


@pytest.mark.parametrize("w", [2, 4])
def test_inbox_rows_are_oracle_partials_fp32(oracle, w):
    # The reference's own shape class: MHA, fp32, every source's row in
    # every rank's inbox is that source's attention_partial.
    p = tf.fd.make_problem(21 + w, 4, 16, 64 * w)
    ln = p.kv_len // w
    for variant in (V.kFused, V.kFineWaits):
        run = tf.fd.run_fd(p, variant, tf.WorldConfig(world_size=w))
        for s in range(w):
            want = oracle.partial_wire(p.q[0], np.ascontiguousarray(p.k[0, :, s * ln:(s + 1) * ln]),
                                       np.ascontiguousarray(p.v[0, :, s * ln:(s + 1) * ln]), p.scale)
            for r in range(w):
                _rows_close(run.inbox[r][s, 0], want, 2e-6)


@pytest.mark.parametrize("w", [1, 2])
def test_inbox_rows_are_oracle_partials_bf16_gqa(oracle, w):
    # The tensor-core path at the BASELINE head shape (64 q / 8 kv heads,
    # d = 128, bf16 K/V): source s's row of q-head g*8 + j is the oracle's
    # partial of the (b, j) restatement over s's shard.
    Hq, Hkv, d, L = 64, 8, 128, 2048 * w
    p = tf.fd.make_problem(31 + w, Hq, d, L)
    p.kv_heads = Hkv
    p.q, _ = oracle.round_bf16(p.q)
    p.k, _ = oracle.round_bf16(np.ascontiguousarray(p.k[:, :Hkv]))
    p.v, _ = oracle.round_bf16(np.ascontiguousarray(p.v[:, :Hkv]))
    run = tf.fd.run_fd(p, V.kFused, tf.WorldConfig(world_size=w), dtype=1, out_dtype=0)
    ln, gs = L // w, Hq // Hkv
    for s in range(w):
        ks = np.ascontiguousarray(p.k[0, :, s * ln:(s + 1) * ln])
        vs = np.ascontiguousarray(p.v[0, :, s * ln:(s + 1) * ln])
        for j in range(gs):
            want = oracle.partial_wire(np.ascontiguousarray(p.q[0, j::gs]), ks, vs, p.scale)
            for r in range(w):
                _rows_close(run.inbox[r][s, 0, j::gs], want, _tol.FD_F32)


def test_partial_and_combine_abi_match_the_fused_schedule():
    # tf_fd_partial_async rows == the rows the fused schedule exchanges;
    # tf_fd_combine_async of their all-gather == the fused output, bitwise.
    W, B, Hq, Hkv, d, L = 2, 2, 64, 8, 128, 4096
    g = torch.Generator(device="cuda").manual_seed(5)
    q = (torch.rand(B, Hq, d, device="cuda", generator=g) * 2 - 1).bfloat16()
    k = (torch.rand(B, Hkv, L, d, device="cuda", generator=g) * 2 - 1).bfloat16()
    v = (torch.rand(B, Hkv, L, d, device="cuda", generator=g) * 2 - 1).bfloat16()
    ln = L // W
    ks = [k[:, :, r * ln:(r + 1) * ln].contiguous() for r in range(W)]
    vs = [v[:, :, r * ln:(r + 1) * ln].contiguous() for r in range(W)]
    row = B * Hq * (d + 2)
    torch.cuda.synchronize()
    with tf.World(W, [0] * W, 256 << 20) as w:
        for out_dtype, tdt in ((_abi.TF_BF16, torch.bfloat16), (_abi.TF_F32, torch.float32)):
            shape = _abi.FdShape(B, Hq, Hkv, d, L, d ** -0.5, _abi.TF_BF16, out_dtype)
            inbox = w.alloc(f"t.inbox.{out_dtype}", 4 * W * row)
            outs = [torch.empty(B, Hq, d, device="cuda", dtype=tdt) for _ in range(W)]
            qp = _abi.ptr_array([q.data_ptr()] * W)
            kp = _abi.ptr_array([t.data_ptr() for t in ks])
            vp = _abi.ptr_array([t.data_ptr() for t in vs])
            _abi.check(w.lib.tf_flash_decode(w.handle, _abi.TF_FD_FUSED, C.byref(shape), qp, kp, vp,
                                             _abi.ptr_array([o.data_ptr() for o in outs]), _abi.ptr_array(inbox),
                                             None))
            rows = [torch.empty(row, device="cuda", dtype=torch.float32) for _ in range(W)]
            _abi.check(w.lib.tf_fd_partial_async(w.handle, C.byref(shape), qp, kp, vp,
                                                 _abi.ptr_array([t.data_ptr() for t in rows]), None))
            _abi.check(w.lib.tf_world_sync(w.handle))
            fused_rows = w.get(inbox[0], (W, row), np.float32)
            for r in range(W):
                assert np.array_equal(rows[r].cpu().numpy().view(np.uint32), fused_rows[r].view(np.uint32)), r
            gathered = torch.cat(rows)  # the all-gather
            gath = [gathered.clone() for _ in range(W)]
            outc = [torch.empty_like(o) for o in outs]
            _abi.check(w.lib.tf_fd_combine_async(w.handle, C.byref(shape), _abi.ptr_array([t.data_ptr() for t in gath]),
                                                 _abi.ptr_array([o.data_ptr() for o in outc]), None))
            _abi.check(w.lib.tf_world_sync(w.handle))
            for r in range(W):
                assert torch.equal(outc[r], outs[r]), (out_dtype, r)


def test_pull_gathered_operand_is_the_logical_a(oracle):
    # tf_ag_gathered after PULL: the inbox the gather warps filled plus the
    # own shard read in place -- bit for bit the logical A (ag_gemm_test.cpp:
    # 113-169's placement check, now also for the fused pull schedule).
    for w in (2, 4):
        p = tf.ag.make_problem(40 + w, 256, 256, 64 * 2 * w)
        p.a, _ = oracle.round_bf16(p.a)
        p.b, _ = oracle.round_bf16(p.b)
        run = tf.ag.run_pull(p, tf.WorldConfig(world_size=w), dtype=1)
        assert len(run.gathered) == w
        for g_ in run.gathered:
            assert np.array_equal(g_.view(np.uint32), p.a.view(np.uint32))
    # fp32 PULL stages nothing: its operand is read in place from the shards.
    p = tf.ag.make_problem(7, 13, 9, 16)
    run = tf.ag.run_pull(p, tf.WorldConfig(world_size=4))
    for g_ in run.gathered:
        assert np.array_equal(g_.view(np.uint32), p.a.view(np.uint32))
