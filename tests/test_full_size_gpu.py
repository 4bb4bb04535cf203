"""GPU parity at BASELINE.json's full sizes (configs 2-4), through the C ABI
on device-resident inputs, checked by size-independent properties:

* AG+GEMM config 2 (M=8192, K=8192, N=28672/W): sampled rows of C against an
  fp32 product of the same bf16 inputs (4e-3 normalised, the bf16 path's
  tolerance); at W=8 (a loopback world on one GPU, each rank its own TP
  column shard of B) every rank's gathered operand is bit-for-bit the
  logical A, push flags all read 1, pull and push agree bitwise.
* Flash Decode configs 3/4: against a torch fp32 attention of the same bf16
  q/K/V -- bf16 output within 2^-8 + 1e-4 (the output's own rounding plus
  the fp32-grade path, tests/_tol.py), fp32 output (hi/lo P on the tensor
  cores) within 1e-4,
  the reference's own fp32 bar at 128K; at W=8 every rank's
  output is bitwise identical and every flag reads 1.
"""
import ctypes as C

import pytest

import paper_2511_02168_b200 as tf
from paper_2511_02168_b200 import _abi
import _tol  # noqa: E402  (tests/_tol.py)

pytestmark = pytest.mark.gpu
M, K, N_TOTAL = 8192, 8192, 28672


def _ptrs(xs):
    return _abi.ptr_array([x if isinstance(x, int) else x.data_ptr() for x in xs])


def _rows_err(A, B, Cout, rows):
    ref = A[rows].float() @ B.float()
    return float(((Cout[rows].float() - ref).abs().max() / ref.abs().max()).item())


def test_ag_config2_single_gpu():
    import torch
    g = torch.Generator(device="cuda").manual_seed(2)
    A = (torch.rand(M, K, device="cuda", generator=g) * 2 - 1).bfloat16()
    B = (torch.rand(K, N_TOTAL, device="cuda", generator=g) * 2 - 1).bfloat16()
    Cout = torch.empty(M, N_TOTAL, device="cuda", dtype=torch.bfloat16)
    torch.cuda.synchronize()
    with tf.World(1, [0], M * K * 2 + (64 << 20)) as w:
        sh = w.alloc("ag.a", M * K * 2)
        w.memcpy(sh[0], A.data_ptr(), M * K * 2)
        shape = _abi.AgShape(M, N_TOTAL, K, 0, 0, 0, _abi.TF_BF16)
        _abi.check(w.lib.tf_ag_gemm(w.handle, _abi.TF_AG_PULL, C.byref(shape), _abi.ptr_array(sh),
                                    _ptrs([B]), _ptrs([Cout]), None, None))
    rows = torch.arange(0, M, M // 64, device="cuda")
    assert _rows_err(A, B, Cout, rows) <= 4e-3


def test_ag_config2_eight_ranks_loopback():
    import torch
    W = 8
    kw, n = K // W, N_TOTAL // W
    g = torch.Generator(device="cuda").manual_seed(3)
    A = (torch.rand(M, K, device="cuda", generator=g) * 2 - 1).bfloat16()
    Bfull = (torch.rand(K, N_TOTAL, device="cuda", generator=g) * 2 - 1).bfloat16()
    Bs = [Bfull[:, r * n:(r + 1) * n].contiguous() for r in range(W)]  # TP column shards
    rows = torch.arange(0, M, M // 32, device="cuda")
    heap = M * kw * 2 + 2 * M * K * 2 + (64 << 20)
    outs = {}
    torch.cuda.synchronize()
    with tf.World(W, [0] * W, heap) as w:
        sh = w.alloc("ag.a", M * kw * 2)
        for r in range(W):
            shard = A[:, r * kw:(r + 1) * kw].contiguous()
            w.memcpy(sh[r], shard.data_ptr(), M * kw * 2)
        shape = _abi.AgShape(M, n, K, 0, 0, 0, _abi.TF_BF16)
        for name, var in (("pull", _abi.TF_AG_PULL), ("push", _abi.TF_AG_PUSH)):
            Cs = [torch.empty(M, n, device="cuda", dtype=torch.bfloat16) for _ in range(W)]
            gath = [torch.empty(M, K, device="cuda", dtype=torch.bfloat16) for _ in range(W)]
            _abi.check(w.lib.tf_ag_gemm(w.handle, var, C.byref(shape), _abi.ptr_array(sh), _ptrs(Bs),
                                        _ptrs(Cs), _ptrs(gath), None))
            for r in range(W):
                # placement: the gathered operand is the logical A, bit for bit
                assert torch.equal(gath[r].view(torch.int16), A.view(torch.int16)), (name, r)
                assert _rows_err(A, Bs[r], Cs[r], rows) <= 4e-3, (name, r)
            if var == _abi.TF_AG_PUSH:
                for r in range(W):
                    cnt = C.c_size_t()
                    _abi.check(w.lib.tf_ag_flag_counts(w.handle, r, None, 0, C.byref(cnt)))
                    buf = (C.c_uint64 * cnt.value)()
                    _abi.check(w.lib.tf_ag_flag_counts(w.handle, r, buf, cnt.value, C.byref(cnt)))
                    assert list(buf) == [1] * cnt.value
            outs[name] = Cs
            del gath
        for r in range(W):
            assert torch.equal(outs["pull"][r], outs["push"][r]), r


def _attention_ref(q, k, v, scale):
    """torch fp32 GQA attention, one batch at a time: q [B][Hq][d],
    k/v [B][Hkv][L][d] -> [B][Hq][d]."""
    import torch
    B, Hq, d = q.shape
    Hkv = k.shape[1]
    gs = Hq // Hkv
    out = torch.empty(B, Hq, d, device=q.device)
    for b in range(B):
        qf = q[b].float().view(Hkv, gs, d)
        kf, vf = k[b].float(), v[b].float()
        s = torch.einsum("hgd,hld->hgl", qf, kf) * scale
        out[b] = torch.einsum("hgl,hld->hgd", torch.softmax(s, -1), vf).reshape(Hq, d)
    return out


def _head_err(out, ref):
    return float(((out.float() - ref).abs().amax(-1) / ref.abs().amax(-1)).max().item())


def _run_fd(w, W, variant, q, ks, vs, scale, out_dtype):
    import torch
    B, Hq, d = q.shape
    Hkv, ln = ks[0].shape[1], ks[0].shape[2]
    tdt = torch.bfloat16 if out_dtype == _abi.TF_BF16 else torch.float32
    outs = [torch.empty(B, Hq, d, device="cuda", dtype=tdt) for _ in range(W)]
    shape = _abi.FdShape(B, Hq, Hkv, d, ln * W, scale, _abi.TF_BF16, out_dtype)
    _abi.check(w.lib.tf_flash_decode(w.handle, variant, C.byref(shape), _ptrs([q] * W), _ptrs(ks), _ptrs(vs),
                                     _ptrs(outs), None, None))
    return outs


@pytest.mark.parametrize("W", [1, 8])
def test_fd_config3(W):
    import torch
    B, Hq, Hkv, d, L = 1, 64, 8, 128, 131072
    g = torch.Generator(device="cuda").manual_seed(4)
    q = (torch.rand(B, Hq, d, device="cuda", generator=g) * 2 - 1).bfloat16()
    k = (torch.rand(B, Hkv, L, d, device="cuda", generator=g) * 2 - 1).bfloat16()
    v = (torch.rand(B, Hkv, L, d, device="cuda", generator=g) * 2 - 1).bfloat16()
    scale = d ** -0.5
    ref = _attention_ref(q, k, v, scale)
    ln = L // W
    ks = [k[:, :, r * ln:(r + 1) * ln].contiguous() for r in range(W)]  # slice_shard
    vs = [v[:, :, r * ln:(r + 1) * ln].contiguous() for r in range(W)]
    torch.cuda.synchronize()
    with tf.World(W, [0] * W, 64 << 20) as w:
        for out_dtype, tol in ((_abi.TF_BF16, _tol.FD_BF16), (_abi.TF_F32, _tol.FD_F32)):
            outs = _run_fd(w, W, _abi.TF_FD_FUSED, q, ks, vs, scale, out_dtype)
            assert _head_err(outs[0], ref) <= tol, out_dtype
            for o in outs[1:]:
                assert torch.equal(o, outs[0])
            # the BSP and owner-combine schedules fold the same partial bits
            bsp = _run_fd(w, W, _abi.TF_FD_BSP, q, ks, vs, scale, out_dtype)
            assert torch.equal(bsp[0], outs[0])
            own = _run_fd(w, W, _abi.TF_FD_FUSED_OWNER, q, ks, vs, scale, out_dtype)
            for o in own:
                assert torch.equal(o, outs[0])
        if W > 1:
            cnt = C.c_size_t()
            _abi.check(w.lib.tf_fd_flag_counts(w.handle, 0, None, 0, C.byref(cnt)))
            buf = (C.c_uint64 * cnt.value)()
            _abi.check(w.lib.tf_fd_flag_counts(w.handle, 0, buf, cnt.value, C.byref(cnt)))
            assert list(buf) == [1] * W


def test_fd_config4_single_gpu():
    import torch
    B, Hq, Hkv, d, L = 32, 64, 8, 128, 32768
    g = torch.Generator(device="cuda").manual_seed(5)
    q = (torch.rand(B, Hq, d, device="cuda", generator=g) * 2 - 1).bfloat16()
    k = (torch.rand(B, Hkv, L, d, device="cuda", generator=g) * 2 - 1).bfloat16()
    v = (torch.rand(B, Hkv, L, d, device="cuda", generator=g) * 2 - 1).bfloat16()
    scale = d ** -0.5
    ref = _attention_ref(q, k, v, scale)
    torch.cuda.synchronize()
    with tf.World(1, [0], 64 << 20) as w:
        for out_dtype, tol in ((_abi.TF_BF16, _tol.FD_BF16), (_abi.TF_F32, _tol.FD_F32)):
            out = _run_fd(w, 1, _abi.TF_FD_FUSED, q, [k], [v], scale, out_dtype)[0]
            assert _head_err(out, ref) <= tol, out_dtype
