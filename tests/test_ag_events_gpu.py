"""GPU: the reference's protocol-safety and overlap witnesses
(ag_gemm_test.cpp:175-244) from the device event log (tf_world_set_events /
tf_ag_events): for every remote (m-block, source) chunk of every rank, the
consumer's first load is stamped after the chunk's store (no inbox block is
read before its owner's store), and in some rank a consumer loads a chunk
before the last chunk is stored (the exchange overlaps the GEMM instead of
completing first, as a bulk-synchronous schedule would)."""
import ctypes as C

import numpy as np
import pytest

import paper_2511_02168_b200 as tf
from paper_2511_02168_b200 import _abi

pytestmark = pytest.mark.gpu
NONE = np.uint64(0xFFFFFFFFFFFFFFFF)


@pytest.mark.parametrize("variant", [_abi.TF_AG_PULL, _abi.TF_AG_PUSH])
def test_safety_and_overlap_witnesses(variant):
    import torch
    W, m, n, k = 4, 2048, 2048, 1024
    kw = k // W
    num_m = m // 128
    g = torch.Generator(device="cuda").manual_seed(11)
    A = (torch.rand(m, k, device="cuda", generator=g) * 2 - 1).bfloat16()
    B = (torch.rand(k, n, device="cuda", generator=g) * 2 - 1).bfloat16()
    Cs = [torch.empty(m, n, device="cuda", dtype=torch.bfloat16) for _ in range(W)]
    torch.cuda.synchronize()
    with tf.World(W, [0] * W, m * kw * 2 + 2 * 2 * m * k * 2 + (64 << 20)) as w:
        sh = w.alloc("ag.a", m * kw * 2)
        for r in range(W):
            s = A[:, r * kw:(r + 1) * kw].contiguous()
            w.memcpy(sh[r], s.data_ptr(), s.numel() * 2)
        _abi.check(w.lib.tf_world_set_events(w.handle, 1))
        shape = _abi.AgShape(m, n, k, 0, 0, 0, _abi.TF_BF16)
        _abi.check(w.lib.tf_ag_gemm(w.handle, variant, C.byref(shape), _abi.ptr_array(sh),
                                    _abi.ptr_array([B.data_ptr()] * W), _abi.ptr_array([c.data_ptr() for c in Cs]),
                                    None, None))
        ref = A.float() @ B.float()
        for c in Cs:
            assert float((c.float() - ref).abs().max() / ref.abs().max()) <= 4e-3
        stores, loads = [], []
        for r in range(W):
            cnt = C.c_size_t()
            _abi.check(w.lib.tf_ag_events(w.handle, r, None, 0, C.byref(cnt)))
            assert cnt.value == num_m * W * 2
            buf = (C.c_uint64 * cnt.value)()
            _abi.check(w.lib.tf_ag_events(w.handle, r, buf, cnt.value, C.byref(cnt)))
            ev = np.frombuffer(buf, dtype=np.uint64).reshape(num_m, W, 2)
            for mb in range(num_m):
                for src in range(W):
                    if src == r:
                        continue  # the rank's own shard: no exchange
                    st, ld = ev[mb, src]
                    assert st != NONE and ld != NONE, (r, mb, src)
                    assert ld >= st, (r, mb, src, int(st), int(ld))  # safety: read after the owner's store
                    stores.append(int(st))
                    loads.append(int(ld))
        # overlap witness: the first consumer load precedes the last store
        assert min(loads) < max(stores)
        _abi.check(w.lib.tf_world_set_events(w.handle, 0))


def test_fd_fused_safety_and_overlap_witnesses():
    """flash_decode_test.cpp:200-247 on the device: every (source, group) row
    set is folded only after its source released it, and some fold starts
    before the last push -- the exchange overlaps the attention compute."""
    import torch
    W, B, Hq, Hkv, d, L = 4, 16, 64, 8, 128, 8192
    G = B * Hkv
    g = torch.Generator(device="cuda").manual_seed(12)
    q = (torch.rand(B, Hq, d, device="cuda", generator=g) * 2 - 1).bfloat16()
    k = (torch.rand(B, Hkv, L, d, device="cuda", generator=g) * 2 - 1).bfloat16()
    v = (torch.rand(B, Hkv, L, d, device="cuda", generator=g) * 2 - 1).bfloat16()
    ln = L // W
    ks = [k[:, :, r * ln:(r + 1) * ln].contiguous() for r in range(W)]
    vs = [v[:, :, r * ln:(r + 1) * ln].contiguous() for r in range(W)]
    outs = [torch.empty(B, Hq, d, device="cuda", dtype=torch.bfloat16) for _ in range(W)]
    torch.cuda.synchronize()
    with tf.World(W, [0] * W, 256 << 20) as w:
        _abi.check(w.lib.tf_world_set_events(w.handle, 1))
        shape = _abi.FdShape(B, Hq, Hkv, d, L, d ** -0.5, _abi.TF_BF16, _abi.TF_BF16)
        _abi.check(w.lib.tf_flash_decode(w.handle, _abi.TF_FD_FUSED, C.byref(shape), _abi.ptr_array([q.data_ptr()] * W),
                                         _abi.ptr_array([x.data_ptr() for x in ks]),
                                         _abi.ptr_array([x.data_ptr() for x in vs]),
                                         _abi.ptr_array([o.data_ptr() for o in outs]), None, None))
        for o in outs[1:]:
            assert torch.equal(o, outs[0])
        stores, loads = [], []
        for r in range(W):
            cnt = C.c_size_t()
            _abi.check(w.lib.tf_fd_events(w.handle, r, None, 0, C.byref(cnt)))
            assert cnt.value == W * G * 2
            buf = (C.c_uint64 * cnt.value)()
            _abi.check(w.lib.tf_fd_events(w.handle, r, buf, cnt.value, C.byref(cnt)))
            ev = np.frombuffer(buf, dtype=np.uint64).reshape(W, G, 2)
            for src in range(W):
                for grp in range(G):
                    st, ld = ev[src, grp]
                    assert st != NONE and ld != NONE, (r, src, grp)
                    assert ld >= st, (r, src, grp)
                    stores.append(int(st))
                    loads.append(int(ld))
        assert min(loads) < max(stores)
