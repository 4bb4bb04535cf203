"""GPU parity: Flash Decode over a paged KV cache (tf_flash_decode_paged).

Paged KV is an extension (the reference's SPEC.md:327 lists it as a
non-goal); its contract is that a paged run is the contiguous run of the
same logical KV: same keys in the same order, so every schedule's output
and every wire row are bitwise those of tf_flash_decode -- which the
other FD tests pin to the oracle.  Pages are scattered by a seeded
permutation over a pool whose unused pages hold NaN (a stray read would
show), and the per-rank length is not a multiple of the page size."""
import numpy as np
import pytest

import paper_2511_02168_b200 as tf
from paper_2511_02168_b200 import _abi
import _tol  # noqa: E402  (tests/_tol.py)

pytestmark = pytest.mark.gpu
V = tf.fd.Variant
ALL = [V.kBsp, V.kIndependentAg, V.kFineWaits, V.kFused]


def same(a, b):
    return np.array_equal(np.asarray(a).view(np.uint32), np.asarray(b).view(np.uint32))


def gqa_problem(seed, batch, kv_len, heads=16, kv_heads=2, d=128):
    p = tf.fd.make_problem(seed, heads, d, kv_len)
    rng = np.random.default_rng(seed)
    p.batch, p.kv_heads = batch, kv_heads
    p.q = rng.uniform(-1, 1, (batch, heads, d)).astype(np.float32)
    p.k = rng.uniform(-1, 1, (batch, kv_heads, kv_len, d)).astype(np.float32)
    p.v = rng.uniform(-1, 1, (batch, kv_heads, kv_len, d)).astype(np.float32)
    return p


@pytest.mark.parametrize("W", [1, 2])
@pytest.mark.parametrize("page_size", [16, 64, 256])
@pytest.mark.parametrize("hnd", [False, True])
def test_paged_fp32_equals_contiguous_every_schedule(W, page_size, hnd, oracle):
    # fp32 K/V: the generic split kernel (any d; here the reference's MHA shape)
    p = tf.fd.make_problem(11, 4, 32, 2 * 600)  # 600 keys per rank at W = 2: ragged last page
    want = oracle.attention(p.q[0], p.k[0], p.v[0], p.scale)
    for variant in ALL:
        cfg = tf.WorldConfig(world_size=W)
        base = tf.fd.run_fd(p, variant, cfg)
        pg = tf.fd.run_fd(p, variant, cfg, paged=tf.fd.PagedLayout(page_size=page_size, seed=W, hnd=hnd))
        for r in range(W):
            assert same(pg.out[r], base.out[r]), (variant, W, page_size, r)
            assert same(pg.inbox[r], base.inbox[r]) or variant == V.kBsp, (variant, W, page_size, r)
        assert oracle.head_rel_err(pg.out[0], want) <= _tol.FD_F32_REF


@pytest.mark.parametrize("W", [1, 2])
@pytest.mark.parametrize("page_size", [16, 32, 128])
@pytest.mark.parametrize("hnd", [False, True])
def test_paged_bf16_tensor_core_equals_contiguous(W, page_size, hnd):
    # bf16 K/V, d = 128, 8 q-heads per KV head: the tensor-core split kernel
    p = gqa_problem(3, batch=3, kv_len=W * 1000, heads=16, kv_heads=2)
    lay = tf.fd.PagedLayout(page_size=page_size, spare_pages=7, seed=5, hnd=hnd)
    for variant in (V.kFused, V.kBsp, V.kFineWaits):
        for odt in (_abi.TF_BF16, _abi.TF_F32):
            cfg = tf.WorldConfig(world_size=W)
            base = tf.fd.run_fd(p, variant, cfg, dtype=_abi.TF_BF16, out_dtype=odt)
            pg = tf.fd.run_fd(p, variant, cfg, dtype=_abi.TF_BF16, out_dtype=odt, paged=lay)
            for r in range(W):
                assert same(pg.out[r], base.out[r]), (variant, W, page_size, odt, r)
            assert not np.isnan(pg.out[0]).any()


def test_paged_owner_combine_and_flags():
    p = gqa_problem(4, batch=2, kv_len=4 * 512, heads=16, kv_heads=2)
    cfg = tf.WorldConfig(world_size=4)
    opts = tf.fd.FdOptions(owner_combine=True)
    base = tf.fd.run_fused(p, cfg, opts, dtype=_abi.TF_BF16, out_dtype=_abi.TF_F32)
    pg = tf.fd.run_fused(p, cfg, opts, dtype=_abi.TF_BF16, out_dtype=_abi.TF_F32,
                         paged=tf.fd.PagedLayout(page_size=64, hnd=True))
    for r in range(4):
        assert same(pg.out[r], base.out[r]), r


def test_paged_bad_block_table_entry_is_a_shape_error():
    p = tf.fd.make_problem(2, 2, 16, 256)
    with pytest.raises(tf.ShapeError, match="outside the pool"):
        tf.fd.run_fused(p, tf.WorldConfig(world_size=1), paged=tf.fd.PagedLayout(page_size=16), bad_page=True)
    # the world recovers: a clean call afterwards succeeds
    run = tf.fd.run_fused(p, tf.WorldConfig(world_size=1), paged=tf.fd.PagedLayout(page_size=16))
    assert np.isfinite(run.out[0]).all()


def test_paged_layout_validation():
    p = tf.fd.make_problem(2, 2, 16, 256)
    with pytest.raises(tf.ConfigError, match="power of two"):
        tf.fd.run_fused(p, tf.WorldConfig(world_size=1), paged=tf.fd.PagedLayout(page_size=24))


@pytest.mark.parametrize("W", [1, 2])
@pytest.mark.parametrize("page_size", [64, 256])
@pytest.mark.parametrize("hnd", [False, True])
def test_paged_stream_kernel_equals_contiguous(monkeypatch, W, page_size, hnd):
    # TFB_FD_STREAM=1: the TMA-fed stream kernel for both runs (pages >= 64
    # keys: one TMA box per 64-key stage, HND as a 3-D map over the pool,
    # NHD as a 4-D one with the key rows Hkv * 256 B apart)
    monkeypatch.setenv("TFB_FD_STREAM", "1")
    p = gqa_problem(9, batch=3, kv_len=W * 1000, heads=16, kv_heads=2)
    lay = tf.fd.PagedLayout(page_size=page_size, spare_pages=5, seed=11, hnd=hnd)
    for variant in (V.kFused, V.kBsp):
        cfg = tf.WorldConfig(world_size=W)
        base = tf.fd.run_fd(p, variant, cfg, dtype=_abi.TF_BF16, out_dtype=_abi.TF_BF16)
        pg = tf.fd.run_fd(p, variant, cfg, dtype=_abi.TF_BF16, out_dtype=_abi.TF_BF16, paged=lay)
        for r in range(W):
            assert same(pg.out[r], base.out[r]), (variant, W, page_size, hnd, r)
        assert not np.isnan(pg.out[0]).any()
    # ... and a bad table entry is still a ShapeError from the stream kernel
    with pytest.raises(tf.ShapeError, match="outside the pool"):
        tf.fd.run_fused(p, tf.WorldConfig(world_size=1), dtype=_abi.TF_BF16, out_dtype=_abi.TF_BF16,
                        paged=tf.fd.PagedLayout(page_size=page_size, hnd=hnd), bad_page=True)
