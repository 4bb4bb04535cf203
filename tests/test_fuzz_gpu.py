"""GPU: seeded random shapes through every schedule (a fuzz pass over the
kernels' edge handling -- ragged M/N tiles, split-K, tail slices, skinny
and wide M, odd world sizes, GQA groupings, short and ragged KV splits).
AG: bf16 vs an fp64 product (4e-3 normalised), fp32 bitwise vs the oracle's
reference::gemm; FD: fp32 head-relative error vs the oracle (1e-5) and
bitwise agreement of every schedule and rank.  TFB_FUZZ_SCALE=k runs k times
as many cases (the first ones are always the default set)."""
import os

import numpy as np
import pytest

import paper_2511_02168_b200 as tf
import _tol  # noqa: E402  (tests/_tol.py)

pytestmark = pytest.mark.gpu
V = tf.fd.Variant
SCALE = max(1, int(os.environ.get("TFB_FUZZ_SCALE", "1")))


def _ag_cases(n=14 * SCALE):
    rng = np.random.default_rng(2024)
    out = []
    for _ in range(n):
        w = int(rng.choice([1, 2, 3, 4, 8]))
        m = int(rng.choice([1, 7, 64, 129, 200, 256, 384, 640, 1024]))
        n_ = int(rng.choice([8, 24, 264, 512, 1032, 2048, 4104]))
        k = 64 * w * int(rng.choice([1, 2, 3, 5]))
        out.append((w, m, n_, k))
    return out


@pytest.mark.parametrize("w,m,n,k", _ag_cases())
def test_ag_bf16_random_shapes(oracle, w, m, n, k):
    import torch
    p = tf.ag.make_problem(m * 31 + n + k + w, m, n, k)
    p.a, _ = oracle.round_bf16(p.a)
    p.b, _ = oracle.round_bf16(p.b)
    ref = (torch.from_numpy(p.a).double() @ torch.from_numpy(p.b).double()).numpy()
    scale = max(np.abs(ref).max(), 1e-30)
    for fn in (tf.ag.run_pull, tf.ag.run_push, tf.ag.run_baseline):
        run = fn(p, tf.WorldConfig(world_size=w), dtype=1)
        for c in run.c:
            assert float(np.abs(c - ref).max() / scale) <= 4e-3, (fn.__name__, w, m, n, k)
        for g in run.gathered:
            assert np.array_equal(g.view(np.uint32), p.a.view(np.uint32))


@pytest.mark.parametrize("seed", range(6 * SCALE))
def test_ag_fp32_random_shapes_bitwise(oracle, seed):
    rng = np.random.default_rng(seed)
    w = int(rng.choice([1, 2, 3, 4]))
    m, n = int(rng.integers(1, 40)), int(rng.integers(1, 40))
    k = w * int(rng.integers(1, 12))
    tiles = tf.TileSpec(int(rng.integers(1, 9)), int(rng.integers(1, 9)), int(rng.integers(1, 9)))
    p = tf.ag.make_problem(seed + 100, m, n, k, tiles)
    want = oracle.gemm(p.a, p.b)
    for fn in (tf.ag.run_pull, tf.ag.run_push, tf.ag.run_baseline):
        for c in fn(p, tf.WorldConfig(world_size=w)).c:
            assert np.array_equal(c.view(np.uint32), want.view(np.uint32)), (fn.__name__, seed)


def _fd_cases(n=10 * SCALE):
    rng = np.random.default_rng(77)
    out = []
    for _ in range(n):
        w = int(rng.choice([1, 2, 3, 4, 8]))
        hkv = int(rng.choice([1, 2, 4]))
        gs = int(rng.choice([1, 2, 8]))
        d = int(rng.choice([4, 16, 64, 128]))
        L = w * int(rng.choice([1, 3, 17, 64, 300]))
        out.append((w, hkv * gs, hkv, d, L))
    return out


@pytest.mark.parametrize("w,hq,hkv,d,L", _fd_cases())
def test_fd_fp32_random_shapes(oracle, w, hq, hkv, d, L):
    rng = np.random.default_rng(w * 1000 + hq * 10 + d + L)
    q = rng.uniform(-1, 1, (1, hq, d)).astype(np.float32)
    k = rng.uniform(-1, 1, (1, hkv, L, d)).astype(np.float32)
    v = rng.uniform(-1, 1, (1, hkv, L, d)).astype(np.float32)
    scale = float(1 / np.sqrt(np.float32(d)))
    p = tf.fd.DecodeProblem(hq, d, L, scale, q, k, v, batch=1, kv_heads=hkv)
    gs = hq // hkv
    want = np.concatenate([oracle.attention(np.ascontiguousarray(q[0, g * gs:(g + 1) * gs]),
                                            np.repeat(k[0, g:g + 1], gs, 0), np.repeat(v[0, g:g + 1], gs, 0), scale)
                           for g in range(hkv)])
    first = None
    for variant in (V.kBsp, V.kIndependentAg, V.kFineWaits, V.kFused, 5):
        run = tf.fd.run_fd(p, variant, tf.WorldConfig(world_size=w))
        for out in run.out:
            if first is None:
                first = out
            assert np.array_equal(out.view(np.uint32), first.view(np.uint32)), (variant, w, hq, hkv, d, L)
        assert oracle.head_rel_err(run.out[0], want) <= 1e-5, (variant, w, hq, hkv, d, L)


def _fd_fast_cases(n=8):
    rng = np.random.default_rng(99)
    out = []
    for _ in range(n):
        w = int(rng.choice([1, 2, 3, 4]))
        b = int(rng.choice([1, 2, 3]))
        hkv = int(rng.choice([1, 2, 3]))
        L = w * int(rng.choice([5, 16, 100, 777, 2048]))
        out.append((w, b, hkv, L))
    return out


@pytest.mark.parametrize("w,b,hkv,L", _fd_fast_cases())
def test_fd_bf16_fast_path_random_shapes(w, b, hkv, L):
    """The tensor-core decode path (gs = 8, d = 128) on ragged lengths,
    batches and world sizes, fp32 output (hi/lo P) vs torch fp32 at 1e-4,
    bf16 output at 2^-8 + 1e-4 (tests/_tol.py); every schedule and rank bitwise equal."""
    import torch
    hq, d = 8 * hkv, 128
    g = torch.Generator().manual_seed(w * 100 + b * 10 + hkv + L)
    q = (torch.rand(b, hq, d, generator=g) * 2 - 1).bfloat16().float()
    k = (torch.rand(b, hkv, L, d, generator=g) * 2 - 1).bfloat16().float()
    v = (torch.rand(b, hkv, L, d, generator=g) * 2 - 1).bfloat16().float()
    scale = float(1 / np.sqrt(np.float32(d)))
    ref = []
    for bb in range(b):
        s = torch.einsum("hgd,hld->hgl", q[bb].view(hkv, 8, d).double(), k[bb].double()) * scale
        ref.append(torch.einsum("hgl,hld->hgd", torch.softmax(s, -1), v[bb].double()).reshape(hq, d))
    ref = torch.stack(ref).float().numpy().reshape(b * hq, d) if b > 1 else ref[0].float().numpy()
    p = tf.fd.DecodeProblem(hq, d, L, scale, q.numpy(), k.numpy(), v.numpy(), batch=b, kv_heads=hkv)
    for out_dtype, tol in ((0, _tol.FD_F32), (1, _tol.FD_BF16)):
        first = None
        for variant in (V.kFused, V.kBsp, 5):
            run = tf.fd.run_fd(p, variant, tf.WorldConfig(world_size=w), dtype=1, out_dtype=out_dtype)
            for out in run.out:
                if first is None:
                    first = out
                assert np.array_equal(out.view(np.uint32), first.view(np.uint32)), (variant, out_dtype)
            err = float((np.abs(run.out[0] - ref).max(-1) / np.abs(ref).max(-1)).max())
            assert err <= tol, (variant, out_dtype, err)
