"""GPU parity: Flash Decode through the C ABI vs the reference.

Mirrors proj/tests/flash_decode_test.cpp and the FD part of
acceptance_test.cpp: every schedule and rank bitwise identical, oracle
within the reference's 1e-5 head-relative tolerance (fp32 path)."""
import numpy as np
import pytest

import paper_2511_02168_b200 as tf
import _tol  # noqa: E402  (tests/_tol.py)

pytestmark = pytest.mark.gpu
V = tf.fd.Variant
ALL = [V.kBsp, V.kIndependentAg, V.kFineWaits, V.kFused]


def unbits(hexes, shape):
    return np.array([int(h, 16) for h in hexes], np.uint32).view(np.float32).reshape(shape)


def test_all_variants_agree_bitwise_and_match_oracle(oracle):
    # flash_decode_test.cpp:63-88
    p = tf.fd.make_problem(5, 2, 8, 96)
    want = oracle.attention(p.q[0], p.k[0], p.v[0], p.scale)
    for w in (1, 2, 4):
        first = None
        for variant in ALL:
            run = tf.fd.run_fd(p, variant, tf.WorldConfig(world_size=w))
            assert len(run.out) == w
            for out in run.out:
                if first is None:
                    first = out
                assert np.array_equal(out.view(np.uint32), first.view(np.uint32)), (variant, w)
            assert oracle.head_rel_err(run.out[0], want) <= 1e-5, (variant, w)


def test_golden_outputs_within_tolerance(golden, oracle):
    for case in golden["fd"]:
        if case["variant"] != 3:
            continue
        p = tf.fd.make_problem(case["seed"], case["heads"], case["d"], case["L"])
        run = tf.fd.run_fused(p, tf.WorldConfig(world_size=case["world"]))
        ref_out = unbits(case["out_rank0"], (case["heads"], case["d"]))
        orc = unbits(case["oracle"], (case["heads"], case["d"]))
        assert oracle.head_rel_err(run.out[0], orc) <= 1e-5, case
        assert oracle.head_rel_err(run.out[0], ref_out) <= 1e-5, case
        assert run.flag_counts == case["flags"], case


def test_world_size_only_perturbs_roundoff():
    # flash_decode_test.cpp:91-102
    p = tf.fd.make_problem(6, 2, 4, 64)
    base = tf.fd.run_fused(p, tf.WorldConfig(world_size=1)).out[0]
    from oracle.oracle import Oracle
    O = Oracle()
    for w in (2, 4, 8):
        out = tf.fd.run_fused(p, tf.WorldConfig(world_size=w)).out[0]
        assert O.head_rel_err(out, base) <= 1e-5, w


def test_inbox_rows_are_every_sources_partial():
    # Placement is bit-exact: every rank's inbox holds the same W wire rows,
    # and for BSP the stage holds exactly what each source published.
    p = tf.fd.make_problem(1, 2, 4, 64)
    for variant in ALL:
        run = tf.fd.run_fd(p, variant, tf.WorldConfig(world_size=4))
        for box in run.inbox[1:]:
            assert np.array_equal(box.view(np.uint32), run.inbox[0].view(np.uint32)), variant
        if variant != V.kBsp:
            for counts in run.flag_counts:
                assert counts == [1, 1, 1, 1]


def test_acceptance_grid(oracle):
    # acceptance_test.cpp:140-202 (sampled): W x H x d x kv, oracle 1e-5,
    # bitwise across ranks.
    seed = 1
    for w in (1, 2, 4, 8):
        for h in (1, 2, 8):
            for d in (4, 16, 128):
                for kv in (64, 512):
                    p = tf.fd.make_problem(seed, h, d, kv)
                    seed += 1
                    run = tf.fd.run_fused(p, tf.WorldConfig(world_size=w))
                    want = oracle.attention(p.q[0], p.k[0], p.v[0], p.scale)
                    assert oracle.head_rel_err(run.out[0], want) <= 1e-5, (w, h, d, kv)
                    for out in run.out[1:]:
                        assert np.array_equal(out.view(np.uint32), run.out[0].view(np.uint32))


def test_gqa_bf16_fast_path_vs_oracle(oracle):
    # GQA restatement: q-head g*(Hq/Hkv)+j reads KV head g.
    B, Hq, Hkv, d, L = 2, 16, 2, 128, 2048
    rng = np.random.default_rng(3)
    q = rng.uniform(-1, 1, (B, Hq, d)).astype(np.float32)
    k = rng.uniform(-1, 1, (B, Hkv, L, d)).astype(np.float32)
    v = rng.uniform(-1, 1, (B, Hkv, L, d)).astype(np.float32)
    qb, _ = oracle.round_bf16(q)
    kb, _ = oracle.round_bf16(k)
    vb, _ = oracle.round_bf16(v)
    p = tf.fd.DecodeProblem(Hq, d, L, float(1 / np.sqrt(np.float32(d))), qb, kb, vb, batch=B, kv_heads=Hkv)
    gs = Hq // Hkv
    want = np.empty((B, Hq, d), np.float32)
    for b in range(B):
        for g in range(Hkv):
            want[b, g * gs:(g + 1) * gs] = oracle.attention(
                np.ascontiguousarray(qb[b, g * gs:(g + 1) * gs]),
                np.repeat(kb[b, g:g + 1], gs, 0), np.repeat(vb[b, g:g + 1], gs, 0), p.scale)
    for w in (1, 2, 4):
        for variant in (V.kFused, V.kBsp):
            # fp32 output: the tensor-core split feeds P as a bf16 hi + lo
            # pair, so bf16 K/V decode is fp32-grade against the oracle.
            run = tf.fd.run_fd(p, variant, tf.WorldConfig(world_size=w), dtype=1, out_dtype=0)
            err = oracle.head_rel_err(run.out[0].reshape(B * Hq, d), want.reshape(B * Hq, d))
            assert err <= 1e-4, (w, variant, err)
            # bf16 output: the same fp32-grade path; its only extra error is
            # the output's own rounding, <= 2^-8 of the head's max (_tol).
            run = tf.fd.run_fd(p, variant, tf.WorldConfig(world_size=w), dtype=1, out_dtype=1)
            err = oracle.head_rel_err(run.out[0].reshape(B * Hq, d).astype(np.float32), want.reshape(B * Hq, d))
            assert err <= _tol.FD_BF16, (w, variant, err)


def test_rejects_bad_shapes():
    p = tf.fd.make_problem(1, 2, 4, 64)
    with pytest.raises(tf.ConfigError):
        tf.fd.run_fused(p, tf.WorldConfig(world_size=3))


def test_edge_shapes(oracle):
    # One key per rank; a single head; tiny head_dim (acceptance grid's corners).
    for (h, d, kv, w) in ((1, 4, 4, 4), (1, 4, 8, 8), (3, 5, 12, 2), (2, 256, 64, 2)):
        p = tf.fd.make_problem(11 + h + d, h, d, kv)
        want = oracle.attention(p.q[0], p.k[0], p.v[0], p.scale)
        for variant in ALL:
            run = tf.fd.run_fd(p, variant, tf.WorldConfig(world_size=w))
            assert oracle.head_rel_err(run.out[0], want) <= 1e-5, (h, d, kv, w, variant)


def test_non_finite_score_raises_numeric_error():
    # tilemath_test.cpp:183-190: a non-finite score is a NumericError that
    # names the head and the position.
    p = tf.fd.make_problem(2, 2, 4, 16)
    p.q = p.q.copy()
    p.q[0, 1, 0] = np.inf
    with pytest.raises(tf.NumericError) as e:
        tf.fd.run_fused(p, tf.WorldConfig(world_size=2))
    assert "head 1" in str(e.value)


def test_gqa_bf16_eight_rank_loopback(oracle):
    # Config-3 geometry (8 q heads per KV head, d=128) in an 8-rank world.
    B, Hq, Hkv, d, L = 1, 16, 2, 128, 8 * 512
    rng = np.random.default_rng(8)
    qb, _ = oracle.round_bf16(rng.uniform(-1, 1, (B, Hq, d)).astype(np.float32))
    kb, _ = oracle.round_bf16(rng.uniform(-1, 1, (B, Hkv, L, d)).astype(np.float32))
    vb, _ = oracle.round_bf16(rng.uniform(-1, 1, (B, Hkv, L, d)).astype(np.float32))
    p = tf.fd.DecodeProblem(Hq, d, L, float(1 / np.sqrt(np.float32(d))), qb, kb, vb, batch=B, kv_heads=Hkv)
    gs = Hq // Hkv
    want = np.concatenate([oracle.attention(np.ascontiguousarray(qb[0, g * gs:(g + 1) * gs]),
                                            np.repeat(kb[0, g:g + 1], gs, 0), np.repeat(vb[0, g:g + 1], gs, 0),
                                            p.scale) for g in range(Hkv)])
    run = tf.fd.run_fused(p, tf.WorldConfig(world_size=8), dtype=1, out_dtype=0)
    assert oracle.head_rel_err(run.out[0], want) <= 1e-4
    for out in run.out[1:]:
        assert np.array_equal(out.view(np.uint32), run.out[0].view(np.uint32))
    for counts in run.flag_counts:
        assert counts == [1] * 8


def test_three_taxes_measured_on_device():
    # flash_decode_test.cpp:136-196 on the GPU: fused pays no bulk-sync tax
    # (no barrier waits), BSP two barriers per rank; every rank stages W wire
    # rows (W*W*wire*4 bytes world-wide).
    w = 4
    p = tf.fd.make_problem(3, 2, 8, 64)
    wire_bytes = p.heads * (p.head_dim + 2) * 4
    fused = tf.fd.run_fused(p, tf.WorldConfig(world_size=w))
    bsp = tf.fd.run_bsp(p, tf.WorldConfig(world_size=w))
    assert fused.taxes[0]["barrier_waits"] == 0
    assert fused.launches == 1
    # per rank, even though the loopback ranks share one device
    assert [t["barrier_waits"] for t in bsp.taxes] == [2] * w
    for t in fused.taxes + bsp.taxes:
        assert t["staged_bytes"] == w * wire_bytes
    for t in fused.taxes:
        assert t["signal_waits"] >= w  # one fold wait per source (per group)


def test_fused_waits_target_the_straggler():
    # flash_decode_test.cpp:250-286: with rank 1 delayed 50 ms, rank 0 pays
    # about the delay waiting for source 1, nobody pays a barrier, and the
    # straggler itself barely waits (every other row landed long ago).
    delay = 0.05
    cfg = tf.WorldConfig(world_size=2)
    tf.inject_skew(cfg, 1, delay)
    p = tf.fd.make_problem(14, 2, 4, 64)
    run = tf.fd.run_fused(p, cfg)
    eps = 0.005
    assert run.taxes[0]["wait_idle_ns"] >= (delay - eps) * 1e9
    assert run.taxes[1]["wait_idle_ns"] < delay / 2 * 1e9
    assert all(t["barrier_waits"] == 0 and t["bulk_sync_ns"] == 0 for t in run.taxes)
    with pytest.raises(tf.ConfigError):
        tf.inject_skew(cfg, 2, delay)
    with pytest.raises(tf.ConfigError):
        tf.inject_skew(cfg, 0, -1.0)


def test_fold_by_arrival_option(oracle):
    # flash_decode.hpp:108-114, 377-408: arrival-order fold; equal to the
    # oracle within tolerance, flags all 1; other schedules reject it.
    p = tf.fd.make_problem(5, 2, 8, 96)
    want = oracle.attention(p.q[0], p.k[0], p.v[0], p.scale)
    for w in (1, 2, 4, 8):
        run = tf.fd.run_fused(p, tf.WorldConfig(world_size=w), tf.fd.FdOptions(fold_by_arrival=True))
        for out in run.out:
            assert oracle.head_rel_err(out, want) <= 1e-5
        for counts in run.flag_counts:
            assert counts == [1] * w
    with pytest.raises(tf.ConfigError):
        tf.fd.run_bsp(p, tf.WorldConfig(world_size=2), opts=tf.fd.FdOptions(fold_by_arrival=True))


@pytest.mark.parametrize("w", [2, 3, 4])
def test_owner_combine_matches_all_gather_bitwise(oracle, w):
    """TF_FD_FUSED_OWNER: group g folded by rank g % W, final
    rows pushed to every rank.  Same fold, same bits as the all-gather
    schedules; groups a rank does not own arrive from their owner; ranks
    that own nothing (W > groups) still end with the full output.
    Interleaved with the other schedules in one world, so the boards'
    epochs must stay consistent."""
    p = tf.fd.make_problem(9, 2, 8, 96)  # 2 groups (MHA): at W = 3, 4 some ranks own none
    want = oracle.attention(p.q[0], p.k[0], p.v[0], p.scale)
    cfg = tf.WorldConfig(world_size=w)
    fused = tf.fd.run_fd(p, V.kFused, cfg)
    owner = tf.fd.run_fd(p, 5, cfg)
    bsp = tf.fd.run_fd(p, V.kBsp, cfg)
    for out in owner.out + bsp.out:
        assert np.array_equal(out.view(np.uint32), fused.out[0].view(np.uint32))
    assert oracle.head_rel_err(owner.out[0], want) <= 1e-5
    assert owner.launches == 1


def test_owner_combine_gqa_bf16_eight_ranks(oracle):
    import torch  # noqa: F401
    p = tf.fd.make_problem(21, 64, 128, 2048)
    p.kv_heads = 8
    p.batch = 1
    p.q, _ = oracle.round_bf16(p.q)
    p.k, _ = oracle.round_bf16(p.k[:, :8])
    p.v, _ = oracle.round_bf16(p.v[:, :8])
    cfg = tf.WorldConfig(world_size=8)
    a = tf.fd.run_fd(p, V.kFused, cfg, dtype=1, out_dtype=0)
    b = tf.fd.run_fd(p, 5, cfg, dtype=1, out_dtype=0)
    c = tf.fd.run_fd(p, 5, cfg, dtype=1, out_dtype=0)  # back to back: epochs / parity
    for out in b.out + c.out:
        assert np.array_equal(out.view(np.uint32), a.out[0].view(np.uint32))
