"""GPU parity: All-Gather+GEMM through the C ABI vs the reference.

Mirrors proj/tests/ag_gemm_test.cpp, the AG part of acceptance_test.cpp and
cli_test.cpp's config-1 case.  fp32 path: bitwise (max_error == 0.0)."""
import numpy as np
import pytest

import paper_2511_02168_b200 as tf

pytestmark = pytest.mark.gpu


def unbits(hexes, shape):
    return np.array([int(h, 16) for h in hexes], np.uint32).view(np.float32).reshape(shape)


RUNS = {0: tf.ag.run_baseline, 1: tf.ag.run_pull, 2: tf.ag.run_push}


def test_golden_cases_bitwise(golden):
    # Config 1 (cli_test.cpp:162-173), the acceptance W=2 cell, and
    # ag_gemm_test.cpp:62-92 -- every variant, every rank, bitwise.
    for case in golden["ag"]:
        p = tf.ag.make_problem(case["seed"], case["m"], case["n"], case["k"], tf.TileSpec(*case["tiles"]))
        run = RUNS[case["variant"]](p, tf.WorldConfig(world_size=case["world"]))
        want = unbits(case["c_rank0"], (case["m"], case["n"]))
        for r, c in enumerate(run.c):
            assert np.array_equal(c.view(np.uint32), want.view(np.uint32)), (case, r)
        if case["variant"] == 2:
            assert run.flag_counts == case["flags"], case


def test_all_variants_match_naive_gemm_bitwise(oracle):
    # ag_gemm_test.cpp:62-83: tiles that do not divide the shape.
    p = tf.ag.make_problem(7, 13, 9, 16, tf.TileSpec(4, 5, 3))
    want = oracle.gemm(p.a, p.b)
    for w in (1, 2, 4):
        for run_fn in RUNS.values():
            run = run_fn(p, tf.WorldConfig(world_size=w))
            for c in run.c:
                assert np.array_equal(c.view(np.uint32), want.view(np.uint32))


def test_gathered_operand_is_bit_exact():
    # The inbox / stage equals the logical A bit for bit.
    p = tf.ag.make_problem(21, 33, 17, 48, tf.TileSpec(8, 8, 5))
    for run_fn in (tf.ag.run_baseline, tf.ag.run_push):
        run = run_fn(p, tf.WorldConfig(world_size=4))
        for g in run.gathered:
            assert np.array_equal(g.view(np.uint32), p.a.view(np.uint32))


def test_structure_launches_and_flags():
    # ag_gemm_test.cpp:101-170: launches per schedule and push flags == 1.
    p = tf.ag.make_problem(13, 8, 8, 16)
    w = 4
    base = tf.ag.run_baseline(p, tf.WorldConfig(world_size=w))
    pull = tf.ag.run_pull(p, tf.WorldConfig(world_size=w))
    push = tf.ag.run_push(p, tf.WorldConfig(world_size=w))
    assert pull.launches == w            # one fused kernel per rank
    assert push.launches == 2 * w        # producer + consumer per rank
    assert base.launches == 4 * w        # sync barrier, gather, barrier, gemm
    n_kb = (16 // w + 15) // 16
    for counts in push.flag_counts:
        assert counts == [1] * (w * n_kb)


def test_acceptance_grid_bitwise(oracle):
    # acceptance_test.cpp:90-135: W x M x N x K grid, bitwise (a sample of
    # the 108 cells that keeps the GPU test short; the CPU oracle runs all).
    seed = 1
    for w in (1, 2, 4, 8):
        for m in (1, 16, 64):
            for nk in ((8, 8), (32, 64), (64, 32)):
                n, k = nk
                if k % w:
                    continue
                p = tf.ag.make_problem(seed, m, n, k)
                want = oracle.gemm(p.a, p.b)
                run = tf.ag.run_pull(p, tf.WorldConfig(world_size=w))
                assert np.array_equal(run.c[0].view(np.uint32), want.view(np.uint32)), (w, m, n, k)
                seed += 1


def test_rejects_non_divisible_k():
    p = tf.ag.make_problem(5, 4, 4, 10)
    with pytest.raises(tf.ConfigError):
        tf.ag.run_pull(p, tf.WorldConfig(world_size=4))


def test_three_taxes_structure():
    # ag_gemm_test.cpp:101-143 on the GPU: pull needs no barrier, baseline
    # two per rank; push and baseline stage the gathered M x K operand.
    w = 4
    p = tf.ag.make_problem(12, 8, 8, 16)
    pull = tf.ag.run_pull(p, tf.WorldConfig(world_size=w))
    push = tf.ag.run_push(p, tf.WorldConfig(world_size=w))
    base = tf.ag.run_baseline(p, tf.WorldConfig(world_size=w))
    assert pull.taxes[0]["barrier_waits"] == 0 and pull.taxes[0]["staged_bytes"] == 0
    assert push.taxes[0]["barrier_waits"] == 0
    assert [t["barrier_waits"] for t in base.taxes] == [2] * w  # per rank
    for t in push.taxes + base.taxes:
        assert t["staged_bytes"] == p.m * p.k * 4
