"""CPU: the restated oracle (oracle/tf_oracle.c) against the reference's own
outputs -- the golden fixtures (tests/golden/make_golden.py, produced by the
reference headers compiled as-is) and, where it is built, oracle/_ref itself.
This pins the checker before any GPU result is judged by it."""
import numpy as np
import pytest

from oracle.oracle import Reference


def unbits(hexes, shape=None):
    a = np.array([int(h, 16) for h in hexes], dtype=np.uint32).view(np.float32)
    return a.reshape(shape) if shape is not None else a


def test_uniform_reals_matches_reference_stream(oracle, golden):
    for seed, hexes in golden["uniform_reals"].items():
        assert np.array_equal(oracle.uniform_reals(int(seed), 64).view(np.uint32),
                              unbits(hexes).view(np.uint32)), seed


def test_survey_known_values(oracle):
    # SURVEY.md Appendix A, computed by the reference: make_problem(1, 8, 8, 8).
    a, b = oracle.ag_problem(1, 8, 8, 8)
    assert np.allclose(a.ravel()[:4], [-0.732246757, -0.727185965, -0.0975701809, -0.957951546], atol=0, rtol=1e-8)
    c = oracle.gemm(a, b)
    assert np.float32(c.ravel()[0]) == np.float32(0.531775355)
    assert np.float32(c.ravel()[7]) == np.float32(-0.815497398)
    assert np.float32(c.ravel()[63]) == np.float32(-0.884664416)


def test_gemm_bitwise_vs_reference_golden(oracle, golden):
    for case in golden["ag"]:
        a, b = oracle.ag_problem(case["seed"], case["m"], case["n"], case["k"])
        c = oracle.gemm(a, b)
        want = unbits(case["c_rank0"], (case["m"], case["n"]))
        assert np.array_equal(c.view(np.uint32), want.view(np.uint32)), case
        assert case["ranks_equal"]
        if case["variant"] == 2:
            assert all(x == 1 for row in case["flags"] for x in row)


def test_fd_world_matches_reference_golden(oracle, golden):
    for case in golden["fd"]:
        q, k, v, s = oracle.fd_problem(case["seed"], case["heads"], case["d"], case["L"])
        wires, out = oracle.fd_world(q, k, v, s, case["world"])
        want = unbits(case["out_rank0"], out.shape)
        # Same ascending fold over the same partial bits: bitwise.
        assert np.array_equal(out.view(np.uint32), want.view(np.uint32)), case
        oracle_out = unbits(case["oracle"], out.shape)
        assert np.array_equal(oracle.attention(q, k, v, s).view(np.uint32), oracle_out.view(np.uint32))


def test_partial_wire_rows_match_reference(oracle, golden):
    for case in golden["fd_partials"]:
        q, k, v, s = oracle.fd_problem(case["seed"], case["heads"], case["d"], case["L"])
        ln = case["L"] // case["world"]
        r = case["rank"]
        wire = oracle.partial_wire(q, k[:, r * ln:(r + 1) * ln], v[:, r * ln:(r + 1) * ln], s)
        assert np.array_equal(wire.ravel().view(np.uint32), unbits(case["wire"]).view(np.uint32))


def test_tilemath_known_answers(oracle):
    # tilemath_test.cpp:130-142: orthogonal key -> m = 0, l = 1, o = v exactly.
    q = np.array([[1.0, 0.0]], np.float32)
    k = np.array([[[0.0, 1.0]]], np.float32)
    v = np.array([[[3.0, -2.0]]], np.float32)
    w = oracle.partial_wire(q, k, v, 1.0)
    assert w[0, 0] == 0.0 and w[0, 1] == 1.0 and w[0, 2] == 3.0 and w[0, 3] == -2.0
    assert np.array_equal(oracle.finalize_wire(w), v[:, 0])
    # :144-158 duplicated key doubles l.
    w2 = oracle.partial_wire(q, np.concatenate([k, k], 1), np.concatenate([v, v], 1), 1.0)
    assert w2[0, 0] == w[0, 0] and w2[0, 1] == 2 * w[0, 1]
    assert np.array_equal(oracle.finalize_wire(w2), oracle.finalize_wire(w))
    # :160-169 zero-length slice is neutral; finalize rejects it.
    neutral = oracle.neutral_wire(3, 2)
    with pytest.raises(ZeroDivisionError):
        oracle.finalize_wire(neutral)
    # :183-190 non-finite score.
    with pytest.raises(FloatingPointError):
        oracle.partial_wire(np.array([[np.inf, 0]], np.float32), k, v, 1.0)
    # :265-276 neutral is a bitwise two-sided identity; :325-342 wire layout.
    x = oracle.partial_wire(q, k, v, 1.0)
    assert np.array_equal(oracle.combine_wire(oracle.neutral_wire(1, 2), x), x)
    assert np.array_equal(oracle.combine_wire(x, oracle.neutral_wire(1, 2)), x)


@pytest.mark.skipif(not Reference.available(), reason="oracle/_ref not built")
def test_restatement_vs_reference_build_random(oracle):
    R = Reference()
    rng = np.random.default_rng(0)
    for _ in range(5):
        m, n, k = rng.integers(1, 24, 3)
        a = rng.standard_normal((m, k)).astype(np.float32)
        b = rng.standard_normal((k, n)).astype(np.float32)
        assert np.array_equal(oracle.gemm(a, b).view(np.uint32), R.gemm(a, b).view(np.uint32))
    for _ in range(5):
        h, L, d = int(rng.integers(1, 4)), int(rng.integers(1, 80)), int(rng.integers(1, 20))
        q = rng.standard_normal((h, d)).astype(np.float32)
        k = rng.standard_normal((h, L, d)).astype(np.float32)
        v = rng.standard_normal((h, L, d)).astype(np.float32)
        s = np.float32(1 / np.sqrt(d))
        assert np.array_equal(oracle.attention(q, k, v, s).view(np.uint32), R.attention(q, k, v, s).view(np.uint32))
        assert np.array_equal(oracle.partial_wire(q, k, v, s).view(np.uint32),
                              R.partial_wire(q, k, v, s).view(np.uint32))
        x, y = oracle.partial_wire(q, k[:, : L // 2], v[:, : L // 2], s), oracle.partial_wire(q, k[:, L // 2:], v[:, L // 2:], s)
        assert np.array_equal(oracle.combine_wire(x, y).view(np.uint32), R.combine_wire(x, y).view(np.uint32))
