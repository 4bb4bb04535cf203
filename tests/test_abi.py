"""CPU: the C-ABI library builds, loads and exports every symbol tf_abi.h
declares; host-side entry points work without a GPU; compute entry points
fail loudly (no CPU fallback)."""
import ctypes as C
import os
import re

import numpy as np

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "tilefabric_b200", "tf_abi.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tf_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2511_02168_b200 import _abi
    L = _abi.lib()
    syms = declared_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(L, s), s
        assert s in _abi.SIGNATURES, f"{s} missing from the ctypes binding"
    assert L.tf_abi_version() == 1


def test_uniform_reals_is_the_reference_stream(oracle, golden):
    import paper_2511_02168_b200 as tf
    for seed, hexes in golden["uniform_reals"].items():
        want = np.array([int(h, 16) for h in hexes], np.uint32)
        assert np.array_equal(tf.uniform_reals(int(seed), 64).view(np.uint32), want)
    assert np.array_equal(tf.uniform_reals(5, 10000), oracle.uniform_reals(5, 10000))


def test_world_config_validation_without_gpu():
    from paper_2511_02168_b200 import _abi
    L = _abi.lib()
    h = C.c_void_p()
    for bad in (0, 65):
        rc = L.tf_world_create(bad, None, 1 << 20, 0.0, C.byref(h))
        assert rc == 1  # TF_ERR_CONFIG, "world_size must be in [1, 64]"
        assert b"world_size must be in [1, 64]" in L.tf_last_error()


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        return
    from paper_2511_02168_b200 import _abi
    L = _abi.lib()
    h = C.c_void_p()
    rc = L.tf_world_create(1, None, 1 << 20, 0.0, C.byref(h))
    assert rc != 0 and not h.value


def test_python_mirror_validation():
    import pytest
    import paper_2511_02168_b200 as tf
    p = tf.ag.make_problem(1, 4, 4, 12)
    p.validate(4)
    with pytest.raises(tf.ConfigError):
        p.validate(5)  # ag_gemm_test.cpp:42-48
    p.m = 0
    with pytest.raises(tf.ConfigError):
        p.validate(4)
    f = tf.fd.make_problem(1, 2, 16, 8)
    assert f.scale == 0.25  # flash_decode_test.cpp:53-56
    f2 = tf.fd.make_problem(1, 2, 4, 64)
    f2.validate(4)
    with pytest.raises(tf.ConfigError):
        f2.validate(3)
    f2.scale = float("inf")
    with pytest.raises(tf.ConfigError):
        f2.validate(4)


def test_world_config_skew_and_devices():
    # fabric_test.cpp:62-73: inject_skew validates eagerly and accumulates.
    import pytest
    import paper_2511_02168_b200 as tf
    cfg = tf.WorldConfig(world_size=4, devices=[0, 0, 0, 0])
    tf.inject_skew(cfg, 1, 0.010)
    tf.inject_skew(cfg, 1, 0.005)
    assert abs(cfg.skew[1] - 0.015) < 1e-12
    cfg.validate()
    assert cfg.device_list() == [0, 0, 0, 0]
    for rank, delay in ((4, 0.001), (-1, 0.001), (0, -0.001)):
        with pytest.raises(tf.ConfigError):
            tf.inject_skew(cfg, rank, delay)
    cfg.skew[7] = 0.001
    with pytest.raises(tf.ConfigError):
        cfg.validate()
