"""GPU: the fabric primitives -- symmetric heap, signal boards, watchdog
diagnostics, device barrier, signal-carries-data soak.  Mirrors the
signal/heap parts of proj/tests/fabric_test.cpp and acceptance_test.cpp:316-381."""
import numpy as np
import pytest

import paper_2511_02168_b200 as tf

pytestmark = pytest.mark.gpu


def world(w, watchdog=0.0):
    return tf.World(w, tf.WorldConfig(world_size=w).device_list(), 64 << 20, watchdog)


def test_heap_zero_filled_and_collective_checks():
    with world(2) as w:
        ptrs = w.alloc("t.zero", 4096)
        for p in ptrs:
            assert not w.get(p, (1024,), np.float32).any()
        assert w.alloc("t.zero", 4096) == ptrs  # same name, same shape: same regions
        with pytest.raises(tf.ConfigError):
            w.alloc("t.zero", 8192)  # shape mismatch (fabric.hpp:304-307)
        with pytest.raises(tf.ConfigError):
            w.alloc("", 16)
        with pytest.raises(tf.ConfigError):
            w.alloc("t.empty", 0)


def test_ring_round_trip_through_peer_regions():
    with world(4) as w:
        ptrs = w.alloc("t.ring", 64)
        for r in range(4):
            w.put(ptrs[(r + 1) % 4], np.full(16, r, np.float32))
        for r in range(4):
            assert (w.get(ptrs[r], (16,), np.float32) == (r - 1) % 4).all()


def test_signal_counting_and_per_destination_grids():
    with world(2) as w:
        w.board("t.flags", 2, 3)
        w.signal("t.flags", 0, 1, 1, 2)
        w.signal("t.flags", 0, 1, 1, 2)
        w.signal("t.flags", 1, 0, 0, 0)
        assert w.read_signal("t.flags", 1, 1, 2) == 2
        assert w.read_signal("t.flags", 0, 1, 2) == 0
        assert w.read_signal("t.flags", 0, 0, 0) == 1
        w.wait_signal("t.flags", 1, 1, 2, 2)  # already satisfied: fast path
        with pytest.raises(tf.BoundsError):
            w.signal("t.flags", 0, 1, 2, 0)
        with pytest.raises(tf.ConfigError):
            w.board("t.flags", 3, 3)


def test_wait_timeout_names_the_cell():
    # acceptance_test.cpp:354-370: the waiter names the board cell and both counts.
    with world(2, watchdog=0.15) as w:
        w.board("soak.never", 1, 1)
        with pytest.raises(tf.DeadlockError) as e:
            w.wait_signal("soak.never", 0, 0, 0, 1)
        msg = str(e.value)
        assert "soak.never" in msg and "expected >= 1" in msg and "observed 0" in msg


def test_signal_carries_data_soak():
    # acceptance_test.cpp:316-341: randomised interleavings, zero stale reads.
    with world(4) as w:
        total = 0
        for seed in range(1, 11):
            total += w.soak(seed, 100)
        assert total == 0


def test_device_barrier_and_mismatch_diagnostic():
    # acceptance_test.cpp:342-353: the lone waiter names the generation and
    # "1 of 2"; the world stays usable afterwards.
    with world(2, watchdog=0.2) as w:
        w.barrier()
        w.barrier()
        with pytest.raises(tf.DeadlockError) as e:
            w.barrier(only_rank=0)
        msg = str(e.value)
        assert "barrier generation" in msg and "1 of 2" in msg, msg
        w.barrier()  # re-aligned


def test_watchdog_is_configurable_and_bounded():
    import time
    with world(2, watchdog=0.1) as w:
        w.board("t.never", 1, 1)
        t0 = time.time()
        with pytest.raises(tf.DeadlockError):
            w.wait_signal("t.never", 1, 0, 0, 5)
        assert time.time() - t0 < 5.0
