"""Generates tests/golden/golden.json from the REFERENCE ITSELF.

Run in the build container, where /root/reference exists:
    make -C oracle && python tests/golden/make_golden.py
It drives oracle/_ref/libtfref.so (the unmodified reference headers compiled
by oracle/Makefile) through the reference's own test cases and records the
results bit-exactly (floats as uint32 hex).  The GPU box never regenerates
this file; tests compare against the committed copy.
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))
from oracle.oracle import Reference  # noqa: E402


def bits(a) -> list:
    return [format(int(x), "08x") for x in np.ascontiguousarray(a, np.float32).view(np.uint32).ravel()]


def main() -> None:
    R = Reference()
    g = {"uniform_reals": {}, "ag": [], "fd": [], "fd_partials": []}
    for seed in (0, 1, 7, 99):
        g["uniform_reals"][str(seed)] = bits(R.uniform_reals(seed, 64))
    # AG: config 1 (cli_test.cpp:162-173), the acceptance W=2 cell
    # (acceptance_test.cpp:90-135, seed 1, 1x8x8), ag_gemm_test.cpp:62-92.
    ag_cases = [
        dict(seed=1, m=8, n=8, k=8, tiles=(16, 16, 16), worlds=(1, 2)),
        dict(seed=1, m=1, n=8, k=8, tiles=(16, 16, 16), worlds=(2,)),
        dict(seed=7, m=13, n=9, k=16, tiles=(4, 5, 3), worlds=(1, 2, 4)),
        dict(seed=3, m=1, n=1, k=1, tiles=(16, 16, 16), worlds=(1,)),
        dict(seed=11, m=8, n=8, k=16, tiles=(16, 16, 16), worlds=(4,)),
    ]
    for c in ag_cases:
        for w in c["worlds"]:
            for variant in (0, 1, 2):
                cc, flags, _, _ = R.ag_run(variant, c["seed"], c["m"], c["n"], c["k"], w, c["tiles"])
                g["ag"].append(dict(seed=c["seed"], m=c["m"], n=c["n"], k=c["k"], tiles=list(c["tiles"]),
                                    world=w, variant=variant, c_rank0=bits(cc[0]),
                                    ranks_equal=bool(all(np.array_equal(cc[0], x) for x in cc)),
                                    flags=None if flags is None else flags.astype(int).tolist()))
    # FD: flash_decode_test.cpp:63-88 (seed 5, 2x8x96), SURVEY App. A
    # (seed 1, 2x4x64), :91-102 (seed 6, 2x4x64), make_problem(1, 2, 16, 8).
    fd_cases = [
        dict(seed=5, heads=2, d=8, L=96, worlds=(1, 2, 4)),
        dict(seed=1, heads=2, d=4, L=64, worlds=(1, 2, 4, 8)),
        dict(seed=6, heads=2, d=4, L=64, worlds=(1, 2, 4, 8)),
        dict(seed=2, heads=8, d=128, L=4096, worlds=(1, 8)),
    ]
    from oracle.oracle import Oracle
    O = Oracle()
    for c in fd_cases:
        q, k, v, scale = O.fd_problem(c["seed"], c["heads"], c["d"], c["L"])
        oracle = R.attention(q, k, v, scale)
        for w in c["worlds"]:
            for variant in (0, 1, 2, 3):
                out, flags, _, _ = R.fd_run(variant, c["seed"], c["heads"], c["d"], c["L"], w)
                g["fd"].append(dict(seed=c["seed"], heads=c["heads"], d=c["d"], L=c["L"], world=w,
                                    variant=variant, out_rank0=bits(out[0]),
                                    oracle=bits(oracle),
                                    head_rel_err=R.head_rel_err(out[0], oracle),
                                    flags=None if variant == 0 else flags.astype(int).tolist()))
    # Per-shard wire rows the reference's fused schedule pushes (inbox contents).
    for c in fd_cases[:2]:
        q, k, v, scale = O.fd_problem(c["seed"], c["heads"], c["d"], c["L"])
        for w in (2,):
            ln = c["L"] // w
            for r in range(w):
                wire = R.partial_wire(q, np.ascontiguousarray(k[:, r * ln:(r + 1) * ln]),
                                      np.ascontiguousarray(v[:, r * ln:(r + 1) * ln]), scale)
                g["fd_partials"].append(dict(seed=c["seed"], heads=c["heads"], d=c["d"], L=c["L"],
                                             world=w, rank=r, wire=bits(wire)))
    path = os.path.join(os.path.dirname(__file__), "golden.json")
    with open(path, "w") as f:
        json.dump(g, f, indent=0)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
