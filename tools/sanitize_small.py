"""compute-sanitizer target: small bf16 AG+GEMM shapes (split-K / L2 exchange, ragged M, pair tiles), every schedule at W = 1, 2."""
import sys, numpy as np
sys.path.insert(0, "/root/repo")
import paper_2511_02168_b200 as tf
import torch
for (m, n, k) in ((128, 2048, 1024), (300, 768, 512), (1024, 1536, 256)):
    p = tf.ag.make_problem(1, m, n, k)
    for W in (1, 2):
        for fn in (tf.ag.run_pull, tf.ag.run_push, tf.ag.run_baseline):
            r = fn(p, tf.WorldConfig(world_size=W), dtype=1)
print("ag ok")
# Flash Decode: GQA bf16 fast path (bf16 and fp32 out) and the fp32 generic
# path, every schedule at W = 1, 2, 4.
rng = np.random.default_rng(3)
B, Hq, Hkv, d, L = 2, 16, 2, 128, 1024
q = rng.uniform(-1, 1, (B, Hq, d)).astype(np.float32)
k = rng.uniform(-1, 1, (B, Hkv, L, d)).astype(np.float32)
v = rng.uniform(-1, 1, (B, Hkv, L, d)).astype(np.float32)
p = tf.fd.DecodeProblem(Hq, d, L, float(1 / np.sqrt(np.float32(d))), q, k, v, batch=B, kv_heads=Hkv)
V = tf.fd.Variant
for W in (1, 2, 4):
    for var in (V.kBsp, V.kIndependentAg, V.kFineWaits, V.kFused):
        for dt, odt in ((1, 1), (1, 0), (0, 0)):
            tf.fd.run_fd(p, var, tf.WorldConfig(world_size=W), dtype=dt, out_dtype=odt)
    tf.fd.run_fd(p, V.kFused, tf.WorldConfig(world_size=W), opts=tf.fd.FdOptions(owner_combine=True), dtype=1)
print("fd ok")
