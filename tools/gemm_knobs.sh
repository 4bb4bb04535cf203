#!/bin/bash
# GEMM bottleneck bisection: knobs 1 = no C stores, 2 = no MMAs, 4 = local full barriers, 8 = force 1-CTA,
# 16 = launch with cluster dim 2 regardless.
for d in 8 24 26 10; do echo "TFB_DEBUG=$d"; TFB_DEBUG=$d timeout 120 python tools/probe_gemm.py 8192 8192 8192 2>&1 | grep -E "ours"; done
