#!/bin/bash
for g in 2 4 8 16 32; do echo "GROUP_M=$g"; TFB_GROUP_M=$g timeout 120 python tools/probe_gemm.py 8192 28672 8192 2>&1 | grep -E "ours"; done
timeout 120 python tools/probe_gemm.py 8192 28672 8192 2>&1 | grep -E "cublas"
