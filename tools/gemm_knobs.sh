#!/bin/bash
for M in 128 256 512 1024 2048; do echo "M=$M"; timeout 120 python tools/probe_gemm.py $M 8192 8192 2>&1 | grep -E "ours|cublas|err"; done
echo "M=128 no split"; TFB_KSPLIT=1 timeout 120 python tools/probe_gemm.py 128 8192 8192 2>&1 | grep -E "ours"
timeout 120 python tools/probe_gemm.py 8192 28672 8192 2>&1 | grep -E "ours|cublas"
