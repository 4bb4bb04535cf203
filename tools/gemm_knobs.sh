#!/bin/bash
run() { echo "DBG=$1 $2"; TFB_DEBUG=$1 timeout 120 python tools/probe_gemm.py $2 2>&1 | grep -E "ours"; }
run 0 "8192 28672 8192"; run 1 "8192 28672 8192"; run 0 "8192 28672 8192"
