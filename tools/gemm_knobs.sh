#!/bin/bash
run() { echo "DBG=$1 $2"; TFB_DEBUG=$1 timeout 120 python tools/probe_gemm.py $2 2>&1 | grep -E "ours|cublas|err"; }
run 0 "8192 28672 8192"; run 2 "8192 28672 8192"; run 0 "8192 8192 8192"; run 0 "4096 4096 4096"
