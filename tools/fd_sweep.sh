#!/bin/bash
for s in 8 16 37 74 148 296 592; do echo "splits $s"; TFB_FD_SPLITS=$s timeout 60 python tools/probe_fd.py 2>&1 | grep "fd3 variant 3"; done
