#!/bin/bash
for s in 18 24 30 37 48 74; do echo "splits $s"; TFB_FD_SPLITS=$s timeout 60 python tools/probe_fd.py 2>&1 | grep "variant 3"; done
