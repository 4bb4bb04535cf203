#!/bin/bash
echo "== shapes"; timeout 300 python tools/debug_fd.py 1,64,8,128,32768 2,64,8,128,32768 4,64,8,128,16384 4,64,8,128,8192 4,16,2,128,32768 32,64,8,128,32768 2>&1 | grep -v finite
