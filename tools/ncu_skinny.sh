timeout 300 python -m pytest tests/test_ag_host_gpu.py -x -q 2>&1 | grep -E "Error|assert|^E" | head -20
timeout 300 ncu --set full --import-source on --clock-control none -k regex:ag_gemm_sm100 -s 3 -c 1 -o gpurun_out/skinny128 python tools/probe_gemm.py 128 8192 8192 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:ag_gemm_sm100 -c 6 --csv python tools/probe_gemm.py 128 8192 8192 2>/dev/null | grep -o '"gpu__time_duration.sum","[^"]*","[0-9.]*"' | tail -3
TFB_DEBUG=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:ag_gemm_sm100 -c 6 --csv python tools/probe_gemm.py 128 8192 8192 2>/dev/null | grep -o '"gpu__time_duration.sum","[^"]*","[0-9.]*"' | tail -3
