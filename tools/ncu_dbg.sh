# Cycles of the config-2 GEMM per TFB_DEBUG value (64: no epilogue, 1: no C stores, 128: direct st.global epilogue).
for d in ${DBGS:-0 1 64 128}; do
  echo "== TFB_DEBUG=$d"
  TFB_DEBUG=$d timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.max,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:ag_gemm -s 2 -c 1 --csv python tools/probe_gemm.py 8192 28672 8192 2>/dev/null | grep -E "duration|cycles_elapsed|tensor" | awk -F'","' '{print $(NF-2), $NF}'
done
