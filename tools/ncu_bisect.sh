# Cycles of the config-2 GEMM per library build (TFB_LIB=<.so>).
for lib in "$@"; do
  echo "== $lib"
  TFB_LIB=$lib timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.max,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed.sum,launch__registers_per_thread --clock-control none -k regex:ag_gemm -s 2 -c 1 --csv python tools/probe_gemm.py 8192 28672 8192 2>/dev/null | grep -E "duration|cycles_elapsed|tensor|inst_exec|registers" | awk -F'","' '{print $(NF-2), $NF}'
done
