# Per-variant cycles of the config-2 GEMM under ncu (clocks vary; cycles don't lie).
M=${M:-8192}; N=${N:-28672}; K=${K:-8192}
for v in "" "TFB_DEBUG=32" "TFB_NO_TAIL_SPLIT=1" "TFB_DEBUG=32 TFB_NO_TAIL_SPLIT=1"; do
  echo "== [$v]"
  env $v timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.max,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed.sum --clock-control none -k regex:ag_gemm -s 2 -c 1 --csv python tools/probe_gemm.py $M $N $K 2>/dev/null | grep -E "duration|cycles_elapsed|tensor|inst_exec" | awk -F'","' '{print $(NF-2), $NF}'
done
