for v in "" "TFB_L2HINT=1" "TFB_L2HINT=2" "TFB_L2HINT=3"; do
  echo "== $v"; env $v ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:ag_gemm -s 1 -c 1 python tools/profile_kernels.py ag 3 2>&1 | grep -E "duration|bytes"
done
