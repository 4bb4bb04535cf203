#!/bin/bash
# One GPU call: bench line, bench launch list, ncu --set full captures of the
# hot kernels.  Usage: bash tools/profile_round.sh <round>   (writes gpurun_out/)
R=${1:-r1}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${R}_launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu \
  > gpurun_out/${R}_bench_under_ncu.log 2>&1
for x in ag fd3 fd4 agM128 agM256; do
  k=ag_gemm_sm100; case $x in fd*) k="fd_(attention|stream)";; esac
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
    -o gpurun_out/${R}_$x -f python tools/profile_kernels.py $x > gpurun_out/${R}_$x.log 2>&1
done
# the TMA push producer (loopback W = 2: the profiler serialises, producers first)
timeout 300 ncu --set full --clock-control none -k regex:ag_push_tma -s 2 -c 1 -o gpurun_out/${R}_push -f \
  python tools/probe_push.py 2 > gpurun_out/${R}_push.log 2>&1
timeout 300 ncu --set full --clock-control none -k regex:nvjet -s 1 -c 1 -o gpurun_out/${R}_cublas_cfg2 -f \
  python tools/probe_cublas.py 8192 28672 8192 > gpurun_out/${R}_cublas.log 2>&1
ls -la gpurun_out/
