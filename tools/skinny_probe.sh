# Config-5 skinny-M probe: ours vs cuBLAS, split-K override sweep.
for M in 128 256 512 1024; do
  echo "== M=$M"; timeout 120 python tools/probe_gemm.py $M 8192 8192 2>&1 | grep -E "ours|cublas|err"
  for ks in 1 2 4 8; do echo -n "ks=$ks "; TFB_KSPLIT=$ks timeout 120 python tools/probe_gemm.py $M 8192 8192 2>&1 | grep -E "ours"; done
done
