# round-2 SPLIT DGEMM check + A/B: parity tests, then TFLOP/s per config (tools/dgemm_ab.py)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_dgemm_gpu.py -q -x -k "paired or split" > gpurun_out/r2_split_tests.txt 2>&1; echo rc=$? >> gpurun_out/r2_split_tests.txt
tail -3 gpurun_out/r2_split_tests.txt
( for n in 1024 2048 4096 8192; do timeout 300 python tools/dgemm_ab.py $n ${CFGS:--1,16,17,18,20,21,22} 3; done
  echo "# KW_SPLIT_DP_TILES=0 (all tiles in equal k-ranges)"
  for n in 4096 8192; do KW_SPLIT_DP_TILES=0 timeout 300 python tools/dgemm_ab.py $n 18,20,21 3; done
  echo "# KW_DGEMM_PDL=0"
  for n in 2048 8192; do KW_DGEMM_PDL=0 timeout 300 python tools/dgemm_ab.py $n -1,16,17,21 3; done ) > gpurun_out/r2_split_ab.txt 2>&1
cat gpurun_out/r2_split_ab.txt
