mkdir -p gpurun_out
( for dp in -1 0 100000; do echo "# KW_SPLIT_DP_TILES=$dp"; for n in 1024 2048 3072; do KW_SPLIT_DP_TILES=$dp timeout 300 python tools/dgemm_ab.py $n 18,20,21,22 3; done; done
  echo "# default tile choice"; for n in 1024 2048 3072; do timeout 300 python tools/dgemm_ab.py $n -1,16,17 3; done ) > gpurun_out/r2_split_ab2.txt 2>&1
cat gpurun_out/r2_split_ab2.txt
