# A/B: batched epilogue (current) vs interleaved (libkw_b200_prev.so), interleaved per size
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_dgemm_gpu.py -q -x -k "paired or split or golden or closed" 2>&1 | tail -1
( for n in 1024 2048 3072 4096 8192; do
    for lib in prev new; do
      if [ $lib = prev ]; then export KW_LIB_PATH=$PWD/paper_1602_08477_b200/_build/libkw_b200_prev.so; else unset KW_LIB_PATH; fi
      echo "# $lib"; timeout 300 python tools/dgemm_ab.py $n -1,16,17,25 3
    done
  done ) > gpurun_out/r2_epi_ab.txt 2>&1
cat gpurun_out/r2_epi_ab.txt
