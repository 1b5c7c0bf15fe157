mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_dgemm_gpu.py -q -x -k "bitwise" 2>&1 | tail -1
( for r in 1 2; do for lib in prev new; do
    if [ $lib = prev ]; then export KW_LIB_PATH=$PWD/paper_1602_08477_b200/_build/libkw_b200_prev.so; else unset KW_LIB_PATH; fi
    echo "# $lib"; timeout 300 python tools/bitwise_rate.py 2048 4096 8192
  done; done ) > gpurun_out/r2_bw_ab.txt 2>&1
cat gpurun_out/r2_bw_ab.txt
