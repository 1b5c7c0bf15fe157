# A/B: two-step fragment prefetch for small warp tiles (new) vs one-step (prev, -DKW_DGEMM_AHEAD2=0)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_dgemm_gpu.py -q -x -k "paired or split" 2>&1 | tail -1
( for r in 1 2; do for lib in prev new; do
    if [ $lib = prev ]; then export KW_LIB_PATH=$PWD/paper_1602_08477_b200/_build/libkw_b200_prev.so; else unset KW_LIB_PATH; fi
    echo "# $lib"; timeout 300 python tools/dgemm_ab.py 1024 18,23 3; timeout 300 python tools/dgemm_ab.py 1280 18 3
  done; done ) > gpurun_out/r2_ahead_ab.txt 2>&1
cat gpurun_out/r2_ahead_ab.txt
