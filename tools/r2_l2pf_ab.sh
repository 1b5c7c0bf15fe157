# A/B: L2 prefetch of the C block at tile start (new) vs none (prev, -DKW_DGEMM_C_L2PF=0)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_dgemm_gpu.py -q -x -k "paired or split or default" 2>&1 | tail -1
( for r in 1 2; do for lib in prev new; do
    if [ $lib = prev ]; then export KW_LIB_PATH=$PWD/paper_1602_08477_b200/_build/libkw_b200_prev.so; else unset KW_LIB_PATH; fi
    echo "# $lib"
    for n in 1536 2048 3072 4096; do timeout 300 python tools/dgemm_ab.py $n -1,17 3; done
    timeout 300 python tools/dgemm_ab.py 8192 -1 2
  done; done ) > gpurun_out/r2_l2pf_ab.txt 2>&1
cat gpurun_out/r2_l2pf_ab.txt
