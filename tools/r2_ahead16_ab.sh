# A/B: two-step fragment prefetch also for the 1-CTA/SM SPLIT config 20 (32x32 warp tiles) — prev = -DKW_DGEMM_AHEAD2_SPLIT16=0
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_dgemm_gpu.py -q -x -k "paired or split" 2>&1 | tail -1
( for r in 1 2; do for lib in prev new; do
    if [ $lib = prev ]; then export KW_LIB_PATH=$PWD/paper_1602_08477_b200/_build/libkw_b200_prev.so; else unset KW_LIB_PATH; fi
    echo "# $lib"; for n in 1152 1280 1536 1664; do timeout 300 python tools/dgemm_ab.py $n 20,-1 3; done
  done; done ) > gpurun_out/r2_ahead16_ab.txt 2>&1
cat gpurun_out/r2_ahead16_ab.txt
