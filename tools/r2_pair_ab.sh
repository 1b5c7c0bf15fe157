mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_dgemm_gpu.py -q -x -k "paired or split" 2>&1 | tail -2
( for n in 1536 2048 2560 3072 4096 8192; do timeout 300 python tools/dgemm_ab.py $n -1,16,17,25,26 3; done ) > gpurun_out/r2_pair_ab.txt 2>&1
cat gpurun_out/r2_pair_ab.txt
