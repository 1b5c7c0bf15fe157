mkdir -p gpurun_out
( for n in 2048 2560 3072 3584 4096 5120 6144 7168 8192; do timeout 300 python tools/dgemm_ab.py $n 16,17,25 3; done ) > gpurun_out/r2_pair3.txt 2>&1
cat gpurun_out/r2_pair3.txt
