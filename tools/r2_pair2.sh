mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_dgemm_gpu.py tests/test_dgemm_soak_gpu.py -q -x 2>&1 | tail -2
( for n in 1024 1536 2048 2560 3072 4096 6144 8192; do timeout 300 python tools/dgemm_ab.py $n -1,16,17 3; done
  python tools/rowshard_rank_probe.py 8 3 ) 2>&1 | grep -v NCCL > gpurun_out/r2_pair2.txt
cat gpurun_out/r2_pair2.txt
