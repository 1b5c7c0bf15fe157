mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "rowsharded or nccl" 2>&1 | tail -2
( for p in 8 4; do echo "# head schedule, panels=$p"; python tools/rowshard_rank_probe.py $p 3; done
  for p in 8 16; do echo "# KW_ROWSHARD_SCHEDULE=equal, panels=$p"; KW_ROWSHARD_SCHEDULE=equal python tools/rowshard_rank_probe.py $p 3; done ) 2>&1 | grep -v NCCL > gpurun_out/r2_rowshard_probe3.txt
cat gpurun_out/r2_rowshard_probe3.txt
