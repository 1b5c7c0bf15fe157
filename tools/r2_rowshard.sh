mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "rowsharded or nccl" 2>&1 | tail -2
( for p in 8 4 16; do echo "# kslab schedule, panels=$p"; python tools/rowshard_rank_probe.py $p 3; done
  echo "# KW_ROWSHARD_SCHEDULE=panels, panels=8"; KW_ROWSHARD_SCHEDULE=panels python tools/rowshard_rank_probe.py 8 3 ) 2>&1 | grep -v NCCL > gpurun_out/r2_rowshard_probe4.txt
cat gpurun_out/r2_rowshard_probe4.txt
