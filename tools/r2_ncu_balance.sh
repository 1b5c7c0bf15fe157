mkdir -p gpurun_out
M=gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.max,sm__pipe_tensor_subpipe_dmma_cycles_active.min,sm__pipe_tensor_subpipe_dmma_cycles_active.avg,sm__cycles_elapsed.max,sm__cycles_active.min,sm__cycles_active.max,sm__warps_active.avg.per_cycle_active,smsp__average_warp_latency_issue_stalled_wait,smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct,smsp__warp_issue_stalled_math_pipe_throttle_per_warp_active.pct,smsp__warp_issue_stalled_wait_per_warp_active.pct,smsp__warp_issue_stalled_barrier_per_warp_active.pct,smsp__warp_issue_stalled_membar_per_warp_active.pct,smsp__warp_issue_stalled_sleeping_per_warp_active.pct,smsp__warp_issue_stalled_short_scoreboard_per_warp_active.pct,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum
for spec in "2048 17" "2048 16" "2048 20" "2048 21" "2048 22" "8192 16" "8192 21"; do
  set -- $spec
  timeout 600 ncu --metrics $M --clock-control none -k regex:dgemm --launch-skip 1 --launch-count 1 --csv \
    python tools/ncu_dgemm.py $1 $2 2 > gpurun_out/r2_bal_$1_$2.csv 2>&1
  echo "$spec rc=$?"
done
