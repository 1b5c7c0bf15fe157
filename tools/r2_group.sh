mkdir -p gpurun_out
( for g in 4 8 16 32 64; do echo "# KW_DGEMM_GROUP=$g"; for n in 4096 8192; do KW_DGEMM_GROUP=$g timeout 300 python tools/dgemm_ab.py $n -1 3; done; done ) > gpurun_out/r2_group_ab.txt 2>&1
cat gpurun_out/r2_group_ab.txt
for g in 8 16 32; do
  KW_DGEMM_GROUP=$g timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum --clock-control none -k regex:dgemm --launch-skip 1 --launch-count 1 --csv python tools/ncu_dgemm.py 8192 -1 2 2>&1 | grep -E '"(gpu__time|dram__bytes|lts__)' | sed "s/^/g=$g /"
done
