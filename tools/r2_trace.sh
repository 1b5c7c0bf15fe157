mkdir -p gpurun_out
KW_EXTRA_NVCC_FLAGS=-DKW_SPLIT_TRACE python -c "from paper_1602_08477_b200 import build as B; B.build_lib(force=True)" > /dev/null 2>&1 || echo BUILD FAILED
for spec in "2048 25" "2048 25" "2048 18"; do set -- $spec; timeout 300 python tools/split_trace.py $1 $2; done > gpurun_out/r2_split_trace2.txt 2>&1
cat gpurun_out/r2_split_trace2.txt
