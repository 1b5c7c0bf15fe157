# full ncu captures (stall reasons, source-level) of the small-DGEMM tile choices: 1024^3 (SPLIT cfg 18), 2048^3 (cfg 17)
mkdir -p gpurun_out
for spec in "1024 18" "2048 17"; do
  set -- $spec
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:dgemm --launch-skip 1 --launch-count 1 \
    -o gpurun_out/r2_full_$1_$2 -f python tools/ncu_dgemm.py $1 $2 2 > gpurun_out/r2_full_$1_$2.log 2>&1
  echo "$spec rc=$?"
done
