# full ncu captures: data-parallel config 16 (two CTAs/SM) vs its two-group single-CTA form 26 at 4096^3
mkdir -p gpurun_out
for spec in "4096 16" "4096 26"; do
  set -- $spec
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:dgemm --launch-skip 1 --launch-count 1 \
    -o gpurun_out/r2_full_$1_$2 -f python tools/ncu_dgemm.py $1 $2 2 > gpurun_out/r2_full_$1_$2.log 2>&1
  echo "$spec rc=$?"
done
