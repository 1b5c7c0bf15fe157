#!/usr/bin/env bash
# BASELINE.json configs[4] — workdiv sweep in the reference's CSV schema (kwbench, backend gpu):
# AXPY fp32 n = 2^28 over threads-per-block x elems-per-thread; DGEMM n = 1024..8192, tile 64/128.
# Verification is on for the AXPY and the smaller DGEMMs (kwbench's CPU check is O(n^3)).
set -euo pipefail
KW=paper_1602_08477_b200/_build/kwbench
OUT=${1:-gpurun_out/kwbench_sweep.csv}
TMP=$(mktemp -d)
i=0
for tpb in 128 256 512 1024; do
  for ept in 4 8 16 32; do
    $KW --kernel axpy --dtype f32 --sizes 268435456 --reps 5 --tpb $tpb --ept $ept --csv $TMP/$i.csv > /dev/null
    i=$((i+1))
  done
done
$KW --kernel axpy --dtype f32 --sizes 1000003 --reps 3 --verify --csv $TMP/$i.csv > /dev/null; i=$((i+1))
for tile in 64 128; do
  $KW --kernel gemm-tiled --sizes 1024,2048 --reps 3 --tile $tile --verify --csv $TMP/$i.csv > /dev/null; i=$((i+1))
  $KW --kernel gemm-tiled --sizes 4096,8192 --reps 3 --tile $tile --csv $TMP/$i.csv > /dev/null; i=$((i+1))
done
head -1 $TMP/0.csv > "$OUT"
for f in $(ls $TMP/*.csv | sort -V); do tail -n +2 "$f" >> "$OUT"; done
rm -rf "$TMP"
echo "wrote $OUT ($(($(wc -l < "$OUT") - 1)) records)"
