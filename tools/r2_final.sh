# round-2 final evidence on one B200: GPU suite, smoke, reference arm, bench N=1 (default flags),
# --force-rowsharded (16384^3 k-slab pipeline with the world-1 NCCL broadcasts), the library's
# DGEMM choice by size, and the ncu launch list of the bench command (after it exited 0 plain)
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/rf_gputests.txt 2>&1; echo rc=$? >> gpurun_out/rf_gputests.txt
tail -3 gpurun_out/rf_gputests.txt
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/rf_smoke.txt 2>&1; tail -2 gpurun_out/rf_smoke.txt
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/rf_ref.json 2> gpurun_out/rf_ref.err; echo ref rc=$?
timeout 900 python bench.py > gpurun_out/rf_bench.json 2> gpurun_out/rf_bench.err; echo bench rc=$?
timeout 900 python bench.py --steps 20 --warmup 5 --force-rowsharded --no-cublas --no-f64 > gpurun_out/rf_force.json 2> gpurun_out/rf_force.err; echo force rc=$?
( for n in 1024 1280 1536 2048 2560 3072 4096 6144 8192; do timeout 300 python tools/dgemm_ab.py $n -1 3; done ) > gpurun_out/rf_default_sweep.txt 2>&1
python bench.py --steps 2 --warmup 3 --no-cpu --no-cublas > gpurun_out/rf_plain.json 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/rf_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-cublas > gpurun_out/rf_ncu.log 2>&1; echo ncu rc=$?
python tools/launch_summary.py gpurun_out/rf_launches.csv > gpurun_out/rf_launches_summary.txt 2>&1; head -12 gpurun_out/rf_launches_summary.txt
