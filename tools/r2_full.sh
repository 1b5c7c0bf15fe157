# full GPU suite + smoke + reference arm + bench (N=1) + the library's DGEMM choice by size
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2_gputests.txt 2>&1; echo rc=$? >> gpurun_out/r2_gputests.txt
tail -4 gpurun_out/r2_gputests.txt
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/r2_smoke.txt 2>&1; tail -2 gpurun_out/r2_smoke.txt
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2_ref.json 2> gpurun_out/r2_ref.err; echo ref rc=$?
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo bench rc=$?
( for n in 1024 1280 1536 2048 2560 3072 4096 6144 8192; do timeout 300 python tools/dgemm_ab.py $n -1 3; done ) > gpurun_out/r2_default_sweep.txt 2>&1
cat gpurun_out/r2_default_sweep.txt
