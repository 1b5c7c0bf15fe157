# full GPU suite + smoke + reference arm + bench (N=1), results under gpurun_out/
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2_gputests.txt 2>&1; echo rc=$? >> gpurun_out/r2_gputests.txt
tail -4 gpurun_out/r2_gputests.txt
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/r2_smoke.txt 2>&1; tail -2 gpurun_out/r2_smoke.txt
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2_ref.json 2> gpurun_out/r2_ref.err; echo ref rc=$?
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo bench rc=$?
