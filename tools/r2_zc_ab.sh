# A/B: e2e AXPY (pinned host X, Y through the public API) with copy-engine staging (zerocopy=0) vs
# the kernel reading/writing the mapped pinned pages directly (zerocopy=1); pcie.cu mix line for the box
mkdir -p gpurun_out
( timeout 100 ./tools/probe/pcie 2>/dev/null | tail -2
  for r in 1 2 3 4 5 6; do for z in 0 1; do KW_AXPY_ZEROCOPY=$z timeout 100 python tools/e2e_sweep.py; done; done
  for z in 0 1; do KW_AXPY_ZEROCOPY=$z timeout 600 python bench.py --steps 5 --warmup 3 --no-dgemm --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench zerocopy=$z e2e', d['e2e']['value'], 'parity', d.get('parity', {}).get('match'))"; done
) > gpurun_out/r2_zc_ab.txt 2>&1
cat gpurun_out/r2_zc_ab.txt
