# round-2 ncu evidence for DGEMM: FP64 DMMA pipe counters + DRAM bytes, one launch per shape
mkdir -p gpurun_out
M=gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__inst_executed_pipe_tensor_subpipe_dmma.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_fp64.sum,sm__ops_path_tensor_src_fp64.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,launch__grid_size,launch__registers_per_thread
for spec in "1024 -1" "2048 -1" "4096 -1" "8192 -1" "1024 17"; do
  set -- $spec
  timeout 600 ncu --metrics $M --clock-control none -k regex:dgemm --launch-skip 1 --launch-count 1 --csv \
    python tools/ncu_dgemm.py $1 $2 2 > gpurun_out/r2_ncu_dgemm_$1_$2.csv 2> gpurun_out/r2_ncu_dgemm_$1_$2.err
  echo "$spec rc=$?"
done
# bit-exact tiled mode (FP64 pipe: DMUL + DADD) at 4096
cat > /tmp/bw.py <<'PY'
import sys; sys.path.insert(0, '.')
import numpy as np
from paper_1602_08477_b200 import _lib as L, kernelweave as kw
lib = L.lib(); dev = kw.Device.gpu(0); q = kw.Queue(dev, kw.QueueFlavor.Async); n = 4096
A, B, Cb = (kw.Buffer(dev, kw.IndexVec(n, n), 8) for _ in range(3))
for b in (A, B, Cb): b.upload(np.random.default_rng(0).random((n, n)))
for _ in range(2):
    L.check(lib.kw_dgemm_bitwise(q.handle(), None, n, n, n, 1.0, A.data(), A.leadingDim(), B.data(), B.leadingDim(), 1.0, Cb.data(), Cb.leadingDim()))
q.wait()
PY
timeout 600 ncu --metrics $M --clock-control none -k regex:dgemm --launch-skip 1 --launch-count 1 --csv python /tmp/bw.py > gpurun_out/r2_ncu_dgemm_bitwise_4096.csv 2>&1; echo "bitwise rc=$?"
