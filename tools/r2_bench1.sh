set -x
mkdir -p gpurun_out
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2b_ref.json 2> gpurun_out/r2b_ref.err
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2b_n1.json 2> gpurun_out/r2b_n1.err; echo rc=$?
timeout 900 python bench.py --steps 20 --warmup 5 --force-rowsharded --no-cublas > gpurun_out/r2b_force.json 2> gpurun_out/r2b_force.err; echo rc=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 20 --warmup 5 --dist-backend gloo --same-gpu > gpurun_out/r2b_same2.json 2> gpurun_out/r2b_same2.err; echo rc=$?
