# two ranks on one GPU (gloo host reduce) exercise the N>1 bench path
WAITSIM_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --reps 2000 > gpurun_out/bench_n2.log 2>&1; echo rc=$?
tail -3 gpurun_out/bench_n2.log | cut -c1-700
WAITSIM_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/bench_n2_ref.log 2>&1; echo rc=$?
tail -2 gpurun_out/bench_n2_ref.log | cut -c1-300
